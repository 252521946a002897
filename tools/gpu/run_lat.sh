mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "npdu or cfg4 or bench_workload or random or identities or kats or goldens" > gpurun_out/lat2_gpu.log 2>&1
tail -2 gpurun_out/lat2_gpu.log
for v in 0 1; do echo "PCS_NPDU_LAT=$v"; PCS_NPDU_LAT=$v python tools/strong_probe.py 16 8 4 2 1; done
