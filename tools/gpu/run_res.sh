mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "stream or bench_workload or forced or engine or 1m" > gpurun_out/res_gpu.log 2>&1
tail -2 gpurun_out/res_gpu.log
bash tools/gpu/run_envab.sh res1 PCS_RESIDENT "0 1" "stream-fps-1m" | sort | uniq
