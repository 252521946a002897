mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "tiny or bench_workload or random or batched or identities" > gpurun_out/tiny_gpu.log 2>&1
tail -3 gpurun_out/tiny_gpu.log
bash tools/gpu/run_envab.sh tiny1 PCS_TINY "0 1" "cfg5-afps256-2048 cfg5-afps256-4096 cfg5-afps256-8192 cfg5-afps64-2048" | sort | uniq
