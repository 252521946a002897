mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "tiny or bench_workload" > gpurun_out/group_gpu.log 2>&1
tail -3 gpurun_out/group_gpu.log
bash tools/gpu/run_envab.sh group1 PCS_GROUP "0 1" "cfg5-afps256-8192 cfg5-afps64-2048 cfg5-afps256-16384 cfg5-afps64-4096" | sort | uniq
