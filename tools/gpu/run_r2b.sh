mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x --durations=10 > gpurun_out/r2b_gpu.log 2>&1
timeout 900 python bench.py --no-workloads > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
echo done
