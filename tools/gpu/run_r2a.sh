mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
nproc >> gpurun_out/r2a_smi.txt
timeout 900 python -m pytest tests/test_gpu_bench_shapes.py -x -q -m gpu --durations=15 > gpurun_out/r2a_shapes.log 2>&1
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r2a_gpu.log 2>&1
echo done
