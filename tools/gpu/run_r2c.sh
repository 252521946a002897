mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "permutation or sort or host" > gpurun_out/r2c_perm.log 2>&1
timeout 900 python -m pytest tests/test_gpu_bench_shapes.py -q -m gpu -x > gpurun_out/r2c_shapes.log 2>&1
timeout 900 python bench.py --workloads cfg2,cfg3,cfg3-afps,cfg5-afps256-8192,cfg5-npdu-8192,cfg5-afps256-32768,cfg5-npdu-32768,cfg5-fps-8192,cfg5-1m --steps 10 > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
echo done
