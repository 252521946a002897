mkdir -p gpurun_out
python tools/sort_sweep.py > gpurun_out/r2d_sort.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "sort or permutation or host" > gpurun_out/r2d_tests.log 2>&1
timeout 900 python bench.py --workloads cfg1,cfg2,cfg3,cfg3-afps,cfg5-afps256-8192,cfg5-npdu-8192,cfg5-afps256-32768,cfg5-npdu-32768 --steps 10 > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
echo done
