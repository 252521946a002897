mkdir -p gpurun_out
timeout 900 python bench.py --workloads cfg3,cfg3-afps,cfg5-afps256-8192,cfg5-afps64-8192,cfg5-afps256-32768 --steps 10 --no-e2e > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
echo done
