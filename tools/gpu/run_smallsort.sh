mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "sort or cfg1 or cfg2 or bench_workload" > gpurun_out/ss_gpu.log 2>&1
tail -1 gpurun_out/ss_gpu.log
for v in 0 1; do
  if [ $v = 1 ]; then export PCS_BK_SMALLOFF=1; fi
  echo "smalloff=$v"
  python tools/sort_sweep.py 1x2048 16x2048 64x2048 148x2048 64x4096 16x1024 256x2048 | sed 's/"copy_ms".*"perm_ms"/perm_ms/'
done
unset PCS_BK_SMALLOFF
python bench.py --workloads cfg1,cfg2,cfg5-afps256-2048,cfg5-npdu-2048 --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/ss_bench.json 2>/dev/null
python tools/design_tables.py gpurun_out/ss_bench.json 2>/dev/null | tail -5 || true
