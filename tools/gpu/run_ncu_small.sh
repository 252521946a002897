mkdir -p gpurun_out
for wl in cfg1 cfg2; do
  ncu --set full --clock-control none --import-source on -k regex:fps_full -s 3 -c 1 -o gpurun_out/ncu_$wl -f python bench.py --workload $wl --no-workloads --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/ncu_$wl.log 2>&1
done
echo done
