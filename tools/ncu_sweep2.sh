#!/bin/bash
# r02: one ncu --set full capture per BASELINE workload of (a) the sampler
# kernel and (b) the axis sort kernel when the workload sorts -- the third
# launch of each (after bench.py's warm-up) -- summarised on the box by
# tools/ncu_summary.py into gpurun_out/ncu2_<workload>_{sampler,sort}.json.
# usage: tools/ncu_sweep2.sh [workloads...]
W=${@:-cfg1 cfg2 cfg3 cfg3-afps cfg3-fps cfg4 cfg5-fps-2048 cfg5-fps-4096 cfg5-fps-8192 cfg5-fps-16384 cfg5-fps-32768 cfg5-afps4-8192 cfg5-afps16-8192 cfg5-afps64-8192 cfg5-afps256-8192 cfg5-afps4-32768 cfg5-afps16-32768 cfg5-afps64-32768 cfg5-afps256-32768 cfg5-npdu-2048 cfg5-npdu-8192 cfg5-npdu-16384 cfg5-npdu-32768 cfg5-1m stream-fps-1m}
mkdir -p gpurun_out
for w in $W; do
  for what in sampler sort; do
    if [ $what = sampler ]; then rx="regex:fps_full|fps_cluster|npdu_|morton_|rows_kernel|stream_sector"; else rx="regex:bucket|radix|bitonic|rs_scatter"; fi
    timeout 900 ncu --set full --clock-control none -k "$rx" -s 2 -c 1 \
      -o gpurun_out/ncu2_${w}_$what -f python bench.py --workload $w --steps 1 --warmup 3 \
      --no-cpu-baseline --no-e2e --no-workloads > gpurun_out/ncu2_${w}_$what.log 2>&1
    if [ -f gpurun_out/ncu2_${w}_$what.ncu-rep ]; then
      python tools/ncu_summary.py gpurun_out/ncu2_${w}_$what.ncu-rep > gpurun_out/ncu2_${w}_$what.json
      [ "$w" = cfg4 ] || rm -f gpurun_out/ncu2_${w}_$what.ncu-rep
    fi
    echo "$w $what done"
  done
done
