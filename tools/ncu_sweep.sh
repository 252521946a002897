#!/bin/bash
# One ncu --set full capture of the sampler kernel per BASELINE workload
# (third launch: after warm-up), summarised on the box with
# tools/ncu_summary.py into gpurun_out/ncu_<workload>.json (the reports
# themselves are too large to bring back).
# usage: tools/ncu_sweep.sh [workloads...]
W=${@:-cfg1 cfg2 cfg3 cfg3-afps cfg3-fps cfg4 cfg5-fps-2048 cfg5-fps-8192 cfg5-fps-32768 cfg5-afps256-32768 cfg5-npdu-8192 cfg5-npdu-32768 cfg5-1m}
mkdir -p gpurun_out
for w in $W; do
  timeout 600 ncu --set full --clock-control none \
    -k "regex:fps_full|npdu_|morton_|rows_kernel|stream_sector" -s 2 -c 1 \
    -o gpurun_out/ncu_$w -f python bench.py --workload $w --steps 1 --warmup 3 \
    --no-cpu-baseline --no-e2e > gpurun_out/ncu_$w.log 2>&1
  echo "$w rc=$?"
  python tools/ncu_summary.py gpurun_out/ncu_$w.ncu-rep > gpurun_out/ncu_$w.json && rm -f gpurun_out/ncu_$w.ncu-rep
done
