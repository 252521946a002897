#!/bin/bash
# Full bench lines (value, e2e, cpu_baseline = the reference on the box's host cores) per workload
mkdir -p gpurun_out
for w in ${@:-cfg1 cfg2 cfg3 cfg3-afps cfg3-fps cfg4 cfg5-fps-8192 cfg5-afps256-32768 cfg5-npdu-8192}; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 2>/dev/null | tail -n 1 > gpurun_out/full_$w.json
  echo "$w rc=$?"
done
