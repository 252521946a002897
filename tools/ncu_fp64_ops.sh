#!/bin/bash
# FP64 instruction mix of the sampler kernels (DFMA must be 0: the reference
# evaluates ((dx*dx + dy*dy) + dz*dz) without contraction) -> gpurun_out/fp64_ops_<w>.csv
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum
for w in ${@:-cfg1 cfg2 cfg3 cfg4 cfg5-fps-8192 cfg5-afps256-32768}; do
  timeout 300 ncu --metrics $M --clock-control none -k "regex:fps_full|npdu_|morton_|rows_kernel|stream_sector" \
    -s 2 -c 1 --csv --log-file gpurun_out/fp64_ops_$w.csv python bench.py --workload $w --steps 1 \
    --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "$w rc=$?"
done
