#!/bin/bash
# Same-box A/B of an environment switch over bench workloads: for each
# workload, alternate OFF/ON runs (3 each), print ms_per_step and kernel_ms.
# usage: tools/ab_bench.sh VAR "wl1 wl2 ..." [steps]
VAR=$1; WLS=$2; STEPS=${3:-20}
for w in $WLS; do
  for rep in 1 2 3; do
    for v in 0 1; do
      out=$(env $VAR=$v python bench.py --workload $w --steps $STEPS --warmup 5 --no-workloads --no-e2e --no-cpu-baseline 2>/dev/null | tail -1)
      python - "$w" "$v" "$out" <<'PY'
import json, sys
w, v, out = sys.argv[1], sys.argv[2], sys.argv[3]
try:
    d = json.loads(out)
    print(f"{w} {v} step_ms={d['ms_per_step']:.4f} kernel_ms={d['roofline']['kernel_ms']:.4f} frac={d['roofline']['frac']:.3f}")
except Exception as e:
    print(w, v, "error", out[:200])
PY
    done
  done
done
