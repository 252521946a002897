#!/bin/bash
# The shared-memory NPDU warp kernel forced (PCS_NPDU_TMEM=0, PCS_NPDU_WIDE=0)
# on cfg4 / cfg3 / cfg5-npdu-8192: this tree vs abtest/head (same box).
for r in 1 2; do
  for tree in . abtest/head; do
    for w in cfg4 cfg3 cfg5-npdu-8192; do
      (cd $tree && PCS_NPDU_TMEM=0 PCS_NPDU_WIDE=0 timeout 120 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys
l=[x for x in sys.stdin if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
r=d.get('roofline') or {}
print('$tree', '$w', d.get('ms_per_step'), r.get('kernel_ms'))")
    done
  done
done
