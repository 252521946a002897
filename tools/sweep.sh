#!/bin/bash
# Quick per-workload timing table (device-resident, no e2e / cpu legs).
# usage: tools/sweep.sh [workloads...]  -> prints "workload ms_per_step pts/s kernel_ms fp64_frac"
W=${@:-cfg1 cfg2 cfg3 cfg3-afps cfg3-fps cfg4 cfg5-fps-2048 cfg5-afps16-8192 cfg5-npdu-8192 cfg5-afps256-32768}
for w in $W; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 \
  | python -c "import json,sys
l=[x for x in sys.stdin if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
r=d.get('roofline') or {}
print('$w', d.get('ms_per_step'), d.get('value'), r.get('kernel_ms'), r.get('frac'))"
done
