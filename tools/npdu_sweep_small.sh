#!/bin/bash
# NPDU workloads, device-resident ms/step and kernel ms (two repetitions)
for r in 1 2; do
  for w in cfg3 cfg4 cfg5-npdu-2048 cfg5-npdu-8192 cfg5-npdu-32768; do
    timeout 120 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys
l=[x for x in sys.stdin if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
r=d.get('roofline') or {}
print('$w', d.get('ms_per_step'), r.get('kernel_ms'))"
  done
done
