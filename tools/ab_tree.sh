#!/bin/bash
# Same-box A/B: this tree vs abtest/head on the given workloads (device ms/step, kernel ms)
W=${@:-cfg4 cfg3 cfg5-npdu-8192}
for r in 1 2 3; do
  for tree in . abtest/head; do
    for w in $W; do
      (cd $tree && timeout 120 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys
l=[x for x in sys.stdin if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
r=d.get('roofline') or {}
print('$tree', '$w', d.get('ms_per_step'), r.get('kernel_ms'))")
    done
  done
done
