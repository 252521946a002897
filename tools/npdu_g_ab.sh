#!/bin/bash
# A/B of warps per CTA for the TMEM NPDU kernel (PCS_NPDU_G) on cfg4 and
# cfg5-npdu-32768: 4 (default for multi-wave batches), 6 and 9 (18 warps/SM).
for g in 4 6 9 4 6 9; do
  for w in cfg4 cfg5-npdu-32768; do
    PCS_NPDU_G=$g timeout 120 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 \
    | python -c "import json,sys
l=[x for x in sys.stdin if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
r=d.get('roofline') or {}
print('G=$g', '$w', d.get('ms_per_step'), r.get('kernel_ms'))"
  done
done
