# A/B: windowed fp32 sectors above PCS_NPDU_BIG_MIN points take the TMEM Morton engine in window mode
for v in 4096 256; do
  for w in cfg5-npdu-32768 cfg5-npdu-16384 cfg4 cfg3; do
    PCS_NPDU_BIG_MIN=$v timeout 120 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys
l=[x for x in sys.stdin if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
r=d.get('roofline') or {}
print('BIG_MIN=$v', '$w', d.get('ms_per_step'), r.get('kernel_ms'))"
  done
done
