mkdir -p gpurun_out
for w in cfg1 cfg2 cfg5-afps64-2048; do for rep in 1 2 3; do for root in abtest/old .; do
 out=$(cd $root && python bench.py --workload $w --steps 50 --warmup 5 --no-workloads --no-cpu-baseline 2>/dev/null | tail -1)
 python - "$w" "$root" "$out" <<'PY' >> gpurun_out/e2e1.log
import json, sys
w, v, out = sys.argv[1], sys.argv[2], sys.argv[3]
try:
    e = json.loads(out)["e2e"]
    print(f"{w} {v} e2e_ms={e['ms_per_step']:.4f} median={e['median_ms']:.4f} min={e['min_ms']:.4f}")
except Exception as ex:
    print(w, v, "error", out[:200])
PY
done; done; done
cat gpurun_out/e2e1.log
