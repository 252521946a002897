# e2e of bench workloads under an env knob: tools/gpu/run_e2e_env.sh TAG VAR "v1 v2" "wl1 wl2 ..."
mkdir -p gpurun_out
tag=$1; var=$2; vals=$3; wls=$4
for w in $wls; do
  for rep in 1 2 3; do
    for v in $vals; do
      out=$(env $var=$v python bench.py --workload $w --steps 30 --warmup 5 --no-workloads --no-cpu-baseline 2>/dev/null | tail -1)
      python - "$w" "$v" "$out" <<'PY' >> gpurun_out/${tag}.log
import json, sys
w, v, out = sys.argv[1], sys.argv[2], sys.argv[3]
try:
    e = json.loads(out)["e2e"]
    print(f"{w} {v} e2e_ms={e['ms_per_step']:.4f} median={e['median_ms']:.4f} min={e['min_ms']:.4f} h2d_floor={e['h2d_floor_ms']:.4f}")
except Exception as ex:
    print(w, v, "error", out[:200])
PY
    done
  done
done
cat gpurun_out/${tag}.log
