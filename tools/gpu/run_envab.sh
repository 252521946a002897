# one env knob over several values, same box: tools/gpu/run_envab.sh TAG VAR "v1 v2 ..." "wl1 wl2 ..."
mkdir -p gpurun_out
tag=$1; var=$2; vals=$3; wls=$4
for w in $wls; do
  for rep in 1 2; do
    for v in $vals; do
      out=$(env $var=$v python bench.py --workload $w --steps 20 --warmup 5 --no-workloads --no-e2e --no-cpu-baseline 2>/dev/null | tail -1)
      python - "$w" "$v" "$out" <<'PY' >> gpurun_out/${tag}.log
import json, sys
w, v, out = sys.argv[1], sys.argv[2], sys.argv[3]
try:
    d = json.loads(out)
    print(f"{w} {v} step_ms={d['ms_per_step']:.4f} kernel_ms={d['roofline']['kernel_ms']:.4f}")
except Exception as e:
    print(w, v, "error", out[:200])
PY
    done
  done
done
cat gpurun_out/${tag}.log
