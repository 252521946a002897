"""Collect gpurun_out/ncu2_<workload>_{sampler,sort}.json (tools/ncu_sweep2.sh)
into profiles/r02_ncu_sweep.json and refresh profiles/ncu_traffic.json, the
per-workload ncu facts bench.py reports beside its live numbers (traffic,
issue rate, executed FP64 fraction)."""
import glob
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
# merge into the committed sweep (a partial re-run refreshes its workloads only)
_prev = os.path.join(ROOT, "profiles", "r02_ncu_sweep.json")
sweep = json.load(open(_prev)) if os.path.exists(_prev) else {}
for path in sorted(glob.glob(os.path.join(src, "ncu2_*_*.json"))):
    m = re.match(r"ncu2_(.+)_(sampler|sort)\.json$", os.path.basename(path))
    try:
        recs = json.load(open(path))
    except ValueError:
        continue
    if not recs:
        continue
    sweep.setdefault(m.group(1), {})[m.group(2)] = recs[0]
with open(os.path.join(ROOT, "profiles", "r02_ncu_sweep.json"), "w") as f:
    json.dump(sweep, f, indent=1)
traffic = {}
for w, d in sweep.items():
    s = d.get("sampler")
    if not s or "dram_bytes" not in s:
        continue
    ev = (s.get("dadd_thread_inst", 0) or 0) / 5.0  # 5 DADD (3 sub + 2 add) per evaluation
    traffic[w] = {"kernel": s["kernel"], "dram_bytes": s["dram_bytes"],
                  "ipc_per_sm": s.get("ipc_per_sm"), "fp64_pipe_pct": s.get("fp64_pipe_pct"),
                  "xu_pipe_pct": s.get("xu_pipe_pct"), "alu_pipe_pct": s.get("alu_pipe_pct"),
                  "duration_ns": s.get("duration_ns"), "executed_evaluations": ev,
                  "dfma_thread_inst": s.get("dfma_thread_inst"),
                  "source": f"profiles/r02_ncu_sweep.json[{w}] (tools/ncu_sweep2.sh: ncu --set "
                            "full, third sampler launch of bench.py --workload " + w + ")"}
    if "sort" in d:
        traffic[w]["sort"] = {k: d["sort"].get(k) for k in ("kernel", "duration_ns", "dram_bytes",
                                                           "ipc_per_sm", "warp_instructions")}
with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
    json.dump(traffic, f, indent=1)
print(len(sweep), "workloads;", len(traffic), "with a sampler capture")
