"""Print the `workloads` object of a bench.py JSON line as a table."""
import json
import sys

line = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
wl = line.get("workloads") or {}
print(f"{'workload':22s} {'ms':>8s} {'sort':>7s} {'samp':>8s} {'pts/s':>9s} {'kernel':20s} "
      f"{'fp64':>5s} {'sortHBM':>7s} {'e2e ms':>7s} {'cpu pts/s':>9s} {'e2e/cpu':>7s} par")
for k, e in wl.items():
    if k.startswith("_"):
        continue
    if "ms_per_step" not in e:
        print(k, e)
        continue
    cpu = e.get("cpu_baseline", {}).get("value")
    par = e.get("parity", {})
    print(f"{k:22s} {e['ms_per_step']:8.3f} {e['sort_ms']:7.3f} {e['sampler_ms']:8.3f} "
          f"{e['sampled_pts_per_s']:9.2e} {e['kernel'][:20]:20s} "
          f"{(e['fp64_frac_algorithmic'] or 0):5.2f} {e.get('sort_hbm_frac', 0):7.3f} "
          f"{e['e2e']['ms_per_step']:7.3f} {(cpu or 0):9.2e} {e.get('e2e_vs_cpu', 0):7.1f} "
          f"{par.get('mismatches')}/{par.get('clouds')}")
print("wall", wl.get("_wall_s"))
