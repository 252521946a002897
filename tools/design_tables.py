"""DESIGN.md §4a tables from one bench.py JSON line.

    python tools/design_tables.py gpurun_out/<run>_bench.json > /tmp/tables.md
"""
import json
import sys


def fmt(v, f="{:.3f}"):
    return "-" if v is None else f.format(v)


def main(path):
    d = json.loads(open(path).read().strip().splitlines()[-1])
    r, e = d["roofline"], d["e2e"]
    print("**Headline (cfg4, N=1):** "
          f"value {d['value']:.3e} sampled pts/s, step {d['ms_per_step']:.4f} ms "
          f"(graph replay; eager {d.get('eager_ms_per_step', 0):.4f}), sampler kernel "
          f"{r['kernel_ms']:.4f} ms = {r['achieved']:.2f} of {r['peak']} FP64 TFLOP/s "
          f"(frac {r['frac']:.3f}), ncu issue {r['issue']['frac']:.2f} of 4 IPC; e2e "
          f"{e['ms_per_step']:.3f} ms (median {e.get('median_ms', 0):.3f}, H2D floor "
          f"{e['h2d_floor_ms']:.3f}) = {e['value']:.3e} pts/s; cpu_baseline "
          f"{d['cpu_baseline']['value']:.3e} pts/s on {d['cpu_baseline']['cores']} cores; "
          f"parity {d['parity']['mismatches']} mismatches over {d['parity']['clouds']} clouds; "
          f"clocks {d['clocks']['sm_mhz']:.0f} MHz {d['clocks']['reasons']}.")
    print()
    print("| workload | step ms | eager ms | sort ms | sampler ms | kernel | FP64 frac (alg / ncu exec) "
          "| sort HBM frac | e2e ms | e2e / 16-core ref | parity |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for k, v in d["workloads"].items():
        if not isinstance(v, dict) or "ms_per_step" not in v:
            continue
        par = v.get("parity", {})
        print(f"| {k} | {v['ms_per_step']:.4f} | {fmt(v.get('eager_ms_per_step'), '{:.4f}')} | "
              f"{v['sort_ms']:.4f} | {v['sampler_ms']:.4f} | `{v['kernel']}` | "
              f"{fmt(v.get('fp64_frac_algorithmic'), '{:.2f}')} / "
              f"{fmt(v.get('fp64_pipe_executed_frac'), '{:.2f}')} | "
              f"{fmt(v.get('sort_hbm_frac'), '{:.2f}')} | {v['e2e']['ms_per_step']:.3f} | "
              f"{fmt(v.get('e2e_vs_cpu'), '{:.1f}')}x | "
              f"{par.get('mismatches', '-')}/{par.get('clouds', '-')} |")


if __name__ == "__main__":
    main(sys.argv[1])
