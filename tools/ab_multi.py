"""Same-box A/B of several builds over bench workloads (see ab_versions.py).

    python tools/ab_multi.py ROOT1,ROOT2,... wl1 [wl2 ...] [--reps 3]

Each (root, workload) runs in its own process, round-robin over the roots;
prints the median sampler-launch and step times per root.
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    reps = 3
    if "--reps" in sys.argv:
        reps = int(sys.argv[sys.argv.index("--reps") + 1])
        args.remove(str(reps))
    roots, names = args[0].split(","), args[1:]
    for name in names:
        rows = {r: [] for r in roots}
        for _ in range(reps):
            for r in roots:
                out = subprocess.run([sys.executable, os.path.join(HERE, "ab_versions.py"), "--one", r, name],
                                     capture_output=True, text=True)
                try:
                    rows[r].append(json.loads(out.stdout.strip().splitlines()[-1]))
                except Exception:
                    print(name, r, "error", out.stderr[-800:])
        for r in roots:
            if rows[r]:
                s = sorted(x["sampler_ms"] for x in rows[r])
                t = sorted(x["step_ms"] for x in rows[r])
                print(f"{name:22s} {os.path.basename(os.path.abspath(r)):8s} sampler {s[len(s)//2]:.4f} "
                      f"step {t[len(t)//2]:.4f}  {rows[r][0]['kernel']}", flush=True)


if __name__ == "__main__":
    main()
