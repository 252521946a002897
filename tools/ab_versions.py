"""Same-box A/B of two builds of the package over bench workloads.

    python tools/ab_versions.py ROOT_A ROOT_B wl1 [wl2 ...] [--reps 3]

ROOT_* is a directory holding a built ``paper_2208_08795_b200`` (e.g. the
repo itself and ``abtest/old``, a ``git archive`` of an older commit built
in place). Each (root, workload) runs in its own process, alternating
A/B/A/B; each prints the median sampler-launch time and the median step
(sort + sampler) over 20 launches (CUDA events, L2 flushed between them).
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)


def one(root, name):
    sys.path.insert(0, root)
    sys.path.insert(1, REPO)
    import numpy as np
    import torch

    import paper_2208_08795_b200 as pcs  # before bench (which puts the repo first on sys.path)

    import bench

    assert os.path.dirname(os.path.dirname(pcs.__file__)) == os.path.abspath(root), pcs.__file__
    w = bench.WORKLOADS[name]
    x = torch.from_numpy(bench.make_input(w)).cuda()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    perm = pcs.sort_perm(x, w["sort"]) if w["sort"] else None

    def sample():
        if perm is None:
            return pcs.sample(x, w["C"], method=w["method"], m=w["M"], k=w["K"])
        return pcs.sample(x, w["C"], method=w["method"], m=w["M"], k=w["K"], _perm=perm)

    def step():
        if w["sort"]:
            p = pcs.sort_perm(x, w["sort"])
            return pcs.sample(x, w["C"], method=w["method"], m=w["M"], k=w["K"], _perm=p)
        return sample()

    res = {}
    for label, fn in (("sampler_ms", sample), ("step_ms", step)):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(20):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[label] = float(np.median(ts))
    res["kernel"] = pcs.kernel_family(w["method"], w["N"], w["M"], w["K"], batch=w["B"], full=True)
    print(json.dumps(res))


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    reps = 3
    if "--reps" in sys.argv:
        reps = int(sys.argv[sys.argv.index("--reps") + 1])
        args.remove(str(reps))
    ra, rb, names = args[0], args[1], args[2:]
    for name in names:
        rows = {ra: [], rb: []}
        for _ in range(reps):
            for r in (ra, rb):
                out = subprocess.run([sys.executable, __file__, "--one", r, name],
                                     capture_output=True, text=True)
                try:
                    rows[r].append(json.loads(out.stdout.strip().splitlines()[-1]))
                except Exception:
                    print(name, r, "error", out.stderr[-800:])
        for r in (ra, rb):
            if rows[r]:
                s = sorted(x["sampler_ms"] for x in rows[r])
                t = sorted(x["step_ms"] for x in rows[r])
                print(f"{name:22s} {os.path.basename(os.path.abspath(r)):8s} sampler {s[len(s)//2]:.4f} "
                      f"step {t[len(t)//2]:.4f}  {rows[r][0]['kernel']}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        one(sys.argv[2], sys.argv[3])
    else:
        main()
