"""`pcsample sample` / `pcsample bench` flows on the GPU path (SURVEY §8(f2, f4)).

    python -m paper_2208_08795_b200.cli sample --in cloud.bin --format f32_bin \\
        --method npdu-afps --c 512 --m 32 --k 16 --seed 7 --out idx.txt
    python -m paper_2208_08795_b200.cli bench --method fps,afps,npdu-afps --n 2048,8192 \\
        --m-list 1,8,32 --k-list 16 --c 512 --trials 3 --out bench.csv

Mirrors proj/tools/pcsample_main.cpp:275-368: `sample` writes one index per
line and prints the stats JSON line (dist_evals, dist_writes, argmax_scans,
iterations, wall_seconds); `bench` writes the reference's CSV schema. Clouds
for `bench` are uniform cubes in [-1, 1]^3 (seed ^ n), sorted along x, or a
file (--in). Exit codes: 0 ok, 1 runtime/argument error, 2 usage error.
"""
from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

from . import _core, harness, synth


def _sample(a) -> int:
    cloud = _core.read_cloud(a.input, a.format)
    if a.sort:
        cloud = _core.exact_sort(cloud, a.sort)
    t0 = time.perf_counter()
    meth = a.method
    if meth == "fps":
        idx, _, st = _core.fps(cloud, a.c, seed=a.seed, first=a.first)
    elif meth == "afps":
        idx, _, st = _core.afps(cloud, a.c, a.m, seed=a.seed, first=a.first)
    elif meth == "npdu-fps":
        idx, _, st = _core.npdu_fps(cloud, a.c, a.k, seed=a.seed, first=a.first)
    elif meth == "npdu-afps":
        idx, _, st = _core.npdu_afps(cloud, a.c, a.m, a.k, seed=a.seed, first=a.first)
    else:
        raise ValueError(f"unknown or non-GPU method: {meth}")
    wall = time.perf_counter() - t0
    with open(a.out, "w") as f:
        f.write("".join(f"{int(i)}\n" for i in idx))
    line = json.dumps({**{k: int(v) for k, v in st.items()}, "wall_seconds": wall})
    print(line)
    if a.stats_json:
        with open(a.stats_json, "w") as f:
            f.write(line + "\n")
    return 0


def _ints(s):
    return [int(x) for x in s.split(",") if x]


def _bench(a) -> int:
    opts = harness.BenchOptions(methods=a.method.split(","), n_values=_ints(a.n),
                                m_values=_ints(a.m_list), k_values=_ints(a.k_list), c=a.c,
                                trials=a.trials, seed=a.seed, first=a.first)
    if a.input:
        cloud = _core.read_cloud(a.input, a.format)
        opts.n_values = [len(cloud)]
        provider = lambda n: cloud  # noqa: E731
    else:
        def provider(n):
            pts = synth.uniform_cube(1, n, a.seed ^ n)[0].astype(np.float64)
            return _core.exact_sort(pts, "x")
    rows = harness.run_bench(opts, provider)
    csv = harness.bench_csv(rows)
    if a.out:
        with open(a.out, "w") as f:
            f.write(csv)
    else:
        sys.stdout.write(csv)
    print(f"{len(rows)} rows", file=sys.stderr)
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="pcsample-gpu")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("sample")
    s.add_argument("--in", dest="input", required=True)
    s.add_argument("--format", default="f32_bin")
    s.add_argument("--method", default="npdu-afps")
    s.add_argument("--c", type=int, required=True)
    s.add_argument("--m", type=int, default=1)
    s.add_argument("--k", type=int, default=1)
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--first", default="random", choices=["random", "fixed"])
    s.add_argument("--sort", default=None, choices=["x", "y", "z"])
    s.add_argument("--out", required=True)
    s.add_argument("--stats-json", default=None)
    b = sub.add_parser("bench")
    b.add_argument("--method", default="fps,afps,npdu-afps")
    b.add_argument("--n", default="2048")
    b.add_argument("--m-list", default="1")
    b.add_argument("--k-list", default="1")
    b.add_argument("--c", type=int, default=512)
    b.add_argument("--trials", type=int, default=1)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--first", default="random", choices=["random", "fixed"])
    b.add_argument("--in", dest="input", default=None)
    b.add_argument("--format", default="f32_bin")
    b.add_argument("--out", default=None)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    try:
        return _sample(a) if a.cmd == "sample" else _bench(a)
    except (ValueError, RuntimeError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
