"""Regenerate tests/golden/*.npz from the REAL reference.

Runs the unmodified reference hot path (oracle/_ref/libpcsref.so, built by
`make -C oracle` from /root/reference/proj/src) on seeded inputs and stores
inputs + outputs. Needs /root/reference at build time only; the fixtures are
committed and travel to the GPU box.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import Reference  # noqa: E402
from paper_2208_08795_b200 import synth  # noqa: E402

M = {"fps": 1, "afps": 2, "npdu_fps": 3, "npdu_afps": 4}


def cases():
    """(name, points float64 (N,3), method, c, m, k, first, seed)."""
    out = []
    line = np.array([[x, 0.0, 0.0] for x in range(8)])
    out += [("line4_fps_c%d" % c, line[:4], "fps", c, 1, 0, "fixed", 0) for c in (2, 3, 4)]
    out += [("line8_npdu_k2", line, "npdu_fps", 3, 1, 2, "fixed", 0),
            ("line8_npdu_k4", line, "npdu_fps", 3, 1, 4, "fixed", 0)]
    rng = np.random.default_rng(20220818)
    for t in range(48):
        n = int(rng.integers(4, 700))
        c = int(rng.integers(1, n + 1))
        m = int(rng.integers(1, c + 1))
        k = int(rng.integers(1, 80))
        meth = ["fps", "afps", "npdu_fps", "npdu_afps"][t % 4]
        pts = synth.random_cloud(n, 1000 + t)
        if t % 5 == 0:
            pts[: n // 2] = 1.0  # coincident points force zero-distance ties
        out.append((f"rand{t}_{meth}", pts, meth, c, m, k, "random" if t % 2 else "fixed", t))
    # fp32 batches shaped like the BASELINE configs (small B)
    cube = synth.uniform_cube(1, 2048, 0)[0].astype(np.float64)
    cube = cube[np.argsort(cube[:, 0], kind="stable")]
    out.append(("cfg1_fps_2048_512", cube, "fps", 512, 1, 0, "fixed", 0))
    prim = synth.primitives(2, 2048, 4, seed=1)
    for b in range(2):
        p = prim[b].astype(np.float64)
        p = p[np.argsort(p[:, 0] + 0.0, kind="stable")]
        out.append((f"cfg2_afps_m8_b{b}", p, "afps", 512, 8, 0, "fixed", 0))
    prim3 = synth.primitives(1, 8192, 6, seed=3)[0].astype(np.float64)
    prim3 = prim3[np.argsort(prim3[:, 0] + 0.0, kind="stable")]
    out.append(("cfg3_npdu_afps_m16_k65", prim3, "npdu_afps", 2048, 16, 65, "fixed", 0))
    out.append(("cfg3_afps_m16", prim3, "afps", 2048, 16, 0, "fixed", 0))
    lid = synth.lidar_sweep(1, seed=4)[0].astype(np.float64)
    out.append(("cfg4_npdu_afps_m32_k129", lid, "npdu_afps", 8192, 32, 129, "fixed", 0))
    out.append(("cfg4_npdu_afps_m32_k129_random", lid, "npdu_afps", 8192, 32, 129, "random", 7))
    return out


def main():
    ref = Reference()
    blobs = {}
    for name, pts, meth, c, m, k, first, seed in cases():
        idx, sec, st = ref.sample(meth, pts, c, m, k, first, seed)
        blobs[name] = dict(points=pts, method=M[meth], c=c, m=m, k=k,
                           random_first=int(first == "random"), seed=np.uint64(seed),
                           indices=idx, sector_of=sec, stats=st)
    flat = {f"{n}/{k}": v for n, d in blobs.items() for k, v in d.items()}
    np.savez_compressed(os.path.join(HERE, "samplers.npz"), **flat)
    # exact_sort goldens: ties, signed zeros, duplicates
    srt = {}
    rng = np.random.default_rng(7)
    for t in range(6):
        n = int(rng.integers(1, 3000))
        pts = np.round(rng.normal(size=(n, 3)), 1)  # many ties
        pts[rng.integers(0, n, size=max(1, n // 10)), t % 3] = -0.0
        for axis in range(3):
            srt[f"s{t}_a{axis}/points"] = pts
            srt[f"s{t}_a{axis}/sorted"] = ref.exact_sort(pts, axis)
    np.savez_compressed(os.path.join(HERE, "exact_sort.npz"), **srt)
    print("wrote", len(blobs), "sampler cases and", len(srt) // 2, "sort cases")


if __name__ == "__main__":
    main()
