"""Per-call latency of the reference-signature drop-in (host float64 cloud in,
host results out, one cloud per call)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2208_08795_b200 as pcs  # noqa: E402
from paper_2208_08795_b200 import synth  # noqa: E402

for n, c, m, k in ((2048, 512, 8, None), (2048, 512, 1, None), (32768, 8192, 32, 129)):
    pts = synth.uniform_cube(1, n, 1)[0].astype(np.float64)
    f = (lambda: pcs.npdu_afps(pts, c, m, k)) if k else (lambda: pcs.afps(pts, c, m))
    for _ in range(5):
        f()
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        f()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(n, c, m, k, "ms/call median %.3f min %.3f" % (float(np.median(ts)), min(ts)))
for n, c in ((8192, 2048), (32768, 1024)):
    pts = synth.uniform_cube(1, n, 2)[0].astype(np.float64)
    for _ in range(3):
        pcs.fps(pts, c)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        pcs.fps(pts, c)
        ts.append((time.perf_counter() - t0) * 1e3)
    print("fps", n, c, "ms/call median %.3f" % float(np.median(ts)))
for n in (2048, 8192, 32768, 131072):
    pts = synth.uniform_cube(1, n, 3)[0].astype(np.float64)
    for _ in range(3):
        pcs.exact_sort(pts, "x")
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        pcs.exact_sort(pts, "x")
        ts.append((time.perf_counter() - t0) * 1e3)
    print("exact_sort", n, "ms/call median %.3f" % float(np.median(ts)))
