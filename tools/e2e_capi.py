"""e2e through the C-ABI host batch entry vs the Python pipelined path (cfg4)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_08795_b200 as pcs  # noqa: E402
from paper_2208_08795_b200 import synth  # noqa: E402

x = torch.from_numpy(synth.lidar_sweep(128, seed=4)).pin_memory()
C = 8192
for name, fn in (("python", lambda: pcs.sample(x, C, method="npdu_afps", m=32, k=129)),
                 ("capi", lambda: pcs.sample_host_batch(x, C, method="npdu_afps", m=32, k=129))):
    t_end = time.perf_counter() + 0.6
    while time.perf_counter() < t_end:
        fn()
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(name, "ms min %.3f med %.3f" % (min(ts), float(np.median(ts))))
for ch in (2, 4, 8, 16):
    ts = []
    for _ in range(15):
        t0 = time.perf_counter()
        pcs.sample_host_batch(x, C, method="npdu_afps", m=32, k=129, chunks=ch)
        ts.append((time.perf_counter() - t0) * 1e3)
    print("capi chunks", ch, "med %.3f" % float(np.median(ts)))
