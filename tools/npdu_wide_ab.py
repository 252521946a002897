"""A/B of the NPDU kernel families on the device (CUDA events, median of 10):
PCS_NPDU_WIDE=0 (one warp per sector: TMEM / shared memory) against the
W-warp latency form, over batch sizes. usage: npdu_wide_ab.py [cfg4|cfg3|cfg5n]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2208_08795_b200 as pcs  # noqa: E402
from paper_2208_08795_b200 import synth  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
if which == "cfg4":
    full = torch.from_numpy(synth.lidar_sweep(128, seed=1)).cuda()
    N, C, M, K, Bs = 32768, 8192, 32, 129, (1, 2, 4, 8, 16, 24, 32, 64, 128)
elif which == "cfg3":
    full = pcs.sort_axis(torch.from_numpy(synth.primitives(64, 8192, 6, seed=3)).cuda(), "x")[0]
    N, C, M, K, Bs = 8192, 2048, 16, 65, (1, 4, 16, 32, 64)
else:
    full = pcs.sort_axis(torch.from_numpy(synth.uniform_cube(256, 8192, 1)).cuda(), "x")[0]
    N, C, M, K, Bs = 8192, 2048, 16, 65, (8, 32, 64, 128, 256)


def t_ms(x):
    for _ in range(2):
        pcs.sample(x, C, method="npdu_afps", m=M, k=K)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pcs.sample(x, C, method="npdu_afps", m=M, k=K)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for B in Bs:
    x = full[:B].contiguous()
    row = []
    for knob in ("0", "100000000"):
        os.environ["PCS_NPDU_WIDE"] = knob
        row.append(t_ms(x))
    print(f"{which} B={B:4d} sectors={B * M:5d} one_warp {row[0]:.4f} ms  wide {row[1]:.4f} ms",
          flush=True)
