"""Time one pcs.sample configuration on the device (CUDA events, median of 10).
usage: time_call.py METHOD B N C [M] [K]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2208_08795_b200 as pcs  # noqa: E402
from paper_2208_08795_b200 import synth  # noqa: E402

meth, B, N, C = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
M = int(sys.argv[5]) if len(sys.argv) > 5 else 1
K = int(sys.argv[6]) if len(sys.argv) > 6 else None
x = pcs.sort_axis(torch.from_numpy(synth.uniform_cube(B, N, 1)).cuda(), "x")[0]
for _ in range(2):
    pcs.sample(x, C, method=meth, m=M, k=K)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    pcs.sample(x, C, method=meth, m=M, k=K)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(meth, B, N, C, M, K, pcs.kernel_family(meth, N, M, K, batch=B), "ms", round(float(np.median(ts)), 3))
