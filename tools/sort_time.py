"""Time pcs.sort_axis on a (B, N, 3) cube batch (CUDA events, per call)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2208_08795_b200 as pcs  # noqa: E402
from paper_2208_08795_b200 import synth  # noqa: E402

B, N = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (1, 1 << 20)
x = torch.from_numpy(synth.uniform_cube(B, N, 1)).cuda()
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for _ in range(3):
    pcs.sort_axis(x, "x")
torch.cuda.synchronize()
ts = []
for i in range(20):
    flush.fill_(float(i))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    pcs.sort_axis(x, "x")
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(B, N, "ms", np.round(ts, 3).tolist())
