"""H2D / D2H bandwidth on the box vs the pipelined public-API path (cfg4)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_08795_b200 as pcs  # noqa: E402
from paper_2208_08795_b200 import synth  # noqa: E402

B, N, C = 128, 32768, 8192
x = torch.from_numpy(synth.lidar_sweep(B, seed=1) if hasattr(synth, "lidar_sweep") else
                     synth.uniform_cube(B, N, 1)).contiguous().pin_memory()
d = torch.empty(x.shape, dtype=x.dtype, device="cuda")
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    ev0.record(); d.copy_(x, non_blocking=True); ev1.record(); torch.cuda.synchronize()
    ts.append(ev0.elapsed_time(ev1))
print(f"H2D {x.numel()*4/1e6:.1f} MB: {min(ts):.3f} ms min, {np.median(ts):.3f} med -> "
      f"{x.numel()*4/min(ts)/1e6:.1f} GB/s")
o = torch.empty((B, C), dtype=torch.int32, device="cuda")
oh = torch.empty((B, C), dtype=torch.int32).pin_memory()
ts = []
for _ in range(10):
    ev0.record(); oh.copy_(o, non_blocking=True); ev1.record(); torch.cuda.synchronize()
    ts.append(ev0.elapsed_time(ev1))
print(f"D2H {o.numel()*4/1e6:.1f} MB: {min(ts):.3f} ms -> {o.numel()*4/min(ts)/1e6:.1f} GB/s")
for ch in (0, 4, 8, 16):
    def run():
        return pcs.sample_host_batch(x, C, method="npdu_afps", m=32, k=129, chunks=ch)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        ev0.record(); run(); ev1.record()
        torch.cuda.synchronize(); ts.append(ev0.elapsed_time(ev1))
    t0 = time.perf_counter()
    for _ in range(10):
        run()
    wall = (time.perf_counter() - t0) / 10 * 1e3
    print(f"chunks {ch or 'default'}: e2e {min(ts):.3f} ms min, {np.median(ts):.3f} med, wall {wall:.3f} ms")
