"""Host-side cost of one pcs.sample / sort_perm call (asynchronous; host
clock over 200 calls) and the device time of the same step replayed from a
CUDA graph. usage: host_overhead.py METHOD B N C M [K]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2208_08795_b200 as pcs  # noqa: E402
from paper_2208_08795_b200 import synth  # noqa: E402

meth, B, N, C, M = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
K = int(sys.argv[6]) if len(sys.argv) > 6 else None
x = torch.from_numpy(synth.primitives(B, N, 4, seed=1)).cuda()
perm = pcs.sort_perm(x, "x")
for name, fn in (("sample", lambda: pcs.sample(x, C, method=meth, m=M, k=K, _perm=perm)),
                 ("sort_perm", lambda: pcs.sort_perm(x, "x")),
                 ("step", lambda: pcs.sample(x, C, method=meth, m=M, k=K, _perm=pcs.sort_perm(x, "x")))):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    # device time from a graph replay
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    ts = []
    for _ in range(30):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts2 = []
    for _ in range(30):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts2.append(a.elapsed_time(b))
    print(f"{name:10s} host {1e3 * (t1 - t0) / 200:.4f} ms/call, queue drain {1e3 * (t2 - t0) / 200:.4f} "
          f"| eager events {np.median(ts2):.4f} ms | graph replay {np.median(ts):.4f} ms")
