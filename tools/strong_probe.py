"""cfg4's per-GPU share under strong scaling (128 / N clouds per GPU): the
sampler launch alone on that many clouds, CUDA-graph replay, L2 flushed.
usage: strong_probe.py [clouds ...]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2208_08795_b200 as pcs  # noqa: E402

w = bench.WORKLOADS["cfg4"]
xa = torch.from_numpy(bench.make_input(w)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for b in [int(a) for a in sys.argv[1:]] or [128, 64, 32, 16]:
    x = xa[:b].contiguous()
    fn = lambda: pcs.sample(x, w["C"], method=w["method"], m=w["M"], k=w["K"])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for i in range(20):
        flush.fill_(i)
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(e))
    ms = float(np.median(ts))
    print(f"clouds {b:4d} ({128 // b} GPUs) {ms:.4f} ms  -> {b * w['C'] / ms / 1e6:.3f} G pts/s per GPU, "
          f"{128 * w['C'] / ms / 1e6:.3f} G pts/s job  {pcs.kernel_family(w['method'], w['N'], w['M'], w['K'], batch=b, full=True)}")
