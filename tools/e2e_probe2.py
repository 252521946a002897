"""Per-call host-clock times of the e2e host-batch call and per-call event
times of the sort for one bench workload (diagnosing outliers)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2208_08795_b200 as pcs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5-afps256-8192"
w = bench.WORKLOADS[name]
xyz = bench.make_input(w)
x = torch.from_numpy(xyz).cuda()
pinned = torch.from_numpy(xyz).pin_memory()
ts = []
for i in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pcs.sample_host_batch(pinned, w["C"], method=w["method"], m=w["M"], k=w["K"], sort=w["sort"])
    ts.append((time.perf_counter() - t0) * 1e3)
print(name, "e2e ms per call", np.round(ts, 3).tolist(), flush=True)
ev = []
for i in range(12):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    pcs.sort_axis(x, w["sort"] or "x")
    b.record()
    torch.cuda.synchronize()
    ev.append(a.elapsed_time(b))
print(name, "sort_axis ms per call", np.round(ev, 4).tolist(), flush=True)
ev = []
for i in range(12):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    pcs.sort_perm(x, w["sort"] or "x")
    b.record()
    torch.cuda.synchronize()
    ev.append(a.elapsed_time(b))
print(name, "sort_perm ms per call", np.round(ev, 4).tolist(), flush=True)
