"""cfg4 e2e pieces on the host clock: plain H2D of the batch, the C-ABI
host-batch call with preallocated pinned outputs (by chunk count), and the
Python wrapper sample_host_batch (median of 25 after 0.6 s of warm-up)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2208_08795_b200 as pcs  # noqa: E402
from paper_2208_08795_b200 import _core  # noqa: E402

w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
x = torch.from_numpy(bench.make_input(w)).pin_memory()
B, N, C = w["B"], w["N"], w["C"]
idx = torch.empty((B, C), dtype=torch.int32, pin_memory=True)
st = torch.empty((B, 4), dtype=torch.int64, pin_memory=True)
perm = torch.empty((B, N), dtype=torch.int32, pin_memory=True) if w["sort"] else None
dev = torch.empty(x.shape, dtype=x.dtype, device="cuda")
axis = {"x": 0, "y": 1, "z": 2}.get(w["sort"], -1)


def med(fn, n=25):
    t_end = time.perf_counter() + 0.6
    while time.perf_counter() < t_end:
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    return float(np.median(ts)), float(min(ts))


def h2d():
    dev.copy_(x, non_blocking=True)
    torch.cuda.synchronize()


def capi(ch):
    def f():
        _core.sample_host_ptr(4 if w["method"] == "npdu_afps" else {"fps": 1, "afps": 2,
                              "npdu_fps": 3}[w["method"]], 0, x.data_ptr(), B, N, C, w["M"],
                              w["K"] or 0, 1, 0, 0, 0, idx.data_ptr(), 0, st.data_ptr(), axis,
                              perm.data_ptr() if perm is not None else 0, ch)
    return f


print("h2d_floor", med(h2d))
for ch in ([int(a) for a in sys.argv[2:]] or (0, 4, 8, 12, 16, 24, 32)):
    print("capi chunks", ch, med(capi(ch)))
print("wrapper", med(lambda: pcs.sample_host_batch(x, C, method=w["method"], m=w["M"], k=w["K"],
                                                   sort=w["sort"])))
