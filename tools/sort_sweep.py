"""Time pcs.sort_axis over the BASELINE batch shapes (CUDA events, L2
flushed before each call; median of 15) -> one JSON line per shape."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2208_08795_b200 as pcs  # noqa: E402
from paper_2208_08795_b200 import synth  # noqa: E402

SHAPES = [(1, 2048), (16, 2048), (64, 8192), (256, 2048), (256, 4096), (256, 8192),
          (256, 16384), (256, 32768), (1, 1 << 20)]
if len(sys.argv) > 1:
    SHAPES = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for B, N in SHAPES:
    x = torch.from_numpy(synth.uniform_cube(B, N, 1)).cuda()
    out, perm = pcs.sort_axis(x, "x")
    want = synth.stable_sort_np(x.cpu().numpy(), 0)[1]
    ok = bool(np.array_equal(perm.cpu().numpy(), want))
    for _ in range(3):
        pcs.sort_axis(x, "x")
    p2 = pcs.sort_perm(x, "x")
    ok = ok and bool(torch.equal(p2, perm))
    res = {"B": B, "N": N, "perm_ok": ok}
    for name, fn in (("copy", lambda: pcs.sort_axis(x, "x")), ("perm", lambda: pcs.sort_perm(x, "x"))):
        fn()
        ts = []
        for i in range(15):
            flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[name + "_ms"] = round(float(np.median(ts)), 4)
    # algorithmic bytes: the perm-only sort reads 12N and writes 4N
    res["perm_hbm_gbps"] = round(B * N * 16 / res["perm_ms"] / 1e6, 1)
    print(json.dumps(res), flush=True)
