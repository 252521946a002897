"""Fixed cost of one sampler launch vs its per-iteration cost: one shape
(B clouds of N points, M sectors) at several C, CUDA events, L2 flushed or
warm. usage: overhead_probe.py METHOD B N M [K]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2208_08795_b200 as pcs  # noqa: E402
from paper_2208_08795_b200 import synth  # noqa: E402

meth, B, N, M = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
K = int(sys.argv[5]) if len(sys.argv) > 5 else None
x = torch.from_numpy(synth.primitives(B, N, 4, seed=1)).cuda()
perm = pcs.sort_perm(x, "x")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def t(fn, fl):
    ts = []
    for i in range(25):
        if fl:
            flush.fill_(i)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts[5:]))


for C in (M, 2 * M, 8 * M, N // 4):
    f = lambda: pcs.sample(x, C, method=meth, m=M, k=K, _perm=perm)
    s = lambda: pcs.sort_perm(x, "x")
    print(f"C={C:5d} iters/sector={C // M - 1:4d} sample warm {t(f, False):.4f} flushed {t(f, True):.4f} | "
          f"sort warm {t(s, False):.4f} flushed {t(s, True):.4f} | {pcs.kernel_family(meth, N, M, K, batch=B, full=True)}")
