"""Cluster-spread full-window kernel vs the single-CTA engines (PCS_CLUSTER
0/1 in one process via reload_knobs): sampler time (CUDA events, median of
10) and equality of the results, for few-sector full-window calls."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2208_08795_b200 as pcs  # noqa: E402
from paper_2208_08795_b200 import synth  # noqa: E402

CASES = [("fps", 1, 2048, 512, 1), ("fps", 4, 2048, 512, 1), ("fps", 1, 4096, 1024, 1),
         ("fps", 1, 8192, 2048, 1), ("fps", 2, 8192, 2048, 1), ("afps", 1, 8192, 2048, 4),
         ("afps", 1, 32768, 8192, 32), ("afps", 4, 4096, 1024, 4), ("fps", 16, 2048, 512, 1)]


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for meth, B, N, C, M in CASES:
    x = torch.from_numpy(synth.stable_sort_np(synth.uniform_cube(B, N, 3), 0)[0]).cuda()
    res = {}
    for knob in ("0", "2", "4", "8"):
        os.environ["PCS_CLUSTER"] = "0" if knob == "0" else "1"
        os.environ["PCS_CLUSTER_CS"] = knob
        pcs.reload_knobs()
        fam = pcs.kernel_family(meth, N, M, batch=B, full=True)
        out = pcs.sample(x, C, method=meth, m=M, first="random", seed=5, return_sector=True)
        ms = timed(lambda: pcs.sample(x, C, method=meth, m=M))
        res[knob] = (fam, ms, [o.cpu() for o in out])
    same = all(torch.equal(a, b) for k in ("2", "4", "8") for a, b in zip(res["0"][2], res[k][2]))
    print(json.dumps({"case": f"{meth} B={B} N={N} C={C} M={M}", "same": same,
                      **{("cs" + k if k != "0" else "off"): res[k][:2] for k in res}}), flush=True)
