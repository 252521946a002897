"""A/B: on-chip radix sort vs the bitonic networks (PCS_SORT_RADIX=0), parity
against numpy's stable argsort and CUDA-event timings per call."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_08795_b200 as pcs  # noqa: E402
from paper_2208_08795_b200 import synth  # noqa: E402


def okey(v):
    return np.where(v == 0, np.float32(0), v)


def check(x, axis=0):
    xd = torch.from_numpy(x).cuda()
    srt, perm = pcs.sort_axis(xd, "xyz"[axis])
    want = np.stack([np.argsort(okey(c[:, axis]), kind="stable") for c in x])
    got = perm.cpu().numpy()
    assert np.array_equal(got, want), (x.shape, np.argwhere(got != want)[:5])
    assert np.array_equal(srt.cpu().numpy(), np.take_along_axis(x, want[..., None], 1))


def timeit(x, reps=10):
    """median per-call time of R back-to-back (flush, sort) pairs minus the
    flushes alone: kernel time without host launch gaps"""
    xd = torch.from_numpy(x).cuda()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(3):
        pcs.sort_axis(xd, "x")

    def run(sort):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        torch.cuda._sleep(2_000_000)  # queue the work ahead of the GPU
        a.record()
        for i in range(reps):
            flush.fill_(float(i))
            if sort:
                pcs.sort_axis(xd, "x")
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)
    ts = [(run(True) - run(False)) / reps for _ in range(5)]
    return float(np.median(ts))


rng = np.random.default_rng(0)
SIZES = (1, 2, 31, 100, 1000, 1024, 1025, 2048, 3000, 4096, 5000, 8192, 8193, 12000, 16384,
         20000, 32768, 50000, 65536, 100000, 131072)
for n in () if os.environ.get("SORT_AB_SKIP_PARITY") else SIZES:
    for b in (1, 3, 150):  # 150 clouds: the one-wave radix_cta path
        if b * n > 150 * 40000:
            continue
        x = rng.standard_normal((b, n, 3)).astype(np.float32)
        x[:, ::7, 0] = np.round(x[:, ::7, 0], 1)       # ties
        x[:, ::11, 0] = 0.0
        x[:, ::13, 0] = -0.0                            # -0 == +0, storage order
        x[:, ::17, 0] = -x[:, ::17, 0]
        if n > 5:
            x[:, 3, 0] = np.inf
            x[:, 4, 0] = -np.inf
        check(x)
        check(x, 2)
    xs = np.ones((1, n, 3), np.float32)                 # one key: identity passes
    check(xs)
print("parity ok", flush=True)
CASES = [(16, 2048), (64, 8192), (256, 2048), (256, 4096), (256, 8192), (256, 16384),
         (256, 32768), (1, 2048), (4, 32768), (8, 131072)]
if os.environ.get("SORT_AB_GRID"):
    CASES = [(b, n) for n in (8192, 16384, 32768) for b in (64, 100, 148, 200, 296)]
if os.environ.get("SORT_AB_SKIP_PARITY"):
    pass
for B, N in CASES:
    x = synth.uniform_cube(B, N, 1)
    res = {}
    for arm, env in (("bitonic", {"PCS_SORT_RADIX": "0"}), ("dispatch", {})):
        os.environ.pop("PCS_SORT_RADIX", None)
        os.environ.update(env)
        res[arm] = timeit(x)
    os.environ.pop("PCS_SORT_RADIX", None)
    gb = B * N * 28 / 1e9
    print(f"{B}x{N}: " + "  ".join(f"{k} {v:.4f}" for k, v in res.items()) +
          f" ms ({gb / min(res.values()) * 1e3:.0f} GB/s alg)", flush=True)
