"""Bit-exact parity at the exact launch shapes bench.py times (GPU only).

Every workload of bench.WORKLOADS (BASELINE cfg1-cfg5, same generator, same
seed, same batch size, so the same kernel family, CTA shape and wave count
run as in the timed region) is sampled on the device in one batched call and
compared, cloud by cloud, against the unmodified reference (oracle/_ref,
proj/src/sampler.cpp:85-204 compiled from its sources; the C restatement
oracle/liboracle.so when _ref is absent) -- indices and all four OpStats
counters, as the reference's own oracle-equivalence criterion does
(proj/tests/acceptance_main.cpp:75-124). Sorted workloads also check the
permutation against a host stable argsort (proj/src/order.cpp:11-24).

The reference is run on all host cores, one cloud per worker thread. Where
the whole batch would take it more than a few seconds (vanilla FPS at
>= 8K points, AFPS M=4 at >= 16K) a spread of clouds is checked -- first,
last and evenly spaced, so every wave of a multi-wave launch is covered.
"""
import os

import numpy as np
import pytest

import bench

pytestmark = pytest.mark.gpu

CORES = os.cpu_count() or 1


def _ref_batch(method, xyz, c, m, k):
    """(idx int64 (b, c), stats uint64 (b, 4)) from the reference."""
    from oracle import Oracle, Reference

    if Reference.available():
        idx, st, _ = Reference().sample_batch_f32(method, xyz, c, m, k or 0, workers=CORES)
        return idx, st
    return Oracle().sample_batch_f32(method, xyz, c, m, k or 0)


def _ref_evals_per_cloud(w):
    """Reference work per cloud (distance evaluations + argmax scans)."""
    n, c, m = w["N"], w["C"], w["M"]
    if w["method"] in ("fps", "npdu_fps"):
        m = 1
    return 2 * (c - m) * (n // m)


def _checked_clouds(w, budget_s=3.0, rate=4e8):
    """Which clouds of the batch the reference re-computes: all of them when
    that is cheap (~budget_s of wall time at `rate` evaluations per second
    per core), else an even spread incl. the first and the last."""
    B = w["B"]
    per = _ref_evals_per_cloud(w)
    want = int(max(min(B, 2 * CORES), budget_s * CORES * rate / max(per, 1)))
    if want >= B:
        return np.arange(B)
    return np.unique(np.linspace(0, B - 1, max(want, 2)).round().astype(np.int64))


SHAPES = [k for k in bench.WORKLOADS if not k.startswith("lat-")]


@pytest.mark.parametrize("workload", SHAPES)
def test_bench_workload_bit_exact(workload):
    import torch

    from paper_2208_08795_b200 import sample, synth

    w = bench.WORKLOADS[workload]
    xyz = bench.make_input(w)
    dev = torch.from_numpy(xyz).cuda()
    res = sample(dev, w["C"], method=w["method"], m=w["M"], k=w["K"], sort=w["sort"])
    torch.cuda.synchronize()
    idx, st = res[0].cpu().numpy(), res[1].cpu().numpy()
    if w["sort"] is not None:
        srt, order = synth.stable_sort_np(xyz, "xyz".index(w["sort"]))
        np.testing.assert_array_equal(res[-1].cpu().numpy(), order, err_msg="perm")
        xyz = srt
    sel = _checked_clouds(w)
    want_idx, want_st = _ref_batch(w["method"], xyz[sel], w["C"], w["M"], w["K"])
    bad = [int(b) for i, b in enumerate(sel) if not np.array_equal(idx[b], want_idx[i])]
    assert not bad, f"{workload}: index mismatch in clouds {bad[:8]} of {len(sel)} checked"
    np.testing.assert_array_equal(st[sel], want_st.astype(np.int64), err_msg="stats")
