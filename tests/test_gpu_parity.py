"""Parity of the CUDA path with the oracle / the real reference (GPU only).

Bit-exact is the bar everywhere: sampled indices, sector_of and all four
OpStats counters (integer work), and the DistanceTrace snapshots (fp64, same
operation order, no FMA -> identical bits). Everything goes through the
C-ABI: the drop-in Python surface (pcs.fps, ...) calls pcs_sample_host, the
batched torch op calls pcs_gpu_sample / pcs_gpu_sort_axis.
"""
import os

import numpy as np
import pytest

from conftest import METHOD_NAMES, load_sampler_goldens, load_sort_goldens, setknob
from paper_2208_08795_b200 import synth

pytestmark = pytest.mark.gpu

LINE = np.array([[float(x), 0.0, 0.0] for x in range(8)])


@pytest.fixture(params=["wide", "one_warp"])
def npdu_engine(request, monkeypatch):
    """NPDU sectors <= 4096 points run on the W-warp latency form
    (npdu_wide_kernel) for small batches and on the one-warp TMEM / shared-
    memory kernels otherwise: force each (PCS_NPDU_WIDE = max sectors)."""
    setknob(monkeypatch, "PCS_NPDU_WIDE", "100000000" if request.param == "wide" else "0")
    return request.param


def _call(pcs, meth, pts, c, m, k, first, seed):
    if meth == "fps":
        return pcs.fps(pts, c, seed=seed, first=first)
    if meth == "afps":
        return pcs.afps(pts, c, m, seed=seed, first=first)
    if meth == "npdu_fps":
        return pcs.npdu_fps(pts, c, k, seed=seed, first=first)
    return pcs.npdu_afps(pts, c, m, k, seed=seed, first=first)


def _same(got, idx, sec, st):
    np.testing.assert_array_equal(got[0], idx)
    np.testing.assert_array_equal(got[1], sec)
    assert [got[2][f] for f in ("dist_evals", "dist_writes", "argmax_scans", "iterations")] == \
        [int(x) for x in st]


@pytest.mark.parametrize("name", sorted(load_sampler_goldens()))
def test_goldens_through_dropin(pcs, name):
    g = load_sampler_goldens()[name]
    got = _call(pcs, METHOD_NAMES[int(g["method"])], g["points"], int(g["c"]), int(g["m"]),
                int(g["k"]), "random" if int(g["random_first"]) else "fixed", int(g["seed"]))
    _same(got, g["indices"], g["sector_of"], g["stats"])


def test_reference_kats(pcs):
    # proj/tests/test_sampler.cpp:88-113, 184-220, 267-344
    assert pcs.fps(LINE[:4], 2, first="fixed")[0].tolist() == [0, 3]
    assert pcs.fps(LINE[:4], 3, first="fixed")[0].tolist() == [0, 3, 1]
    assert pcs.fps(LINE[:4], 4, first="fixed")[0].tolist() == [0, 3, 1, 2]
    idx, _, st = pcs.npdu_fps(LINE, 3, 2, first="fixed")
    assert idx.tolist() == [0, 1, 2]
    assert (st["dist_evals"], st["dist_writes"], st["iterations"]) == (3, 2, 2)
    assert pcs.npdu_fps(LINE, 3, 4, first="fixed")[0].tolist() == [0, 2, 4]
    one = pcs.fps(synth.random_cloud(100, 17), 1, first="fixed")
    assert one[0].tolist() == [0] and set(one[2].values()) == {0}
    r = pcs.fps(synth.random_cloud(100, 17), 25, seed=5)
    assert r[2]["dist_evals"] == 2400 and r[2]["argmax_scans"] == 2400 and r[2]["iterations"] == 24
    cloud = synth.random_cloud(2048, 2)
    r = pcs.afps(cloud, 512, 32, seed=1)
    assert r[2]["dist_evals"] == 30720 and len(set(r[0].tolist())) == 512
    assert pcs.afps(synth.random_cloud(10, 3), 4, 3, first="fixed")[2]["dist_evals"] == 4
    r = pcs.afps(synth.random_cloud(100, 5), 20, 20, seed=77)
    assert r[2]["dist_evals"] == 0 and r[1].tolist() == list(range(20))
    assert pcs.npdu_fps(synth.random_cloud(64, 4), 10, 1, seed=8)[2]["dist_evals"] == 9
    r = pcs.npdu_afps(synth.random_cloud(2048, 6), 512, 32, 16, seed=2)
    assert r[2]["dist_evals"] <= 7680 and len(set(r[0].tolist())) == 512
    a = pcs.npdu_afps(synth.random_cloud(2048, 6), 512, 32, 16, seed=2, threads=4)
    assert a[0].tolist() == r[0].tolist() and a[2] == r[2]


def test_reduction_identities(pcs, npdu_engine):
    # proj/tests/acceptance_main.cpp:128-171
    rng = np.random.default_rng(260856)
    for trial in range(25):
        n = int(rng.integers(16, 416))
        c = int(rng.integers(2, n + 1))
        m = int(rng.integers(1, c + 1))
        k = int(rng.integers(1, 25))
        seed = int(rng.integers(0, 2**63))
        first = "random" if trial % 2 else "fixed"
        pts = synth.random_cloud(n, int(rng.integers(0, 2**63)))
        f = pcs.fps(pts, c, seed=seed, first=first)
        a1 = pcs.afps(pts, c, 1, seed=seed, first=first)
        assert f[0].tolist() == a1[0].tolist() and f[2] == a1[2]
        nf = pcs.npdu_fps(pts, c, k, seed=seed, first=first)
        na1 = pcs.npdu_afps(pts, c, 1, k, seed=seed, first=first)
        assert nf[0].tolist() == na1[0].tolist() and nf[2] == na1[2]
        big = pcs.npdu_fps(pts, c, 2 * n, seed=seed, first=first)
        assert big[0].tolist() == f[0].tolist() and big[2] == f[2]
        maxsec = -(-n // m)
        wa = pcs.npdu_afps(pts, c, m, 2 * maxsec, seed=seed, first=first)
        a = pcs.afps(pts, c, m, seed=seed, first=first)
        assert wa[0].tolist() == a[0].tolist() and wa[2] == a[2]


def test_random_configs_vs_oracle(pcs, oracle, npdu_engine):
    rng = np.random.default_rng(7777)
    for t in range(160):
        n = int(rng.integers(4, 3000 if t % 8 else 8193))
        c = int(rng.integers(1, n + 1))
        m = int(rng.integers(1, c + 1)) if t % 3 else 1
        k = int(rng.integers(1, 200))
        meth = ("fps", "afps", "npdu_fps", "npdu_afps")[t % 4]
        first = "random" if t % 2 else "fixed"
        pts = synth.random_cloud(n, 40000 + t)
        if t % 5 == 0:
            pts[: n // 2] = 1.0
        if t % 7 == 0:
            pts = np.round(pts)  # heavy ties
        want = oracle.sample(meth, pts, c, m, k, first, t)
        got = _call(pcs, meth, pts, c, m, k, first, t)
        _same(got, *want)


def test_distance_trace_bit_exact(pcs, oracle, npdu_engine):
    pts = synth.random_cloud(300, 404)
    for k in (None, 7):
        idx, _, st, tr = pcs.local_fps(pts, 40, 290, 60, k=k, seed=3, first="random", trace=True)
        widx, wst, wtr = oracle.local_fps(pts, 40, 290, 60, k=k or 0, first="random", seed=3,
                                          trace=True)
        np.testing.assert_array_equal(idx, widx)
        np.testing.assert_array_equal(tr, wtr)
        assert (tr[1:] <= tr[:-1]).all()  # monotone (inf - inf would be nan)


@pytest.mark.parametrize("morton", ["1", "0"])
def test_distance_trace_rows_engines(pcs, oracle, monkeypatch, morton):
    """Trace through the pruned-row engines (the Morton engine writes d[] back
    through its slot -> index map; the trace entry is the fp64 drop-in)."""
    setknob(monkeypatch, "PCS_SAMPLER", "rows")
    setknob(monkeypatch, "PCS_MORTON", morton)
    pts = synth.random_cloud(700, 405)
    pts[100:200] = pts[3]
    idx, _, st, tr = pcs.local_fps(pts, 20, 690, 40, k=None, seed=5, first="random", trace=True)
    widx, wst, wtr = oracle.local_fps(pts, 20, 690, 40, k=0, first="random", seed=5, trace=True)
    np.testing.assert_array_equal(idx, widx)
    np.testing.assert_array_equal(tr, wtr)


def test_batched_configs_vs_oracle(oracle, npdu_engine):
    import torch

    from paper_2208_08795_b200 import sample

    cases = [
        ("cfg1", synth.uniform_cube(1, 2048, 0), "fps", 512, 1, None, "x"),
        ("cfg2", synth.primitives(16, 2048, 4, seed=1), "afps", 512, 8, None, "x"),
        ("cfg3n", synth.primitives(4, 8192, 6, seed=3), "npdu_afps", 2048, 16, 65, "x"),
        ("cfg3a", synth.primitives(2, 8192, 6, seed=3), "afps", 2048, 16, None, "x"),
        ("cfg3f", synth.primitives(1, 8192, 6, seed=3), "fps", 2048, 1, None, "x"),
        ("cfg4", synth.lidar_sweep(2, seed=4), "npdu_afps", 8192, 32, 129, None),
        ("cfg5a", synth.uniform_cube(3, 4096, 9), "afps", 1024, 4, None, "x"),
        ("cfg5n", synth.uniform_cube(3, 4096, 9), "npdu_afps", 1024, 16, 65, "x"),
    ]
    for name, xyz, meth, c, m, k, axis in cases:
        dev = torch.from_numpy(xyz).cuda()
        res = sample(dev, c, method=meth, m=m, k=k, sort=axis)
        torch.cuda.synchronize()
        if axis is not None:
            host_sorted, order = synth.stable_sort_np(xyz, 0)
            np.testing.assert_array_equal(res[-1].cpu().numpy(), order)
            xyz = host_sorted
        want_idx, want_st = oracle.sample_batch_f32(meth, xyz, c, m, k or 0)
        np.testing.assert_array_equal(res[0].cpu().numpy(), want_idx, err_msg=name)
        np.testing.assert_array_equal(res[1].cpu().numpy(), want_st.astype(np.int64), err_msg=name)


def test_random_first_and_per_cloud_seeds(oracle, npdu_engine):
    import torch

    from paper_2208_08795_b200 import sample

    xyz = synth.uniform_cube(6, 1000, 21)
    seeds = torch.tensor([3, 99, 2**62 + 5, 0, 7, 123456789], dtype=torch.int64)
    res = sample(torch.from_numpy(xyz).cuda(), 100, method="npdu_afps", m=5, k=17,
                 first="random", seeds=seeds, index_dtype=torch.int64, return_sector=True)
    for b in range(6):
        idx, sec, st = oracle.sample("npdu_afps", xyz[b].astype(np.float64), 100, 5, 17,
                                     "random", int(seeds[b]))
        np.testing.assert_array_equal(res[0][b].cpu().numpy(), idx)
        np.testing.assert_array_equal(res[2][b].cpu().numpy(), sec)
        np.testing.assert_array_equal(res[1][b].cpu().numpy(), st.astype(np.int64))


def test_sort_parity(pcs):
    import torch

    from paper_2208_08795_b200 import sort_axis

    for name, g in load_sort_goldens().items():
        np.testing.assert_array_equal(pcs.exact_sort(g["points"], "xyz"[int(name[-1])]), g["sorted"])
    rng = np.random.default_rng(3)
    for n in (1, 2, 17, 1000, 3000, 5000, 12000, 16384, 16385, 40000, 70000, 200000, 300000):
        xyz = np.round(rng.normal(size=(3, n, 3)), 2).astype(np.float32)
        xyz[:, :: 7, 1] = -0.0
        xyz[:, 1:: 7, 1] = 0.0
        for axis in range(3):
            out, perm = sort_axis(torch.from_numpy(xyz).cuda(), axis)
            want, order = synth.stable_sort_np(xyz, axis)
            np.testing.assert_array_equal(perm.cpu().numpy(), order)
            np.testing.assert_array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("radix", ["1", "0"])
def test_sort_kernel_families(pcs, monkeypatch, radix):
    """Every on-chip sort variant (radix_reg_kernel: one CTA, clusters of
    2K- and 4K-point CTAs; radix_cta_kernel: one 16K-point CTA per cloud or
    a merging pair, for a wave of clouds; PCS_SORT_RADIX=0 forces the bitonic
    networks)
    against numpy's stable argsort: ties, signed zeros, infinities, a
    constant axis (identity passes), ragged sizes."""
    import torch

    from paper_2208_08795_b200 import sort_axis

    setknob(monkeypatch, "PCS_SORT_RADIX", radix)
    rng = np.random.default_rng(29)
    cases = [(b, n) for n in (3, 1024, 1500, 2048, 4096, 4097, 8192, 12000, 16384, 30000, 32768,
                              40000, 65536) for b in (1, 16, 37, 38) if b * n <= 40 * 65536]
    # a wave of clouds (>= 148): one CTA per cloud, or a pair merging halves
    cases += [(150, n) for n in (5000, 8192, 12000, 16384, 20000, 32768)]
    for b, n in cases:
        xyz = np.round(rng.normal(size=(b, n, 3)), 1).astype(np.float32)
        xyz[:, ::9, 0] = -0.0
        xyz[:, 4::9, 0] = 0.0
        xyz[:, 2::97, 0] = np.inf
        xyz[:, 3::89, 0] = -np.inf
        xyz[:, :, 1] = 0.5
        for axis in (0, 1):
            out, perm = sort_axis(torch.from_numpy(xyz).cuda(), axis)
            want, order = synth.stable_sort_np(xyz, axis)
            np.testing.assert_array_equal(perm.cpu().numpy(), order, err_msg=f"{b}x{n} ax{axis}")
            np.testing.assert_array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("n", [700, 1500, 4096, 5000, 8192, 12000, 16384, 20000, 32768])
def test_bucket_sort_and_flagged_fallback(pcs, n):
    """The value-bucket sort (permutation requested: <= 148 clouds of <= 4K
    in 1024-thread CTAs, 38+ clouds of 4K-32K) in one batch with every kind
    of cloud: uniform keys, keys with exact duplicates inside buckets (ties
    ordered by storage index), signed zeros, a constant axis (identity), a
    huge bucket and infinities (flagged and re-sorted by the radix CTA
    kernel in a second launch, or ranked all-pairs inside the CTA for <= 4K
    points) -- against numpy's stable argsort, perm and gathered copy, both
    launch forms of the flagged fallback (one CTA / a pair per cloud)."""
    import torch

    from paper_2208_08795_b200 import sort_axis, sort_perm

    rng = np.random.default_rng(n)
    for b in (40, 150):
        xyz = rng.random((b, n, 3), dtype=np.float32)
        xyz[1::6, :, 0] = np.round(xyz[1::6, :, 0] * n / 3) / (n / 3)   # duplicates, small buckets
        xyz[2::6, ::5, 0] = -0.0
        xyz[2::6, 1::5, 0] = 0.0
        xyz[3::6, :, 0] = 0.25                                           # constant
        xyz[4::6, : n // 2, 0] = 0.5                                     # one huge bucket
        xyz[5::6, 7, 0] = np.inf
        xyz[5::6, 8, 0] = -np.inf
        x = torch.from_numpy(xyz).cuda()
        want, order = synth.stable_sort_np(xyz, 0)
        out, perm = sort_axis(x, 0)
        np.testing.assert_array_equal(perm.cpu().numpy(), order, err_msg=f"{b}x{n}")
        np.testing.assert_array_equal(out.cpu().numpy(), want)
        np.testing.assert_array_equal(sort_perm(x, "x").cpu().numpy(), order)


def test_exact_sort_dropin_fp32_keys(pcs):
    """pcs.exact_sort on float64 clouds whose axis column is fp32-exact sorts
    fp32 keys on the device and gathers the float64 points on the host: the
    other columns keep full double precision, ties keep storage order, -0.0
    equals +0.0; a column with one non-fp32 value takes the fp64 path."""
    rng = np.random.default_rng(31)
    for n in (1, 2, 100, 2048, 5000, 32768, 70000, 300000):
        pts = rng.normal(size=(n, 3))                      # full-precision doubles
        col = np.round(rng.normal(size=n), 2).astype(np.float32).astype(np.float64)
        col[::13] = -0.0
        col[1::13] = 0.0
        if n > 10:
            col[5] = np.inf
            col[6] = -np.inf
        for axis in (0, 2):
            p = pts.copy()
            p[:, axis] = col
            want = synth.stable_sort_np(p[None], axis)[0][0]
            np.testing.assert_array_equal(pcs.exact_sort(p, "xyz"[axis]), want, err_msg=f"{n}")
            if n > 10:
                p[7, axis] = 0.1  # not representable in fp32
                want = synth.stable_sort_np(p[None], axis)[0][0]
                np.testing.assert_array_equal(pcs.exact_sort(p, "xyz"[axis]), want)


def test_device_wide_radix_sort(pcs):
    """Clouds past one CTA / one cluster: the multi-CTA LSD radix (fp32 >
    256K points, fp64 >= 64K), stable with ties and signed zeros, batched."""
    import torch

    from paper_2208_08795_b200 import sort_axis

    rng = np.random.default_rng(11)
    for n, b, dt in ((262145, 2, np.float32), (1 << 20, 1, np.float32), (65536, 3, np.float64),
                     (100003, 2, np.float64)):
        xyz = np.round(rng.normal(size=(b, n, 3)), 3).astype(dt)
        xyz[:, ::5, 0] = -0.0
        xyz[:, 1::5, 0] = 0.0
        for axis in (0, 2):
            out, perm = sort_axis(torch.from_numpy(xyz).cuda(), axis)
            want, order = synth.stable_sort_np(xyz, axis)
            np.testing.assert_array_equal(perm.cpu().numpy(), order, err_msg=f"{n} {dt}")
            np.testing.assert_array_equal(out.cpu().numpy(), want)
    pts = synth.random_cloud(70000, 5)
    pts[::3, 1] = pts[0, 1]
    np.testing.assert_array_equal(pcs.exact_sort(pts, "y"), synth.stable_sort_np(pts[None], 1)[0][0])


def test_full_size_properties_cfg4():
    """BASELINE cfg4 at full size (128 x 32768, NPDU-AFPS M=32, k=129,
    C=8192): size-independent properties on every cloud (distinct indices,
    sector confinement, quotas, dist_evals = the windows along the path).
    The bit-exact comparison of the same batch with the reference is
    tests/test_gpu_bench_shapes.py::test_bench_workload_bit_exact[cfg4]."""
    import torch

    from paper_2208_08795_b200 import sample

    xyz = synth.lidar_sweep(128, seed=4)
    idx, st, sec = sample(torch.from_numpy(xyz).cuda(), 8192, method="npdu_afps", m=32, k=129,
                          return_sector=True)
    idx, st, sec = idx.cpu().numpy(), st.cpu().numpy(), sec.cpu().numpy()
    n, m, q = 32768, 32, 256
    for b in range(128):
        assert len(np.unique(idx[b])) == 8192
        s = idx[b] // (n // m)
        np.testing.assert_array_equal(s, sec[b])
        np.testing.assert_array_equal(np.bincount(s, minlength=m), np.full(m, q))
        # dist_evals == sum of the windows along the returned path
        loc = (idx[b] % (n // m)).reshape(m, q)[:, :-1]
        lo = np.maximum(loc - 64, 0)
        hi = np.minimum(loc + 65, n // m)
        assert st[b, 0] == (hi - lo).sum()
        assert st[b, 2] == m * (q - 1) * (n // m) and st[b, 3] == m * (q - 1)
        assert st[b, 1] <= st[b, 0]


def test_determinism_across_calls():
    import torch

    from paper_2208_08795_b200 import sample

    xyz = torch.from_numpy(synth.primitives(8, 8192, 6, seed=5)).cuda()
    a = sample(xyz, 2048, method="afps", m=16, sort="x")
    b = sample(xyz, 2048, method="afps", m=16, sort="x")
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_large_sectors_cluster_engine(pcs, oracle):
    """Sectors beyond one SM's shared memory run on the pruned-row engine over
    a thread-block cluster (FPS at 16K/32K, NPDU on whole clouds)."""
    import torch

    from paper_2208_08795_b200 import sample

    cases = [(16384, 2048, "fps", 1, None), (32768, 1024, "fps", 1, None),
             (20000, 3000, "npdu_fps", 1, 65), (40000, 4000, "afps", 4, None),
             (12000, 1500, "npdu_afps", 1, 129)]
    for n, c, meth, m, k in cases:
        xyz = synth.uniform_cube(1, n, n)
        xyz = synth.stable_sort_np(xyz, 0)[0]
        idx, st = sample(torch.from_numpy(xyz).cuda(), c, method=meth, m=m, k=k)
        want_idx, want_st = oracle.sample_batch_f32(meth, xyz, c, m, k or 0)
        np.testing.assert_array_equal(idx.cpu().numpy(), want_idx, err_msg=f"{meth} {n}")
        np.testing.assert_array_equal(st.cpu().numpy(), want_st.astype(np.int64))
    # fp64 input through the drop-in, 10K points (double staging, cluster of 2)
    pts = synth.random_cloud(10000, 77)
    got = pcs.fps(pts, 700, seed=3)
    want = oracle.sample("fps", pts, 700, first="random", seed=3)
    _same(got, *want)


@pytest.mark.parametrize("morton", ["1", "0"])
@pytest.mark.parametrize("meth,n,c,m,k", [("fps", 2048, 512, 1, 0), ("afps", 4096, 1024, 4, 0),
                                          ("npdu_afps", 8192, 2048, 16, 65),
                                          ("npdu_fps", 3000, 700, 1, 33), ("afps", 700, 90, 3, 0)])
def test_rows_engine_forced_matches_oracle(oracle, monkeypatch, meth, n, c, m, k, morton):
    """The pruned-row engines (Morton rows and storage-order rows) on sizes the
    other kernels normally take (PCS_SAMPLER=rows), including coincident
    points and random starts."""
    import torch

    from paper_2208_08795_b200 import sample

    setknob(monkeypatch, "PCS_SAMPLER", "rows")
    setknob(monkeypatch, "PCS_MORTON", morton)
    xyz = synth.stable_sort_np(synth.uniform_cube(3, n, 5), 0)[0]
    xyz[1, : n // 3] = xyz[1, 0]  # many coincident points
    for first in ("fixed", "random"):
        idx, st = sample(torch.from_numpy(xyz).cuda(), c, method=meth, m=m, k=k or None,
                         first=first, seed=11)
        want_idx, want_st = oracle.sample_batch_f32(meth, xyz, c, m, k, first, 11)
        np.testing.assert_array_equal(idx.cpu().numpy(), want_idx)
        np.testing.assert_array_equal(st.cpu().numpy(), want_st.astype(np.int64))


@pytest.mark.parametrize("engine", ["auto", "rows", "slab"])
def test_subnormal_and_signed_zero_coordinates(oracle, monkeypatch, engine):
    """fp32 subnormals take the exact F2F widening path; +-0 the integer one."""
    import torch

    from paper_2208_08795_b200 import sample

    if engine != "auto":
        setknob(monkeypatch, "PCS_SAMPLER", "rows")
        setknob(monkeypatch, "PCS_MORTON", "0" if engine == "slab" else "1")
    xyz = synth.uniform_cube(2, 3000, 8) * np.float32(1e-36)
    xyz[0, ::5, 0] = np.float32(3e-41)   # subnormal
    xyz[0, 1::5, 1] = np.float32(-0.0)
    xyz[1, ::3, 2] = np.float32(0.0)
    for meth, m, k in (("npdu_afps", 3, 33), ("afps", 2, 0), ("fps", 1, 0)):
        idx, st = sample(torch.from_numpy(xyz).cuda(), 600, method=meth, m=m, k=k or None)
        want_idx, want_st = oracle.sample_batch_f32(meth, xyz, 600, m, k)
        np.testing.assert_array_equal(idx.cpu().numpy(), want_idx, err_msg=meth)
        np.testing.assert_array_equal(st.cpu().numpy(), want_st.astype(np.int64))


@pytest.mark.parametrize("tmem", ["1", "0"])
@pytest.mark.parametrize("cloud", ["cube", "primitives", "dupes", "f64", "f64exact"])
def test_morton_rows_large_sectors(pcs, oracle, monkeypatch, cloud, tmem):
    """Full-window sectors past 3072 points take the Morton-row engines (CTA
    Morton sort, orig-index row keys; per-point state in TMEM for fp32 input,
    or in shared memory): one CTA up to 8K/16K, clusters beyond; clustered,
    duplicated and fp64 inputs; random starts."""
    import torch

    from paper_2208_08795_b200 import sample

    setknob(monkeypatch, "PCS_MORTON_TMEM", tmem)
    if cloud in ("f64", "f64exact") and tmem == "0":
        pytest.skip("fp64 input always uses the shared-memory engine")

    for n, c, m in ((8192, 2048, 1), (16384, 1500, 1), (32768, 700, 1), (60000, 300, 1),
                    (40000, 4000, 4)):
        if cloud == "primitives":
            xyz = synth.primitives(1, n, 6, seed=n)
        else:
            xyz = synth.uniform_cube(1, n, n + 1)
        if cloud == "dupes":
            xyz[0, 1::3] = xyz[0, 0]
            xyz[0, 2::7] = xyz[0, 5]
        if cloud in ("f64", "f64exact"):
            # f64exact: float64 holding fp32 values -> the drop-in samples
            # from an fp32 copy (same results by construction)
            pts = (synth.random_cloud(n, n) if cloud == "f64" else
                   xyz[0].astype(np.float64))
            got = pcs.afps(pts, c, m, seed=n) if m > 1 else pcs.fps(pts, c, seed=n)
            want = oracle.sample("afps" if m > 1 else "fps", pts, c, m, first="random", seed=n)
            _same(got, *want)
            continue
        idx, st = sample(torch.from_numpy(xyz).cuda(), c, method="afps" if m > 1 else "fps",
                         m=m, first="random", seed=n)
        want_idx, want_st = oracle.sample_batch_f32("afps" if m > 1 else "fps", xyz, c, m, 0,
                                                    "random", n)
        np.testing.assert_array_equal(idx.cpu().numpy(), want_idx, err_msg=f"{cloud} {n}")
        np.testing.assert_array_equal(st.cpu().numpy(), want_st.astype(np.int64))


@pytest.mark.parametrize("index_dtype", ["int32", "int64"])
def test_npdu_tmem_slow_path_and_output_blocks(oracle, npdu_engine, index_dtype):
    """fp32 NPDU sectors <= 4096 points (the TMEM kernel, 1-4 rows per lane): heavily duplicated
    clouds drive the all-zero slow path (lowest unsampled index) many times;
    quotas that are not multiples of 32 exercise the buffered output flush."""
    import torch

    from paper_2208_08795_b200 import sample

    rng = np.random.default_rng(9)
    for n, c, m, k in ((4096, 1232, 4, 129), (3000, 2995, 3, 65), (1024, 77, 1, 33),
                       (2048, 2048, 2, 97), (8192, 2001, 2, 129), (6000, 1500, 3, 65),
                       (4000, 999, 1, 33)):
        xyz = synth.uniform_cube(3, n, n)
        xyz[0] = xyz[0][rng.integers(0, 40, n)]            # 40 distinct points
        xyz[1, : n // 2] = xyz[1, 7]                        # half coincident
        for first in ("fixed", "random"):
            idx, st = sample(torch.from_numpy(xyz).cuda(), c, method="npdu_afps", m=m, k=k,
                             first=first, seed=n, index_dtype=getattr(torch, index_dtype))
            want_idx, want_st = oracle.sample_batch_f32("npdu_afps", xyz, c, m, k, first, n)
            np.testing.assert_array_equal(idx.cpu().numpy(), want_idx, err_msg=f"{n} {first}")
            np.testing.assert_array_equal(st.cpu().numpy(), want_st.astype(np.int64))


@pytest.mark.parametrize("grid", [0, 8, 64, 1 << 20])
def test_npdu_tmem_high_word_ties(oracle, monkeypatch, grid):
    """TMEM NPDU kernel row keys under ties: coordinates on a coarse grid
    (many equal distances), a fine grid (high words of d tie, low words
    differ) and uniform ones, every sector size family."""
    import torch

    from paper_2208_08795_b200 import sample

    setknob(monkeypatch, "PCS_NPDU_WIDE", "0")
    rng = np.random.default_rng(grid + 1)
    for n, c, m, k in ((1024, 256, 1, 129), (4096, 1024, 4, 65), (2048, 700, 1, 33),
                       (3000, 900, 2, 97), (512, 200, 1, 65), (8192, 2048, 8, 129)):
        xyz = synth.uniform_cube(4, n, n + grid)
        if grid:
            xyz = (np.round(xyz * grid) / grid).astype(np.float32)
        if grid == 1 << 20:  # distances within a few ulps of each other
            xyz = (1.0 + rng.integers(0, 4, xyz.shape) * 2.0 ** -22).astype(np.float32)
        idx, st = sample(torch.from_numpy(xyz).cuda(), c, method="npdu_afps", m=m, k=k)
        want_idx, want_st = oracle.sample_batch_f32("npdu_afps", xyz, c, m, k)
        np.testing.assert_array_equal(idx.cpu().numpy(), want_idx, err_msg=f"{n} {grid}")
        np.testing.assert_array_equal(st.cpu().numpy(), want_st.astype(np.int64))


@pytest.mark.parametrize("n,k,clouds", [(256, 65, 150), (2048, 65, 170), (4096, 129, 150)])
@pytest.mark.parametrize("grid", [0, 8, 1 << 20])
@pytest.mark.parametrize("key", [None, "2"])
def test_npdu_tmem_high_word_keys_multiwave(reference, monkeypatch, n, k, clouds, grid, key):
    """Multi-wave TMEM NPDU launches take the high-word row keys with
    per-row lowest-lane indices (npdu_tmem_kernel<R,NCAP,3>; key "2": the
    high-word keys with the ballot argmax), 1, 2 and 4 cached rows per lane
    -- under ties: coarse grids (equal distances), distances a few ulps apart
    (high words tie, low words differ) and uniform coordinates; every cloud
    against the reference."""
    import torch

    import paper_2208_08795_b200 as pcs
    from paper_2208_08795_b200 import sample

    setknob(monkeypatch, "PCS_NPDU_KEY", key)
    m = 32
    N, c = n * m, n * m // 4
    fam = pcs.kernel_family("npdu_afps", N, m, k, batch=clouds, full=True)
    assert fam.startswith("npdu_tmem_kernel<") and fam.endswith(f",{key or 3}>"), fam
    rng = np.random.default_rng(grid + n)
    xyz = synth.uniform_cube(clouds, N, n + grid)
    if grid == 8:
        xyz = (np.round(xyz * grid) / grid).astype(np.float32)
    if grid == 1 << 20:
        xyz = (1.0 + rng.integers(0, 4, xyz.shape) * 2.0 ** -22).astype(np.float32)
    idx, st = sample(torch.from_numpy(xyz).cuda(), c, method="npdu_afps", m=m, k=k)
    want_idx, want_st, _ = reference.sample_batch_f32("npdu_afps", xyz, c, m, k,
                                                      workers=os.cpu_count())
    np.testing.assert_array_equal(idx.cpu().numpy(), want_idx, err_msg=f"{n} {grid}")
    np.testing.assert_array_equal(st.cpu().numpy(), want_st.astype(np.int64))


@pytest.mark.parametrize("n,m,c", [(2048, 256, 512), (4000, 256, 700), (4096, 256, 1024),
                                   (1024, 128, 300), (3000, 300, 900)])
@pytest.mark.parametrize("first", ["fixed", "random"])
def test_tiny_sectors_thread_per_sector(oracle, n, m, c, first):
    """>= 2048 sectors of <= 16 points take fps_tiny_kernel (a thread per
    sector): AFPS and NPDU-AFPS, ragged sector sizes and quotas, coincident
    points (the all-zero lowest-unsampled path), fp32 and fp64 input, int64
    indices and sector_of, index / sector bases -- every cloud against the
    oracle."""
    import torch

    import paper_2208_08795_b200 as pcs
    from paper_2208_08795_b200 import sample

    B = max(8, -(-2048 // m))
    xyz = synth.uniform_cube(B, n, n + m)
    xyz[1, : n // 2] = xyz[1, 0]                       # coincident points
    xyz[2] = np.round(xyz[2] * 4) / 4                  # coarse grid: many ties
    x = torch.from_numpy(xyz).cuda()
    for meth, k in (("afps", None), ("npdu_afps", 3), ("npdu_afps", 9)):
        fam = pcs.kernel_family(meth, n, m, k, batch=B, full=True)
        assert fam.startswith("fps_tiny_kernel"), fam
        want_idx, want_st = oracle.sample_batch_f32(meth, xyz, c, m, k or 0, first, 5)
        for xx in (x, x.double()):
            idx, st, sec = sample(xx, c, method=meth, m=m, k=k, first=first, seed=5,
                                  index_dtype=torch.int64, return_sector=True)
            np.testing.assert_array_equal(idx.cpu().numpy(), want_idx, err_msg=f"{meth} {k} {xx.dtype}")
            np.testing.assert_array_equal(st.cpu().numpy(), want_st.astype(np.int64))
        for b in (0, 1, B - 1):
            w_idx, w_sec, _ = oracle.sample(meth, xyz[b].astype(np.float64), c, m, k or 0, first, 5)
            np.testing.assert_array_equal(sec[b].cpu().numpy(), w_sec)
        idx, st = sample(x, c, method=meth, m=m, k=k, first=first, seed=5, index_base=1000)
        np.testing.assert_array_equal(idx.cpu().numpy(), want_idx + 1000)


def test_streaming_engine_beyond_on_chip_sectors(oracle):
    """Sectors larger than every on-chip engine (d[] in global memory, one
    cooperative launch per sector, grid barrier per iteration): FPS and NPDU
    on a 300K-point cloud against the oracle."""
    import torch

    from paper_2208_08795_b200 import sample

    xyz = synth.uniform_cube(1, 300000, 3)
    dev = torch.from_numpy(xyz).cuda()
    for meth, c, k, first in (("fps", 600, None, "random"), ("npdu_fps", 1500, 129, "fixed")):
        idx, st = sample(dev, c, method=meth, k=k, first=first, seed=5)
        want_idx, want_st = oracle.sample_batch_f32(meth, xyz, c, 1, k or 0, first, 5)
        np.testing.assert_array_equal(idx.cpu().numpy(), want_idx, err_msg=meth)
        np.testing.assert_array_equal(st.cpu().numpy(), want_st.astype(np.int64))


@pytest.mark.parametrize("meth,n,c,m,k", [("fps", 3000, 2990, 1, 0), ("afps", 5000, 900, 3, 0),
                                          ("npdu_afps", 4099, 1200, 2, 65)])
def test_streaming_engine_forced_matches_oracle(oracle, monkeypatch, meth, n, c, m, k):
    """The streaming engine forced onto small sectors (PCS_SAMPLER=stream):
    coincident points drive the all-zero slow path; fp64 drop-in too."""
    import torch

    from paper_2208_08795_b200 import sample

    setknob(monkeypatch, "PCS_SAMPLER", "stream")
    xyz = synth.uniform_cube(2, n, 9)
    xyz[1, : n // 2] = xyz[1, 0]
    for first in ("fixed", "random"):
        idx, st = sample(torch.from_numpy(xyz).cuda(), c, method=meth, m=m, k=k or None,
                         first=first, seed=3)
        want_idx, want_st = oracle.sample_batch_f32(meth, xyz, c, m, k, first, 3)
        np.testing.assert_array_equal(idx.cpu().numpy(), want_idx)
        np.testing.assert_array_equal(st.cpu().numpy(), want_st.astype(np.int64))
    pts = synth.random_cloud(3001, 4)
    got = _core_sample(meth, pts, c, m, k)
    want = oracle.sample(meth, pts, c, m, k)
    _same(got, *want)


def _core_sample(meth, pts, c, m, k):
    import paper_2208_08795_b200 as pcs

    if meth == "fps":
        return pcs.fps(pts, c, first="fixed")
    if meth == "afps":
        return pcs.afps(pts, c, m, first="fixed")
    return pcs.npdu_afps(pts, c, m, k, first="fixed")


@pytest.mark.parametrize("meth,B,n,c,m,k", [
    ("fps", 3, 1, 1, 1, 0), ("afps", 2, 5, 5, 5, 0), ("npdu_afps", 2, 7, 7, 7, 1),
    ("npdu_fps", 2, 40, 40, 1, 1), ("npdu_fps", 2, 40, 17, 1, 1000), ("afps", 5000, 2, 2, 1, 0),
    ("npdu_afps", 300, 96, 33, 3, 3), ("fps", 2, 4096, 1, 1, 0), ("afps", 1, 3073, 3073, 1, 0)])
def test_edge_shapes(oracle, npdu_engine, meth, B, n, c, m, k):
    """Degenerate shapes: one point, quota 1, every point sampled, window 1,
    window wider than the sector, thousands of two-point clouds."""
    import torch

    from paper_2208_08795_b200 import sample

    xyz = synth.uniform_cube(B, n, n + B)
    idx, st = sample(torch.from_numpy(xyz).cuda(), c, method=meth, m=m, k=k or None)
    want_idx, want_st = oracle.sample_batch_f32(meth, xyz, c, m, k)
    np.testing.assert_array_equal(idx.cpu().numpy(), want_idx)
    np.testing.assert_array_equal(st.cpu().numpy(), want_st.astype(np.int64))


def test_busy_afps_takes_morton_engine(oracle):
    """Many (>= 4 per SM) full-window sectors of 1025-3072 points take the
    TMEM Morton engine (small CTAs, many per SM); bit-exact with the oracle."""
    import torch

    import paper_2208_08795_b200 as pcs
    from paper_2208_08795_b200 import sample

    B, n, m, c = 150, 4400, 4, 1000
    if os.environ.get("PCS_MORTON_TMEM", "1") != "0":
        assert pcs.kernel_family("afps", n, m, batch=B) == "morton_tmem_kernel"
    xyz = synth.stable_sort_np(synth.primitives(B, n, 5, seed=12), 0)[0]
    idx, st = sample(torch.from_numpy(xyz).cuda(), c, method="afps", m=m, first="random", seed=2)
    want_idx, want_st = oracle.sample_batch_f32("afps", xyz, c, m, 0, "random", 2)
    np.testing.assert_array_equal(idx.cpu().numpy(), want_idx)
    np.testing.assert_array_equal(st.cpu().numpy(), want_st.astype(np.int64))


@pytest.mark.parametrize("meth,n,c,m,k", [("afps", 1 << 20, 1 << 18, 1024, None),
                                          ("npdu_afps", 65536, 8192, 64, 65),
                                          ("afps", 100003, 9001, 37, None)])
def test_sector_shards_reassemble_on_device(meth, n, c, m, k):
    """The multi-GPU sector split (shard.sector_shard + index_base /
    sector_base) run shard by shard on one device: the concatenated shards
    equal the whole-cloud call bit for bit -- indices, sector ids and the
    per-sector random starts (seed ^ global sector)."""
    import torch

    from paper_2208_08795_b200 import sample, shard

    xyz = torch.from_numpy(synth.uniform_cube(1, n, 17)).cuda()
    xs = sample(xyz, c, method=meth, m=m, k=k, sort="x", first="random", seed=9,
                return_sector=True)
    whole_idx, whole_st, whole_sec = xs[0], xs[1], xs[2]
    srt = pcs_sort(xyz)
    for world in (2, 3, 8):
        parts_i, parts_s, st = [], [], torch.zeros(4, dtype=torch.int64, device="cuda")
        for rank in range(world):
            sh = shard.sector_shard(n, c, m, world, rank)
            i, s_, sec = sample(srt[:, sh.point_lo:sh.point_hi], sh.c, method=meth, m=sh.m, k=k,
                                first="random", seed=9, return_sector=True,
                                index_base=sh.point_lo, sector_base=sh.sector_lo)
            parts_i.append(i)
            parts_s.append(sec)
            st += s_[0]
        assert torch.equal(torch.cat(parts_i, 1), whole_idx), world
        assert torch.equal(torch.cat(parts_s, 1), whole_sec), world
        assert torch.equal(st, whole_st[0]), world


def pcs_sort(xyz):
    from paper_2208_08795_b200 import sort_axis

    return sort_axis(xyz, "x")[0]


@pytest.mark.parametrize("n,c,m,k", [(8192, 2048, 1, 65), (20000, 3000, 1, 129), (40000, 4000, 1, 33),
                                     (32768, 4096, 4, 65), (5000, 2500, 1, 7)])
def test_npdu_big_sectors_tmem_rows(oracle, n, c, m, k):
    """Windowed sectors past 4096 points (fp32): the TMEM row engine in
    storage order with window-restricted rows (1 CTA or a cluster);
    coincident points and random starts."""
    import torch

    import paper_2208_08795_b200 as pcs
    from paper_2208_08795_b200 import sample

    meth = "npdu_afps" if m > 1 else "npdu_fps"
    assert pcs.kernel_family(meth, n, m, k) == "morton_tmem_kernel"
    xyz = synth.stable_sort_np(synth.uniform_cube(2, n, n), 0)[0]
    xyz[1, 100:600] = xyz[1, 99]
    for first in ("fixed", "random"):
        idx, st = sample(torch.from_numpy(xyz).cuda(), c, method=meth, m=m, k=k, first=first,
                         seed=4)
        want_idx, want_st = oracle.sample_batch_f32(meth, xyz, c, m, k, first, 4)
        np.testing.assert_array_equal(idx.cpu().numpy(), want_idx, err_msg=f"{n} {first}")
        np.testing.assert_array_equal(st.cpu().numpy(), want_st.astype(np.int64))


def test_host_pipelined_path_matches_device_path():
    """CPU (pinned or not) input: chunked H2D/compute/D2H gives the same
    results as the device path."""
    import torch

    from paper_2208_08795_b200 import sample, sample_host_batch

    xyz = synth.primitives(10, 4096, 5, seed=2)
    dev = sample(torch.from_numpy(xyz).cuda(), 1024, method="npdu_afps", m=8, k=65, sort="x",
                 return_sector=True)
    host = sample(torch.from_numpy(xyz), 1024, method="npdu_afps", m=8, k=65, sort="x",
                  return_sector=True)
    for a, b in zip(dev, host):
        assert not b.is_cuda
        np.testing.assert_array_equal(a.cpu().numpy(), b.numpy())
    npi = sample_host_batch(xyz, 1024, method="npdu_afps", m=8, k=65, sort="x")
    np.testing.assert_array_equal(npi[0], dev[0].cpu().numpy())
    # the C-ABI host batch entry: pinned and pageable, several chunkings,
    # every output (indices, stats, sector_of, perm)
    pinned = torch.from_numpy(xyz).pin_memory()
    for src, chunks in ((xyz, 0), (pinned, 1), (pinned, 3), (pinned, 10)):
        h = sample_host_batch(src, 1024, method="npdu_afps", m=8, k=65, sort="x",
                              return_sector=True, chunks=chunks)
        for a, b in zip(dev, h):
            np.testing.assert_array_equal(a.cpu().numpy(), b)
    h64 = sample_host_batch(xyz.astype(np.float64), 500, method="afps", m=4, first="random",
                            seed=3, index_dtype=np.int64)
    d64 = sample(torch.from_numpy(xyz.astype(np.float64)).cuda(), 500, method="afps", m=4,
                 first="random", seed=3, index_dtype=torch.int64)
    np.testing.assert_array_equal(h64[0], d64[0].cpu().numpy())
    np.testing.assert_array_equal(h64[1], d64[1].cpu().numpy())


def test_host_batch_chunk_schedules():
    """pcs_sample_host_batch chunk boundaries: the default schedule, uneven
    chunks, more chunks than the stream events hold, and one chunk per cloud
    all give the device path's results."""
    import torch

    from paper_2208_08795_b200 import sample, sample_host_batch

    xyz = synth.lidar_sweep(2, seed=7)[:, :4096].copy()
    xyz = np.concatenate([xyz] * 19 + [xyz[:1]])  # 39 clouds
    dev = sample(torch.from_numpy(xyz).cuda(), 1024, method="npdu_afps", m=4, k=129)
    pinned = torch.from_numpy(xyz).pin_memory()
    for chunks in (0, 5, 39, 100):
        h = sample_host_batch(pinned, 1024, method="npdu_afps", m=4, k=129, chunks=chunks)
        np.testing.assert_array_equal(h[0], dev[0].cpu().numpy(), err_msg=str(chunks))
        np.testing.assert_array_equal(h[1], dev[1].cpu().numpy(), err_msg=str(chunks))


def test_one_million_point_afps_vs_oracle(oracle):
    """BASELINE cfg5's single N=2^20 cloud, AFPS M=1024 (1024-point sectors,
    quota 256) after the GPU axis sort (global-memory bitonic network)."""
    import torch

    from paper_2208_08795_b200 import sample

    n = 1 << 20
    xyz = synth.uniform_cube(1, n, 2024)
    idx, st, perm = sample(torch.from_numpy(xyz).cuda(), n // 4, method="afps", m=1024, sort="x")
    srt, order = synth.stable_sort_np(xyz, 0)
    np.testing.assert_array_equal(perm.cpu().numpy(), order)
    want_idx, want_st = oracle.sample_batch_f32("afps", srt, n // 4, 1024, 0)
    np.testing.assert_array_equal(idx.cpu().numpy(), want_idx)
    np.testing.assert_array_equal(st.cpu().numpy(), want_st.astype(np.int64))


# ---------------------------------------------------------------- §8(f) rows
def test_quality_metrics_bit_exact(pcs, reference, oracle):
    """coverage_radius / separation (proj/src/metrics.cpp:16-52) on the GPU."""
    import torch

    rng = np.random.default_rng(5)
    for t in range(6):
        n = int(rng.integers(10, 3000))
        pts = synth.random_cloud(n, 70 + t)
        if t % 2:
            pts[: n // 3] = pts[0]
        idx = pcs.npdu_afps(pts, max(2, n // 7), 3, 33, seed=t)[0]
        assert pcs.coverage_radius(pts, idx) == reference.coverage_radius(pts, idx)
        assert pcs.separation(pts, idx) == reference.separation(pts, idx)
        assert pcs.coverage_radius(pts, idx) == oracle.coverage_radius(pts, idx)
    with pytest.raises(ValueError, match="coverage_radius: sample set is empty"):
        pcs.coverage_radius(pts, np.zeros(0, np.int64))
    with pytest.raises(ValueError, match="separation: need at least 2 samples"):
        pcs.separation(pts, np.zeros(1, np.int64))
    with pytest.raises(ValueError, match="coverage_radius: index out of range"):
        pcs.coverage_radius(pts, np.array([0, 10**6]))
    # batched, device-resident
    xyz = synth.primitives(4, 2048, 4, seed=3)
    dx = torch.from_numpy(xyz).cuda()
    idx, _ = pcs.sample(dx, 512, method="afps", m=8)
    cov, sep = pcs.quality(dx, idx)
    for b in range(4):
        p64 = xyz[b].astype(np.float64)
        ib = idx[b].cpu().numpy()
        assert cov[b].item() == reference.coverage_radius(p64, ib)
        assert sep[b].item() == reference.separation(p64, ib)


def test_bench_harness_csv_matches_reference(reference):
    """run_bench / bench_csv schema and every non-timing column
    (proj/src/bench.cpp:34-136) against the real reference."""
    from paper_2208_08795_b200 import harness

    clouds = {n: synth.stable_sort_np(synth.uniform_cube(1, n, n), 0)[0][0].astype(np.float64)
              for n in (300, 1000)}
    opts = harness.BenchOptions(methods=["fps", "afps", "npdu-fps", "npdu-afps"],
                                n_values=[300, 1000], m_values=[1, 4, 400], k_values=[8, 33],
                                c=120, trials=2, seed=99)
    mine = harness.bench_csv(harness.run_bench(opts, lambda n: clouds[n]))
    ref = reference.run_bench_csv(opts.methods, [clouds[300], clouds[1000]], opts.m_values,
                                  opts.k_values, opts.c, trials=2, seed=99)

    def mask(csv):
        out = []
        for line in csv.strip().split("\n"):
            f = line.split(",")
            if f[0] != "method":
                f[6] = "*"
            out.append(",".join(f))
        return out

    assert mask(mine) == mask(ref)
    assert any("allocate_samples: m exceeds sample count" in l for l in mask(mine))


def test_cli_sample_flow(pcs, reference, tmp_path):
    from paper_2208_08795_b200 import cli

    pts = synth.random_cloud(2000, 4)
    path = tmp_path / "in.bin"
    pcs.write_cloud(pts, str(path), "f32_bin")
    out = tmp_path / "idx.txt"
    assert cli.main(["sample", "--in", str(path), "--method", "npdu-afps", "--c", "256",
                     "--m", "8", "--k", "17", "--seed", "5", "--out", str(out)]) == 0
    got = np.loadtxt(out, dtype=np.int64)
    cloud = reference.read_cloud(path, "f32_bin")
    want = reference.sample("npdu_afps", cloud, 256, 8, 17, "random", 5)[0]
    np.testing.assert_array_equal(got, want)


def test_cuda_graph_capture_and_replay():
    """§8(f1): the batched op is stream-ordered and capturable."""
    import torch

    from paper_2208_08795_b200 import sample

    xyz = torch.from_numpy(synth.primitives(8, 4096, 5, seed=6)).cuda()
    ref = sample(xyz, 1024, method="npdu_afps", m=8, k=65, sort="x")
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        sample(xyz, 1024, method="npdu_afps", m=8, k=65, sort="x")  # warm (attributes set)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = sample(xyz, 1024, method="npdu_afps", m=8, k=65, sort="x")
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(ref, out):
        assert torch.equal(a, b)
    xyz.copy_(torch.from_numpy(synth.primitives(8, 4096, 5, seed=7)).cuda())
    g.replay()
    want = sample(xyz, 1024, method="npdu_afps", m=8, k=65, sort="x")
    torch.cuda.synchronize()
    for a, b in zip(want, out):
        assert torch.equal(a, b)


def test_cpp_dropin_api_kats():
    """The C++ drop-in (include/pcs/*.hpp) against the reference's unit-test
    known answers: tests/cpp/test_pcs_api.cpp, built by _build.py."""
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_2208_08795_b200", "build", "test_pcs_api")
    assert os.path.exists(exe), "run __graft_entry__.build() first"
    p = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    assert "all checks passed" in p.stdout


# ---------------------------------------------------------------- §8(e) multi-GPU
def test_host_multi_device_batch_split():
    """pcs_sample_host_multi, batch split by cloud: several shards on this
    box's one GPU (repeated ordinals run in turn on its stream set) give the
    one-device results -- indices, sector_of, stats, permutation."""
    from paper_2208_08795_b200 import sample_host_batch

    xyz = synth.primitives(13, 4096, 5, seed=6)
    one = sample_host_batch(xyz, 1024, method="npdu_afps", m=8, k=65, sort="x",
                            return_sector=True, first="random", seed=11,
                            seeds=np.arange(13) * 7 + 1)
    for devices in ([0], [0, 0], [0, 0, 0], [0] * 13, [0] * 20):
        got = sample_host_batch(xyz, 1024, method="npdu_afps", m=8, k=65, sort="x",
                                return_sector=True, first="random", seed=11,
                                seeds=np.arange(13) * 7 + 1, devices=devices)
        for a, b in zip(one, got):
            np.testing.assert_array_equal(a, b, err_msg=str(devices))


@pytest.mark.parametrize("meth,n,c,m,k", [("afps", 1 << 20, 1 << 18, 1024, None),
                                          ("npdu_afps", 100003, 9001, 37, 33)])
def test_host_multi_device_sector_split(oracle, meth, n, c, m, k):
    """pcs_sample_host_multi on ONE large cloud: sector runs per device
    (BASELINE cfg5's 1M-point cloud, M=1024), every device sorting the cloud
    itself; equal to the one-device call and to the oracle."""
    from paper_2208_08795_b200 import sample_host_batch

    xyz = synth.uniform_cube(1, n, 23)
    one = sample_host_batch(xyz, c, method=meth, m=m, k=k, sort="x", return_sector=True,
                            first="random", seed=5)
    for devices in ([0, 0], [0, 0, 0], [0] * 8):
        got = sample_host_batch(xyz, c, method=meth, m=m, k=k, sort="x", return_sector=True,
                                first="random", seed=5, devices=devices)
        for a, b in zip(one, got):
            np.testing.assert_array_equal(a, b, err_msg=str(devices))
    srt = synth.stable_sort_np(xyz, 0)[0]
    idx, sec, st = oracle.sample(meth, srt[0].astype(np.float64), c, m, k or 0, "random", 5)
    np.testing.assert_array_equal(one[0][0], idx)
    np.testing.assert_array_equal(one[2][0], sec)
    np.testing.assert_array_equal(one[1][0], st.astype(np.int64))


def _rank_worker(rank, world, port, q):
    """One rank of the torchrun layout, both on cuda:0: the product path
    (sort + sample of this rank's sectors with the global bases, or of its
    clouds), then the end-of-batch gather over gloo."""
    import torch
    import torch.distributed as dist

    from paper_2208_08795_b200 import sample, shard, sort_axis

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    n, c, m, k = 65536, 8192, 64, 65
    xyz = torch.from_numpy(synth.uniform_cube(1, n, 31)).cuda()
    srt = sort_axis(xyz, "x")[0]
    sh = shard.sector_shard(n, c, m, world, rank)
    idx, st, sec = shard.sample_sector_shard(srt, sh, "npdu_afps", k, first="random", seed=3)
    rows = shard.gather_rows(torch.stack([idx[0], sec[0]], 1).cpu(), c, world)
    stats = st[0].cpu()
    dist.all_reduce(stats)
    clouds = synth.primitives(6, 2048, 4, seed=2)
    b0, b1 = shard.split(6, world, rank)
    bi = sample(torch.from_numpy(clouds[b0:b1]).cuda(), 512, method="afps", m=8)[0].cpu()
    brows = shard.gather_rows(bi, 6, world)
    if rank == 0:
        q.put((rows.numpy(), stats.numpy(), brows.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_on_the_product_path_equal_one_call(world):
    """The multi-GPU layout of bench.py / shard.py with `world` ranks (all on
    this box's cuda:0, gloo for the one end-of-batch gather): sector-split
    NPDU-AFPS of one cloud and cloud-split AFPS of a batch equal the
    single-process call bit for bit."""
    import socket

    import torch
    import torch.multiprocessing as mp

    from paper_2208_08795_b200 import sample

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    rows, stats, brows = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    xyz = torch.from_numpy(synth.uniform_cube(1, 65536, 31)).cuda()
    idx, st, sec, _ = sample(xyz, 8192, method="npdu_afps", m=64, k=65, sort="x",
                             first="random", seed=3, return_sector=True)
    np.testing.assert_array_equal(rows[:, 0], idx[0].cpu().numpy())
    np.testing.assert_array_equal(rows[:, 1], sec[0].cpu().numpy())
    np.testing.assert_array_equal(stats, st[0].cpu().numpy())
    clouds = synth.primitives(6, 2048, 4, seed=2)
    want = sample(torch.from_numpy(clouds).cuda(), 512, method="afps", m=8)[0].cpu().numpy()
    np.testing.assert_array_equal(brows, want)


def test_concurrent_callers_equal_serial(pcs):
    """The b4 contract (reentrant, schedule-independent calls,
    proj/tests/test_sampler.cpp:245-252): 8 host threads calling the drop-in
    samplers and the host-batch entry at once (the GIL is released around
    the native calls) get exactly the serial results."""
    from concurrent.futures import ThreadPoolExecutor

    clouds = [synth.random_cloud(3000 + 97 * i, 40 + i) for i in range(8)]
    batch = synth.primitives(6, 4096, 4, seed=8)

    def job(i):
        if i % 3 == 0:
            return pcs.npdu_afps(clouds[i], 600, 6, 33, seed=i, first="random")
        if i % 3 == 1:
            return pcs.afps(clouds[i], 500, 4, seed=i)
        return pcs.sample_host_batch(batch, 1024, method="npdu_afps", m=8, k=65, sort="x")

    serial = [job(i) for i in range(8)]
    for _ in range(3):
        with ThreadPoolExecutor(8) as ex:
            par = list(ex.map(job, range(8)))
        for a, b in zip(serial, par):
            np.testing.assert_array_equal(a[0], b[0])
            if isinstance(a[2], dict):
                assert a[2] == b[2]
            else:
                np.testing.assert_array_equal(a[1], b[1])


@pytest.mark.parametrize("meth,B,n,c,m,k,dtype,knob", [
    ("afps", 9, 3000, 700, 3, None, "float32", None),             # fps_full
    ("npdu_afps", 3, 4096, 1024, 8, 65, "float32", None),         # npdu_wide
    ("npdu_afps", 40, 4096, 1024, 8, 129, "float32", None),       # npdu_tmem
    ("npdu_afps", 40, 4096, 1024, 8, 129, "float64", None),       # npdu_warp (fp64)
    ("fps", 3, 9000, 700, 1, None, "float32", None),              # morton_tmem
    ("npdu_fps", 2, 9000, 900, 1, 65, "float32", None),           # morton_tmem, window mode
    ("fps", 2, 9000, 700, 1, None, "float64", None),              # morton_rows (fp64)
    ("afps", 2, 5000, 600, 2, None, "float32", ("PCS_SAMPLER", "rows")),
    ("afps", 2, 5000, 300, 2, None, "float32", ("PCS_SAMPLER", "stream")),
])
def test_sampling_through_the_sort_permutation(monkeypatch, meth, B, n, c, m, k, dtype, knob):
    """sample(..., sort=axis) hands the sampler the sort permutation only
    (pcs_gpu_args.perm: staging gathers through it, or a sorted copy for the
    engines that re-read global memory); every kernel family gives exactly
    the results of sampling the gathered sorted copy."""
    import torch

    import paper_2208_08795_b200 as pcs
    from paper_2208_08795_b200 import sample, sort_axis

    if knob:
        setknob(monkeypatch, *knob)
    xyz = synth.primitives(B, n, 4, seed=n + B).astype(dtype)
    xyz[:, 10:40] = xyz[:, 9:10]  # coincident points: ties in the sort and the argmax
    x = torch.from_numpy(xyz).cuda()
    fused = sample(x, c, method=meth, m=m, k=k, sort="y", first="random", seed=7,
                   return_sector=True)
    srt, perm = sort_axis(x, "y")
    copy = sample(srt, c, method=meth, m=m, k=k, first="random", seed=7, return_sector=True)
    assert torch.equal(fused[3], perm)
    for a, b in zip(fused[:3], copy):
        assert torch.equal(a, b), pcs.kernel_family(meth, n, m, k, dtype=dtype, batch=B)
