"""CPU-only checks of the boundary and host logic: the C-ABI library loads and
exports every entry point include/pcs_gpu.h declares, argument validation
matches the reference's exceptions, the generators are deterministic, and the
multi-GPU sharding math reproduces the single-process result (gloo, 2 ranks).
No kernel is launched here."""
import ctypes
import os
import re
import socket

import numpy as np
import pytest

from conftest import ROOT, setknob
from paper_2208_08795_b200 import shard, synth


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "pcs_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pcs_[a-z_0-9]+)\s*\(", src)))


def test_cabi_exports_every_declared_symbol(pcs):
    lib = ctypes.CDLL(pcs.LIB_PATH)
    names = _declared_functions()
    assert {"pcs_gpu_sample", "pcs_gpu_sort_axis", "pcs_sample_host", "pcs_local_fps_host",
            "pcs_exact_sort_host", "pcs_last_error"} <= set(names)
    for name in names:
        assert hasattr(lib, name), name
    lib.pcs_abi_version.restype = ctypes.c_int
    assert lib.pcs_abi_version() == 2
    lib.pcs_status_string.restype = ctypes.c_char_p
    assert lib.pcs_status_string(1) == b"invalid argument"


def test_cabi_rejects_before_touching_the_device(pcs):
    # pcs_sample_host validates on the host first: no GPU needed for errors.
    lib = ctypes.CDLL(pcs.LIB_PATH)
    lib.pcs_last_error.restype = ctypes.c_char_p
    pts = np.zeros((4, 3))
    out = np.zeros(8, np.int64)
    st = np.zeros(4, np.uint64)
    rc = lib.pcs_sample_host(2, pts.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(4),
                             ctypes.c_int64(3), ctypes.c_int64(5), ctypes.c_int64(0), 1,
                             ctypes.c_uint64(0), 1, out.ctypes.data_as(ctypes.c_void_p),
                             out.ctypes.data_as(ctypes.c_void_p), st.ctypes.data_as(ctypes.c_void_p))
    assert rc == 1
    assert lib.pcs_last_error() == b"partition_sectors: m exceeds point count"


class _Args(ctypes.Structure):
    """pcs_gpu_args (include/pcs_gpu.h, ABI v2)."""
    _fields_ = [("method", ctypes.c_int32), ("coord_dtype", ctypes.c_int32),
                ("xyz", ctypes.c_void_p), ("batch", ctypes.c_int64), ("n", ctypes.c_int64),
                ("c", ctypes.c_int64), ("m", ctypes.c_int64), ("k", ctypes.c_int64),
                ("seed_policy", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("seeds", ctypes.c_void_p), ("index_dtype", ctypes.c_int32),
                ("out_indices", ctypes.c_void_p), ("out_sector", ctypes.c_void_p),
                ("out_stats", ctypes.c_void_p), ("index_base", ctypes.c_int64),
                ("sector_base", ctypes.c_int64), ("perm", ctypes.c_void_p)]


def test_multi_device_and_plan_entries_validate_on_the_host(pcs):
    """pcs_sample_host_multi / pcs_kernel_family reject bad arguments with
    the reference's messages (or their own) before any device call."""
    lib = ctypes.CDLL(pcs.LIB_PATH)
    lib.pcs_last_error.restype = ctypes.c_char_p
    pts = np.zeros((1, 10, 3), np.float32)
    out = np.zeros(16, np.int32)
    a = _Args(method=2, coord_dtype=0, xyz=pts.ctypes.data, batch=1, n=10, c=4, m=5, k=0,
              seed_policy=1, index_dtype=0, out_indices=out.ctypes.data)
    devs = (ctypes.c_int32 * 2)(0, 0)
    assert lib.pcs_sample_host_multi(ctypes.byref(a), -1, None, devs, 2) == 1
    assert lib.pcs_last_error() == b"allocate_samples: m exceeds sample count"
    a.m = 2
    assert lib.pcs_sample_host_multi(ctypes.byref(a), -1, None, devs, 0) == 1
    assert lib.pcs_last_error() == b"pcs_sample_host_multi: need at least one device"
    a.perm = out.ctypes.data
    assert lib.pcs_sample_host_batch(ctypes.byref(a), -1, None, 0) == 1
    assert b"perm is a device-call field" in lib.pcs_last_error()
    a.perm = None
    name = ctypes.create_string_buffer(64)
    assert lib.pcs_kernel_family(ctypes.byref(a), name, 64) == 0
    assert name.value == b"fps_full_kernel<1,1,1>"
    a.c = 11
    assert lib.pcs_kernel_family(ctypes.byref(a), name, 64) == 1
    assert lib.pcs_last_error() == b"afps: c exceeds point count"


BAD = [("fps", 0, 1, 1), ("fps", 11, 1, 1), ("afps", 4, 5, 1), ("afps", 11, 2, 1),
       ("afps", 4, 0, 1), ("npdu_afps", 4, 20, 3), ("npdu_fps", 4, 1, 0), ("npdu_afps", 4, 2, 0),
       ("npdu_afps", 10, 10, 0)]


@pytest.mark.parametrize("meth,c,m,k", BAD)
def test_validation_messages_match_reference(pcs, reference, meth, c, m, k):
    pts = synth.random_cloud(10, 1)
    with pytest.raises(ValueError) as mine:
        pcs._core.validate({"fps": 1, "afps": 2, "npdu_fps": 3, "npdu_afps": 4}[meth], 10, c, m, k)
    with pytest.raises(ValueError) as ref:
        reference.sample(meth, pts, c, m, k)
    assert str(mine.value) == str(ref.value)


def test_python_surface_matches_reference_signatures(pcs):
    # proj/bindings/pcsample_module.cpp:150-190: names, kwargs, defaults
    pts = synth.random_cloud(10, 1)
    with pytest.raises(ValueError, match="c must be >= 1"):
        pcs.fps(pts, 0)
    with pytest.raises(ValueError, match="first must be 'random' or 'fixed'"):
        pcs.afps(pts, 4, 2, seed=0, first="bogus", threads=4)
    with pytest.raises(ValueError, match="expected an \\(N, 3\\) array"):
        pcs.npdu_fps(np.zeros((4, 2)), 2, 3)
    with pytest.raises(ValueError, match="axis must be x, y, or z"):
        pcs.exact_sort(pts, axis="w")
    with pytest.raises(ValueError, match="local_fps: window size must be >= 1"):
        pcs.npdu_afps(pts, 4, 2, 0, seed=1, first="random", threads=2)


def test_generators_deterministic_and_shaped():
    a = synth.uniform_cube(2, 100, 5)
    assert a.dtype == np.float32 and a.shape == (2, 100, 3)
    np.testing.assert_array_equal(a, synth.uniform_cube(2, 100, 5))
    assert np.abs(a).max() <= 1.0
    p = synth.primitives(2, 2048, 4, seed=1)
    assert p.shape == (2, 2048, 3) and np.isfinite(p).all()
    assert np.linalg.norm(p, axis=-1).max() <= 1.0 + 1e-6
    np.testing.assert_array_equal(p, synth.primitives(2, 2048, 4, seed=1))
    lid = synth.lidar_sweep(1, seed=3)
    r = np.linalg.norm(lid[0].astype(np.float64), axis=1)
    assert lid.shape == (1, 32768, 3) and r.min() > 1.9 and r.max() < 80.2


def test_split_and_sector_shards_tile_the_plan():
    for total, world in [(128, 8), (10, 3), (3, 8), (1024, 8)]:
        spans = [shard.split(total, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == total
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    n, c, m = 10007, 2501, 37
    shards = [shard.sector_shard(n, c, m, 4, r) for r in range(4)]
    assert shards[0].point_lo == 0 and shards[-1].point_hi == n
    assert sum(s.c for s in shards) == c and sum(s.m for s in shards) == m


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_q):
    import torch
    import torch.distributed as dist

    from oracle import Oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    # one big cloud, AFPS sectors split across ranks (the 1M-point row of
    # BASELINE cfg5 in miniature)
    n, c, m, k = 4099, 1031, 16, 9
    pts = synth.uniform_cube(1, n, 11)[0].astype(np.float64)
    sh = shard.sector_shard(n, c, m, world, rank)
    idx, sec, st = orc.sample("npdu_afps", pts[sh.point_lo:sh.point_hi], sh.c, sh.m, k)
    local = torch.from_numpy(np.stack([idx + sh.point_lo, sec + sh.sector_lo], 1))
    rows = shard.gather_rows(local, c, world)
    stats = torch.from_numpy(st.astype(np.int64))
    dist.all_reduce(stats)
    # batch of clouds split by cloud
    clouds = synth.uniform_cube(5, 300, 3)
    b0, b1 = shard.split(5, world, rank)
    bi, bst = orc.sample_batch_f32("afps", clouds[b0:b1], 64, 4) if b1 > b0 else (
        np.zeros((0, 64), np.int64), np.zeros((0, 4), np.uint64))
    brows = shard.gather_rows(torch.from_numpy(bi), 5, world)
    if rank == 0:
        result_q.put((rows.numpy(), stats.numpy(), brows.numpy()))
    dist.destroy_process_group()


def test_gloo_two_rank_sharding_equals_single_process(oracle):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    rows, stats, brows = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, c, m, k = 4099, 1031, 16, 9
    pts = synth.uniform_cube(1, n, 11)[0].astype(np.float64)
    idx, sec, st = oracle.sample("npdu_afps", pts, c, m, k)
    np.testing.assert_array_equal(rows[:, 0], idx)
    np.testing.assert_array_equal(rows[:, 1], sec)
    np.testing.assert_array_equal(stats, st.astype(np.int64))
    bi, _ = oracle.sample_batch_f32("afps", synth.uniform_cube(5, 300, 3), 64, 4)
    np.testing.assert_array_equal(brows, bi)


# ---------------------------------------------------------------- f2: io
def test_cloud_files_round_trip_and_match_reference(pcs, reference, tmp_path):
    pts = synth.random_cloud(50, 9)
    pts[3] = [-0.0, 1e-300, 3.5e38]
    for fmt in ("xyz_text", "f32_bin"):
        p = tmp_path / f"c.{fmt}"
        pcs.write_cloud(pts, str(p), fmt)
        mine = pcs.read_cloud(str(p), fmt)
        np.testing.assert_array_equal(mine, reference.read_cloud(p, fmt))
        q = tmp_path / f"r.{fmt}"
        reference.write_cloud(q, fmt, pts)
        assert p.read_bytes() == q.read_bytes()
    np.testing.assert_array_equal(pcs.read_cloud(str(tmp_path / "c.xyz_text"), "xyz_text"), pts)


@pytest.mark.parametrize("content,fmt", [
    (b"", "xyz_text"), (b"# only a comment\n\n", "xyz_text"), (b"1 2\n", "xyz_text"),
    (b"1 2 3\n4 5 6 7\n", "xyz_text"), (b"", "f32_bin"), (b"\x00" * 13, "f32_bin")])
def test_cloud_file_errors_match_reference(pcs, reference, tmp_path, content, fmt):
    p = tmp_path / "bad"
    p.write_bytes(content)
    with pytest.raises(RuntimeError) as mine:
        pcs.read_cloud(str(p), fmt)
    with pytest.raises(RuntimeError) as ref:
        reference.read_cloud(p, fmt)
    assert str(mine.value) == str(ref.value)
    with pytest.raises(RuntimeError, match="cannot open"):
        pcs.read_cloud(str(tmp_path / "missing"), fmt)


def test_cli_usage_errors_exit_2():
    from paper_2208_08795_b200 import cli

    assert cli.main(["sample"]) == 2
    assert cli.main(["frobnicate"]) == 2


def test_kernel_family_is_the_dispatch_decision(pcs, monkeypatch):
    """pcs_kernel_family runs csrc/sample_dispatch.cu in plan mode (no GPU
    needed): the 8-warp NPDU form for calls of <= 148 sectors
    (PCS_NPDU_WIDE moves it), the one-warp TMEM kernel above, full / Morton
    kernels for full windows, the streaming engine past every on-chip one."""
    for var in ("PCS_NPDU_WIDE", "PCS_SAMPLER", "PCS_MORTON", "PCS_MORTON_MIN", "PCS_NPDU_TMEM"):
        setknob(monkeypatch, var, None)
    kf = pcs.kernel_family
    assert kf("npdu_afps", 32768, 32, 129, batch=4) == "npdu_wide_kernel"      # 128 sectors
    assert kf("npdu_afps", 32768, 32, 129, batch=5) == "npdu_tmem_kernel"      # 160 sectors
    assert kf("npdu_afps", 32768, 32, 129, batch=128) == "npdu_tmem_kernel"    # cfg4
    assert kf("npdu_fps", 4096, 1, 65, batch=1) == "npdu_wide_kernel"
    assert kf("npdu_fps", 8192, 1, 65, batch=1) == "morton_tmem_kernel"        # > 4096 points
    assert kf("afps", 2048, 8, batch=16) == "fps_full_kernel"                  # cfg2
    assert kf("fps", 8192, 1, batch=64) == "morton_tmem_kernel"                # cfg3 FPS
    assert kf("npdu_afps", 32768, 32, 129, batch=128, full=True) == "npdu_tmem_kernel<5,1024,3>"
    assert kf("npdu_afps", 32768, 32, 129, batch=16, full=True) == "npdu_tmem_kernel<5,1024,1>"
    assert kf("npdu_afps", 8192, 16, 65, batch=64, full=True) == "npdu_tmem_kernel<3,512,0>"
    assert kf("fps", 1 << 20) == "stream_sector_kernel"
    assert kf("afps", 1 << 20, 1024, batch=1, full=True) == "fps_full_kernel<8,4,1>"
    setknob(monkeypatch, "PCS_NPDU_WIDE", "0")
    assert kf("npdu_afps", 32768, 32, 129, batch=1) == "npdu_tmem_kernel"
