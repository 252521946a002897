"""CPU checkers -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs. Two ctypes faces:

* ``Oracle``    -- oracle/liboracle.so, the plain-C restatement of the
  reference hot path (pcs_oracle.c, each function cites the reference
  file:line it follows).
* ``Reference`` -- oracle/_ref/libpcsref.so, the unmodified reference
  (/root/reference/proj/src) compiled by oracle/Makefile, plus ref_shim.cpp.

Methods are numbered as in the C-ABI (include/pcs_gpu.h): 1 fps, 2 afps,
3 npdu_fps, 4 npdu_afps. ``k=0`` means "no window".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
METHODS = {"fps": 1, "afps": 2, "npdu_fps": 3, "npdu_afps": 4}

_u64, _i64p, _u64p = C.c_uint64, C.POINTER(C.c_int64), C.POINTER(C.c_uint64)
_dp, _fp = C.POINTER(C.c_double), C.POINTER(C.c_float)


class OracleError(ValueError):
    pass


def build():
    """Compile liboracle.so and, when /root/reference is present, _ref/."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a, t):
    return a.ctypes.data_as(t)


def _load(path):
    if not os.path.exists(path):
        raise FileNotFoundError(path + " (run `make -C oracle`)")
    return C.CDLL(path)


class Oracle:
    """C restatement (pcs_oracle.c)."""

    def __init__(self):
        lib = _load(os.path.join(HERE, "liboracle.so"))
        lib.or_sample.argtypes = [C.c_int, _dp, _u64, _u64, _u64, _u64, C.c_int, _u64,
                                  _i64p, _i64p, _u64p, C.c_char_p, C.c_size_t]
        lib.or_local_fps.argtypes = [_dp, _u64, _u64, _u64, _u64, C.c_int, _u64, C.c_int,
                                     _u64, _i64p, _u64p, _dp, C.c_char_p, C.c_size_t]
        lib.or_exact_sort.argtypes = [_dp, _u64, C.c_int, _i64p, _dp]
        lib.or_sample_batch_f32.argtypes = [C.c_int, _fp, _u64, _u64, _u64, _u64, _u64,
                                            _u64, C.c_int, _u64, _i64p, _u64p,
                                            C.c_char_p, C.c_size_t]
        lib.or_coverage_radius.argtypes = [_dp, _u64, _i64p, _u64]
        lib.or_coverage_radius.restype = C.c_double
        lib.or_separation.argtypes = [_dp, _i64p, _u64]
        lib.or_separation.restype = C.c_double
        lib.or_splitmix_next.argtypes = [_u64p]
        lib.or_splitmix_next.restype = _u64
        lib.or_splitmix_below.argtypes = [_u64p, _u64]
        lib.or_splitmix_below.restype = _u64
        lib.or_update_window.argtypes = [_u64, _u64, _u64, _u64, _u64p, _u64p]
        lib.or_sector_plan.argtypes = [_u64, _u64, _u64, _u64p, _u64p, _u64p,
                                       C.c_char_p, C.c_size_t]
        self.lib = lib

    def sample(self, method, pts, c, m=1, k=0, first="fixed", seed=0):
        """-> (int64 idx[c], int64 sector_of[c], uint64 stats[4])."""
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        idx = np.zeros(max(c, 1), np.int64)
        sec = np.zeros(max(c, 1), np.int64)
        st = np.zeros(4, np.uint64)
        err = C.create_string_buffer(256)
        rc = self.lib.or_sample(METHODS[method] if isinstance(method, str) else method,
                                _ptr(pts, _dp), len(pts), c, m, k, first == "random",
                                seed, _ptr(idx, _i64p), _ptr(sec, _i64p), _ptr(st, _u64p),
                                err, 256)
        if rc:
            raise OracleError(err.value.decode())
        return idx[:c], sec[:c], st

    def local_fps(self, pts, sb, se, quota, k=0, first="fixed", seed=0, trace=False):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        idx = np.zeros(max(quota, 1), np.int64)
        st = np.zeros(4, np.uint64)
        tr = np.zeros((max(quota - 1, 1), se - sb)) if trace else None
        err = C.create_string_buffer(256)
        rc = self.lib.or_local_fps(_ptr(pts, _dp), len(pts), sb, se, quota, int(k > 0), k,
                                   first == "random", seed, _ptr(idx, _i64p),
                                   _ptr(st, _u64p), _ptr(tr, _dp) if trace else None,
                                   err, 256)
        if rc:
            raise OracleError(err.value.decode())
        return (idx[:quota], st, tr[: quota - 1]) if trace else (idx[:quota], st)

    def exact_sort(self, pts, axis=0):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        perm = np.zeros(len(pts), np.int64)
        out = np.zeros_like(pts)
        self.lib.or_exact_sort(_ptr(pts, _dp), len(pts), axis, _ptr(perm, _i64p),
                               _ptr(out, _dp))
        return perm, out

    def sample_batch_f32(self, method, xyz, c, m=1, k=0, first="fixed", seed=0,
                         lo=0, hi=None):
        """xyz float32 (B, N, 3) -> (int64 (B, c), uint64 (B, 4)); clouds [lo, hi)."""
        xyz = np.ascontiguousarray(xyz, dtype=np.float32)
        B, N = xyz.shape[0], xyz.shape[1]
        hi = B if hi is None else hi
        idx = np.zeros((B, c), np.int64)
        st = np.zeros((B, 4), np.uint64)
        err = C.create_string_buffer(256)
        rc = self.lib.or_sample_batch_f32(METHODS[method] if isinstance(method, str) else method,
                                          _ptr(xyz, _fp), lo, hi, N, c, m, k,
                                          first == "random", seed, _ptr(idx, _i64p),
                                          _ptr(st, _u64p), err, 256)
        if rc:
            raise OracleError(err.value.decode())
        return idx, st

    def coverage_radius(self, pts, samples):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        s = np.ascontiguousarray(samples, dtype=np.int64)
        return self.lib.or_coverage_radius(_ptr(pts, _dp), len(pts), _ptr(s, _i64p), len(s))

    def separation(self, pts, samples):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        s = np.ascontiguousarray(samples, dtype=np.int64)
        return self.lib.or_separation(_ptr(pts, _dp), _ptr(s, _i64p), len(s))

    def splitmix(self, seed, count):
        s = C.c_uint64(seed)
        return [self.lib.or_splitmix_next(C.byref(s)) for _ in range(count)]

    def update_window(self, sb, se, idx, k):
        a, b = C.c_uint64(), C.c_uint64()
        self.lib.or_update_window(sb, se, idx, k, C.byref(a), C.byref(b))
        return a.value, b.value


class Reference:
    """The unmodified reference, compiled into oracle/_ref/libpcsref.so."""

    PATH = os.path.join(HERE, "_ref", "libpcsref.so")

    @classmethod
    def available(cls):
        return os.path.exists(cls.PATH)

    def __init__(self):
        lib = _load(self.PATH)
        lib.ref_sample.argtypes = [C.c_int, _dp, _u64, _u64, _u64, _u64, C.c_int, _u64,
                                   C.c_uint, _i64p, _i64p, _u64p, C.c_char_p, C.c_size_t]
        lib.ref_local_fps_trace.argtypes = [_dp, _u64, _u64, _u64, _u64, C.c_int, _u64,
                                            C.c_int, _u64, _i64p, _u64p, _dp, C.c_char_p,
                                            C.c_size_t]
        lib.ref_exact_sort.argtypes = [_dp, _u64, C.c_int, _dp]
        lib.ref_sample_batch_f32.argtypes = [C.c_int, _fp, _u64, _u64, _u64, _u64, _u64,
                                             C.c_int, _u64, C.c_uint, _i64p, _u64p, _dp,
                                             C.c_char_p, C.c_size_t]
        lib.ref_metric.argtypes = [C.c_int, _dp, _u64, _i64p, _u64, _dp, C.c_char_p, C.c_size_t]
        lib.ref_read_cloud.argtypes = [C.c_char_p, C.c_int, _dp, _u64, C.c_char_p, C.c_size_t]
        lib.ref_read_cloud.restype = C.c_longlong
        lib.ref_write_cloud.argtypes = [C.c_char_p, C.c_int, _dp, _u64]
        lib.ref_run_bench_csv.restype = C.c_longlong
        self.lib = lib

    def metric(self, which, pts, samples):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        s = np.ascontiguousarray(samples, dtype=np.int64)
        out = np.zeros(1)
        err = C.create_string_buffer(256)
        if self.lib.ref_metric(which, _ptr(pts, _dp), len(pts), _ptr(s, _i64p), len(s),
                               _ptr(out, _dp), err, 256):
            raise OracleError(err.value.decode())
        return float(out[0])

    def coverage_radius(self, pts, samples):
        return self.metric(0, pts, samples)

    def separation(self, pts, samples):
        return self.metric(1, pts, samples)

    def read_cloud(self, path, fmt):
        cap = 1 << 22
        buf = np.zeros((cap, 3))
        err = C.create_string_buffer(512)
        n = self.lib.ref_read_cloud(str(path).encode(), 0 if fmt == "xyz_text" else 1,
                                    _ptr(buf, _dp), cap, err, 512)
        if n < 0:
            raise RuntimeError(err.value.decode())
        return buf[:n].copy()

    def write_cloud(self, path, fmt, pts):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        self.lib.ref_write_cloud(str(path).encode(), 0 if fmt == "xyz_text" else 1,
                                 _ptr(pts, _dp), len(pts))

    def run_bench_csv(self, methods, clouds, m_values, k_values, c, trials=1, seed=0,
                      first="random", threads=1, g=40):
        """clouds: list of float64 (n, 3) arrays (distinct n). Methods are
        pcs::Method names (rps, fps, afps, npdu-fps, npdu-afps, grid)."""
        names = ["rps", "fps", "afps", "npdu-fps", "npdu-afps", "grid"]
        meth = np.array([names.index(m) for m in methods], np.int32)
        offs, at = [], 0
        for cl in clouds:
            offs.append(at)
            at += len(cl)
        xyz = np.ascontiguousarray(np.concatenate(clouds), dtype=np.float64)
        offs = np.array(offs, np.uint64)
        ns = np.array([len(cl) for cl in clouds], np.uint64)
        ms, ks = np.array(m_values, np.uint64), np.array(k_values, np.uint64)
        cap = 1 << 20
        out = C.create_string_buffer(cap)
        self.lib.ref_run_bench_csv(
            meth.ctypes.data_as(C.c_void_p), C.c_uint64(len(meth)), _ptr(xyz, _dp),
            offs.ctypes.data_as(C.c_void_p), ns.ctypes.data_as(C.c_void_p), C.c_uint64(len(ns)),
            ms.ctypes.data_as(C.c_void_p), C.c_uint64(len(ms)), ks.ctypes.data_as(C.c_void_p),
            C.c_uint64(len(ks)), C.c_uint64(c), C.c_uint64(g), C.c_uint64(trials),
            C.c_uint64(seed), C.c_int(first == "random"), C.c_uint(threads), out, C.c_size_t(cap))
        return out.value.decode()

    def sample(self, method, pts, c, m=1, k=0, first="fixed", seed=0, threads=1):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        idx = np.zeros(max(c, 1), np.int64)
        sec = np.zeros(max(c, 1), np.int64)
        st = np.zeros(4, np.uint64)
        err = C.create_string_buffer(256)
        rc = self.lib.ref_sample(METHODS[method] if isinstance(method, str) else method,
                                 _ptr(pts, _dp), len(pts), c, m, k, first == "random",
                                 seed, threads, _ptr(idx, _i64p), _ptr(sec, _i64p),
                                 _ptr(st, _u64p), err, 256)
        if rc:
            raise OracleError(err.value.decode())
        return idx[:c], sec[:c], st

    def local_fps_trace(self, pts, sb, se, quota, k=0, first="fixed", seed=0):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        idx = np.zeros(max(quota, 1), np.int64)
        st = np.zeros(4, np.uint64)
        tr = np.zeros((max(quota - 1, 1), se - sb))
        err = C.create_string_buffer(256)
        rc = self.lib.ref_local_fps_trace(_ptr(pts, _dp), len(pts), sb, se, quota,
                                          int(k > 0), k, first == "random", seed,
                                          _ptr(idx, _i64p), _ptr(st, _u64p), _ptr(tr, _dp),
                                          err, 256)
        if rc:
            raise OracleError(err.value.decode())
        return idx[:quota], st, tr[: quota - 1]

    def exact_sort(self, pts, axis=0):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        out = np.zeros_like(pts)
        self.lib.ref_exact_sort(_ptr(pts, _dp), len(pts), axis, _ptr(out, _dp))
        return out

    def sample_batch_f32(self, method, xyz, c, m=1, k=0, first="fixed", seed=0, workers=1):
        """-> (idx int64 (B, c), stats uint64 (B, 4), seconds of the worker phase)."""
        xyz = np.ascontiguousarray(xyz, dtype=np.float32)
        B, N = xyz.shape[0], xyz.shape[1]
        idx = np.zeros((B, c), np.int64)
        st = np.zeros((B, 4), np.uint64)
        secs = np.zeros(1)
        err = C.create_string_buffer(256)
        rc = self.lib.ref_sample_batch_f32(METHODS[method] if isinstance(method, str) else method,
                                           _ptr(xyz, _fp), B, N, c, m, k, first == "random",
                                           seed, workers, _ptr(idx, _i64p), _ptr(st, _u64p),
                                           _ptr(secs, _dp), err, 256)
        if rc < 0:
            raise OracleError(err.value.decode())
        return idx, st, float(secs[0])
