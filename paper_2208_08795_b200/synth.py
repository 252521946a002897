"""Seeded synthetic inputs for the BASELINE.json configurations (host numpy).

Not on the hot path: these make the fp32 ``(B, N, 3)`` batches that both the
GPU kernels and the CPU reference consume, byte for byte. The reference's own
generators (proj/src/synth.cpp) do not produce these shapes, so they are
written fresh here, as SURVEY.md §8(d) specifies:

* ``splitmix_uniform`` / ``random_cloud`` -- SplitMix64 ``uniform(lo, hi)``
  streams (proj/include/pcs/rng.hpp:16-36), identical to the reference test
  helpers' ``random_cloud`` (proj/tests/test_helpers.hpp:20-26,
  proj/tests/acceptance_main.cpp:42-50), so the reference's known-answer
  tests replay on the same doubles.
* ``uniform_cube``   -- cfg1 / cfg5: iid uniform in [-1, 1]^3, cloud b from
  SplitMix64(seed + b), point-major x, y, z, narrowed to fp32.
* ``primitives``     -- cfg2 / cfg3: sphere / box / cylinder surfaces, centre
  U[-0.5, 0.5]^3, size U[0.1, 0.5], points proportional to area,
  N(0, 0.005) noise, centred and scaled into the unit sphere.
* ``lidar_sweep``    -- cfg4: 64 rings (elevation -25..+3 deg) x 512
  azimuths ray-cast against the ground plane z = -1.7 m and 20 random
  axis-aligned boxes (edges 1-5 m), range clipped to [2, 80] m (no hit ->
  80 m), N(0, 0.02 m) range noise, stored azimuth-major (no sort).
"""
from __future__ import annotations

import numpy as np

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix_next(seed: int, count: int, start: int = 0) -> np.ndarray:
    """Outputs start+1 .. start+count of SplitMix64(seed).next(), vectorised
    (state after i calls is seed + i * golden, mod 2^64)."""
    i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & (2**64 - 1)) + i * _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def splitmix_uniform(seed: int, count: int, lo: float, hi: float) -> np.ndarray:
    u = (splitmix_next(seed, count) >> np.uint64(11)).astype(np.float64) * 2.0**-53
    return lo + (hi - lo) * u


def random_cloud(n: int, seed: int, extent: float = 10.0) -> np.ndarray:
    """float64 (n, 3): the reference tests' random_cloud(n, seed, extent)."""
    return splitmix_uniform(seed, 3 * n, 0.0, extent).reshape(n, 3)


def uniform_cube(batch: int, n: int, seed: int = 0) -> np.ndarray:
    out = np.empty((batch, n, 3), np.float32)
    for b in range(batch):
        out[b] = splitmix_uniform(seed + b, 3 * n, -1.0, 1.0).reshape(n, 3).astype(np.float32)
    return out


def _sphere(rng, k, c, s):
    v = rng.normal(size=(k, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return c + v * (s / 2)


def _box(rng, k, c, dims):
    a, b, h = dims
    faces = np.array([a * b, a * b, b * h, b * h, a * h, a * h])
    f = rng.choice(6, size=k, p=faces / faces.sum())
    u = rng.uniform(-0.5, 0.5, size=(k, 3)) * dims
    axis = np.array([2, 2, 0, 0, 1, 1])[f]
    sign = np.array([1, -1, 1, -1, 1, -1])[f]
    u[np.arange(k), axis] = sign * dims[axis] / 2
    return c + u


def _cylinder(rng, k, c, r, h):
    lat, cap = 2 * np.pi * r * h, 2 * np.pi * r * r
    on_lat = rng.uniform(size=k) < lat / (lat + cap)
    th = rng.uniform(0, 2 * np.pi, size=k)
    rad = np.where(on_lat, r, r * np.sqrt(rng.uniform(size=k)))
    z = np.where(on_lat, rng.uniform(-h / 2, h / 2, size=k),
                 np.where(rng.uniform(size=k) < 0.5, -h / 2, h / 2))
    return c + np.stack([rad * np.cos(th), rad * np.sin(th), z], axis=1)


def primitives(batch: int, n: int, n_prims: int, seed: int = 0) -> np.ndarray:
    out = np.empty((batch, n, 3), np.float32)
    for b in range(batch):
        rng = np.random.default_rng(np.random.SeedSequence([seed, b, n_prims]))
        kinds = rng.integers(0, 3, size=n_prims)
        centres = rng.uniform(-0.5, 0.5, size=(n_prims, 3))
        sizes = rng.uniform(0.1, 0.5, size=(n_prims, 3))
        areas = np.empty(n_prims)
        for p in range(n_prims):
            s = sizes[p]
            if kinds[p] == 0:
                areas[p] = np.pi * s[0] ** 2
            elif kinds[p] == 1:
                areas[p] = 2 * (s[0] * s[1] + s[1] * s[2] + s[0] * s[2])
            else:
                r = s[0] / 2
                areas[p] = 2 * np.pi * r * s[2] + 2 * np.pi * r * r
        share = areas / areas.sum() * n
        counts = np.floor(share).astype(np.int64)
        counts[np.argsort(-(share - counts), kind="stable")[: n - counts.sum()]] += 1
        parts = []
        for p in range(n_prims):
            k, s, c = int(counts[p]), sizes[p], centres[p]
            if k == 0:
                continue
            if kinds[p] == 0:
                parts.append(_sphere(rng, k, c, s[0]))
            elif kinds[p] == 1:
                parts.append(_box(rng, k, c, s))
            else:
                parts.append(_cylinder(rng, k, c, s[0] / 2, s[2]))
        pts = np.concatenate(parts)
        pts = pts + rng.normal(0.0, 0.005, size=pts.shape)
        pts = pts - pts.mean(axis=0)
        pts = pts / np.linalg.norm(pts, axis=1).max()
        out[b] = pts[rng.permutation(n)].astype(np.float32)
    return out


def lidar_sweep(batch: int, seed: int = 0, rings: int = 64, azimuths: int = 512,
                n_boxes: int = 20) -> np.ndarray:
    n = rings * azimuths
    out = np.empty((batch, n, 3), np.float32)
    el = np.deg2rad(np.linspace(-25.0, 3.0, rings))
    az = np.linspace(0.0, 2 * np.pi, azimuths, endpoint=False)
    A, E = np.meshgrid(az, el, indexing="ij")  # azimuth-major storage order
    d = np.stack([np.cos(E) * np.cos(A), np.cos(E) * np.sin(A), np.sin(E)], -1).reshape(n, 3)
    ground = -1.7
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
    for b in range(batch):
        rng = np.random.default_rng(np.random.SeedSequence([seed, b, 4]))
        t = np.where(d[:, 2] < 0, ground / d[:, 2], np.inf)
        rho = rng.uniform(5.0, 45.0, n_boxes)
        phi = rng.uniform(0, 2 * np.pi, n_boxes)
        edges = rng.uniform(1.0, 5.0, size=(n_boxes, 3))
        lo = np.stack([rho * np.cos(phi), rho * np.sin(phi), np.full(n_boxes, ground)], 1)
        lo[:, :2] -= edges[:, :2] / 2
        hi = lo + edges
        for q in range(n_boxes):
            with np.errstate(invalid="ignore"):
                t1 = (lo[q] - 0.0) * inv
                t2 = (hi[q] - 0.0) * inv
            a, c = np.minimum(t1, t2), np.maximum(t1, t2)
            # NaN-ignoring max / min over the three slabs (= nanmax / nanmin)
            tn = np.fmax(np.fmax(a[:, 0], a[:, 1]), a[:, 2])
            tf = np.fmin(np.fmin(c[:, 0], c[:, 1]), c[:, 2])
            hit = (tf >= tn) & (tf > 0)
            t = np.where(hit & (tn > 0), np.minimum(t, tn), t)
        r = np.where(np.isfinite(t), t, 80.0)
        r = np.clip(r, 2.0, 80.0) + rng.normal(0.0, 0.02, size=n)
        out[b] = (d * r[:, None]).astype(np.float32)
    return out


def stable_sort_np(xyz: np.ndarray, axis: int = 0) -> np.ndarray:
    """Host stable sort (test helper): exact_sort semantics on fp32 batches."""
    key = xyz[..., axis].astype(np.float64) + 0.0  # -0.0 -> +0.0
    order = np.argsort(key, axis=-1, kind="stable")
    return np.take_along_axis(xyz, order[..., None], axis=1), order
