"""Benchmark harness with the reference's row schema.

``run_bench`` / ``bench_csv`` mirror ``pcs::run_bench`` / ``pcs::bench_csv``
(proj/src/bench.cpp:34-136): the methods x n x m x k x trials expansion,
per-trial seeds from ``SplitMix64(seed).next()``, one cloud per n from a
provider, ``wall_seconds`` around the sampler call only, quality columns
(coverage_radius, separation — computed by the GPU metric kernels), the
input's locality score, and infeasible rows kept with the error message. Every
non-timing column equals the reference's (tests/test_gpu_parity.py compares
the CSV against the real reference's run_bench). Rows run in order on the GPU;
``threads`` is accepted for parity and ignored (the output is
schedule-independent either way).
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Callable, List

import numpy as np

from . import _core
from .synth import splitmix_next

_SAMPLERS = {"fps", "afps", "npdu-fps", "npdu-afps"}


@dataclass
class BenchOptions:
    methods: List[str]
    n_values: List[int]
    m_values: List[int] = field(default_factory=lambda: [1])
    k_values: List[int] = field(default_factory=lambda: [1])
    c: int = 1
    g: int = 40
    trials: int = 1
    seed: int = 0
    first: str = "random"
    threads: int = 1


@dataclass
class BenchRow:
    method: str
    n: int
    c: int
    m: int
    k: int
    trial: int
    wall_seconds: float = 0.0
    dist_evals: int = 0
    coverage_radius: float = 0.0
    separation: float = 0.0
    locality_score: float = 0.0
    error: str = ""


def locality_score(points: np.ndarray, axis: int = 0) -> float:
    """Adjacent-inversion rate along ``axis`` (proj/src/order.cpp:55-65)."""
    a = points[:, axis]
    if len(a) < 2:
        raise ValueError("locality_score: need at least 2 points")
    return float(np.count_nonzero(a[:-1] > a[1:])) / float(len(a) - 1)


def _run_sampler(method, cloud, c, m, k, seed, first):
    if method == "fps":
        return _core.fps(cloud, c, seed=seed, first=first)
    if method == "afps":
        return _core.afps(cloud, c, m, seed=seed, first=first)
    if method == "npdu-fps":
        return _core.npdu_fps(cloud, c, k, seed=seed, first=first)
    if method == "npdu-afps":
        return _core.npdu_afps(cloud, c, m, k, seed=seed, first=first)
    raise ValueError(f"run_sampler: {method} is not on the GPU sampling path")


def run_bench(options: BenchOptions, provider: Callable[[int], np.ndarray]) -> List[BenchRow]:
    if not options.methods:
        raise ValueError("run_bench: no methods")
    if not options.n_values:
        raise ValueError("run_bench: no input sizes")
    if options.trials < 1:
        raise ValueError("run_bench: trials must be >= 1")
    clouds = [np.ascontiguousarray(provider(n), dtype=np.float64) for n in options.n_values]
    locality = [locality_score(cl, 0) if len(cl) >= 2 else 0.0 for cl in clouds]
    trial_seeds = [int(v) for v in splitmix_next(options.seed, options.trials)]
    rows = []
    for method in options.methods:
        for ni, cloud in enumerate(clouds):
            for m in options.m_values:
                for k in options.k_values:
                    for trial in range(options.trials):
                        row = BenchRow(method, len(cloud), options.c, m, k, trial,
                                       locality_score=locality[ni])
                        try:
                            t0 = time.perf_counter()
                            idx, _, stats = _run_sampler(method, cloud, options.c, m, k,
                                                         trial_seeds[trial], options.first)
                            row.wall_seconds = time.perf_counter() - t0
                            row.dist_evals = int(stats["dist_evals"])
                            row.coverage_radius = _core.coverage_radius(cloud, idx)
                            row.separation = _core.separation(cloud, idx) if len(idx) >= 2 else 0.0
                        except (ValueError, RuntimeError) as exc:
                            row.error = str(exc)
                        rows.append(row)
    return rows


def _g17(v: float) -> str:
    return "%.17g" % v


def bench_csv(rows: List[BenchRow]) -> str:
    out = ["method,n,c,m,k,trial,wall_seconds,dist_evals,coverage_radius,separation,"
           "locality_score,error\n"]
    for r in rows:
        out.append(f"{r.method},{r.n},{r.c},{r.m},{r.k},{r.trial},{_g17(r.wall_seconds)},"
                   f"{r.dist_evals},{_g17(r.coverage_radius)},{_g17(r.separation)},"
                   f"{_g17(r.locality_score)},{r.error}\n")
    return "".join(out)
