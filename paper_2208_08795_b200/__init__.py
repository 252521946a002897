"""B200-native point-cloud sampling: FPS, AFPS and NPDU-AFPS (arXiv 2208.08795).

Two faces over the same sm_100a kernels (C-ABI: include/pcs_gpu.h):

* the reference's Python API, ``pcsample._core`` compatible
  (proj/bindings/pcsample_module.cpp:122-190): ``fps``, ``afps``,
  ``npdu_fps``, ``npdu_afps``, ``exact_sort`` (and ``local_fps`` with the
  DistanceTrace) taking float64 ``(N, 3)`` arrays and returning
  ``(int64 idx, int64 sector_of, stats dict)``;
* a batched, stream-ordered torch op, :func:`sample` / :func:`sort_axis`,
  taking CUDA tensors ``(B, N, 3)`` and returning ``int32 (B, C)`` indices plus
  ``(B, 4)`` OpStats, capturable in CUDA graphs.

There is no CPU fallback: importing without the built extension raises.
"""
from __future__ import annotations

import os as _os

_PKG = _os.path.dirname(_os.path.abspath(__file__))

try:
    from . import _core  # noqa: F401  (loads lib/libpcs_gpu.so)
except ImportError as exc:  # pragma: no cover - exercised only when unbuilt
    raise ImportError(
        "paper_2208_08795_b200: native extension not built "
        "(run `python paper_2208_08795_b200/_build.py`); there is no CPU fallback"
    ) from exc

from ._core import (afps, coverage_radius, exact_sort, fps, local_fps, npdu_afps,  # noqa: E402
                    npdu_fps, read_cloud, separation, write_cloud)
from .ops import (METHODS, kernel_family, quality, reload_knobs, sample,  # noqa: E402
                  sample_host_batch, sort_axis, sort_perm)

LIB_PATH = _os.path.join(_PKG, "lib", "libpcs_gpu.so")

__all__ = [
    "fps", "afps", "npdu_fps", "npdu_afps", "exact_sort", "local_fps", "coverage_radius",
    "separation", "quality", "read_cloud", "write_cloud",
    "sample", "sort_axis", "sort_perm", "sample_host_batch", "kernel_family", "reload_knobs", "METHODS",
    "LIB_PATH",
]
