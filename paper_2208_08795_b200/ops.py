"""Batched torch-facing sampling op over the C-ABI (include/pcs_gpu.h).

The reference samples one cloud per call (proj/include/pcs/sampler.hpp:41-66);
PointNet++-style callers sample a whole batch per set-abstraction layer. This
module is that batched entry: CUDA tensors in, CUDA tensors out, enqueued on
the current torch stream, no host synchronisation, so it can sit inside a
CUDA graph. Torch is plumbing here (device memory, streams); every FLOP runs
in the sm_100a kernels of libpcs_gpu.so.
"""
from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import _core

METHODS = {"fps": 1, "afps": 2, "npdu_fps": 3, "npdu_afps": 4}
_AXES = {"x": 0, "y": 1, "z": 2, 0: 0, 1: 1, 2: 2}


def _stream_handle(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _as_batch(xyz: torch.Tensor) -> torch.Tensor:
    if xyz.dim() == 2:
        xyz = xyz.unsqueeze(0)
    if xyz.dim() != 3 or xyz.shape[-1] != 3:
        raise ValueError("expected an (N, 3) or (B, N, 3) tensor")
    if not xyz.is_cuda:
        raise ValueError("xyz must be a CUDA tensor (use sample_host_batch for host arrays)")
    if xyz.dtype not in (torch.float32, torch.float64):
        raise ValueError("xyz must be float32 or float64")
    return xyz.contiguous()


def sort_axis(xyz: torch.Tensor, axis="x"):
    """Stable per-cloud sort along ``axis`` (pcs::exact_sort semantics,
    proj/src/order.cpp:11-24). Returns ``(sorted_xyz, perm int32)`` with
    ``sorted_xyz[b, i] == xyz[b, perm[b, i]]``."""
    if axis not in _AXES:
        raise ValueError("axis must be x, y, or z")
    x = _as_batch(xyz)
    B, N = x.shape[0], x.shape[1]
    out = torch.empty_like(x)
    perm = torch.empty((B, N), dtype=torch.int32, device=x.device)
    _core.sort_device(1 if x.dtype == torch.float64 else 0, x.data_ptr(), B, N, _AXES[axis],
                      out.data_ptr(), perm.data_ptr(), _stream_handle(x.device))
    return out, perm


def sort_perm(xyz: torch.Tensor, axis="x") -> torch.Tensor:
    """The permutation of :func:`sort_axis` alone (int32 (B, N)), without the
    gathered copy -- what :func:`sample` passes to the sampler."""
    if axis not in _AXES:
        raise ValueError("axis must be x, y, or z")
    x = _as_batch(xyz)
    B, N = x.shape[0], x.shape[1]
    perm = torch.empty((B, N), dtype=torch.int32, device=x.device)
    _core.sort_device(1 if x.dtype == torch.float64 else 0, x.data_ptr(), B, N, _AXES[axis],
                      0, perm.data_ptr(), _stream_handle(x.device))
    return perm


def sample_with_perm(xyz: torch.Tensor, perm: torch.Tensor, c: int, **kw):
    """:func:`sample` of the clouds in the order of ``perm`` (int32 (B, N),
    sorted position -> storage index, e.g. from :func:`sort_perm`): the
    results of sampling the gathered copy, without the copy."""
    return sample(xyz, c, _perm=perm, **kw)


def sample(xyz: torch.Tensor, c: int, method: str = "afps", m: int = 1, k: Optional[int] = None,
           first: str = "fixed", seed: int = 0, seeds: Optional[torch.Tensor] = None,
           sort: Optional[str] = None, index_dtype: torch.dtype = torch.int32,
           return_sector: bool = False, index_base: int = 0, sector_base: int = 0,
           _perm: Optional[torch.Tensor] = None):
    """Sample ``c`` points from every cloud of ``xyz`` (``(B, N, 3)``).

    CUDA input: stream-ordered on the current stream, results on the device,
    no synchronisation (CUDA-graph capturable). CPU input (pinned or not):
    pipelined H2D / compute / D2H, results returned as CPU tensors.

    ``method`` is one of fps / afps / npdu_fps / npdu_afps; ``m`` sectors for
    the AFPS variants, ``k`` window for the NPDU variants (the reference's
    ``k``; BASELINE's "w neighbours each side" is ``k = 2w + 1``). ``first``
    is "fixed" (FixedFirstPoint) or "random" (SplitMix64(seed ^ sector)).
    ``sort``: optional axis; clouds are first stably sorted (exact_sort) and
    the indices then refer to the sorted clouds, exactly as
    ``afps(exact_sort(cloud), ...)`` does in the reference.

    Returns ``(indices (B, c), stats int64 (B, 4))`` plus ``sector_of``
    (int32) when ``return_sector`` and ``perm`` (int32) when ``sort``.
    Stats columns: dist_evals, dist_writes, argmax_scans, iterations.
    ``index_base`` / ``sector_base`` shift output indices / sector ids when
    the batch is a shard (a storage slice) of a larger cloud.
    """
    if method not in METHODS:
        raise ValueError(f"unknown method {method!r}")
    if first not in ("fixed", "random"):
        raise ValueError("first must be 'random' or 'fixed'")
    if isinstance(xyz, torch.Tensor) and not xyz.is_cuda:
        # host tensor: the C-ABI host batch entry (pipelined H2D / sort +
        # sample / D2H in one native call); results come back on the host
        if index_dtype not in (torch.int32, torch.int64):
            raise ValueError("index_dtype must be torch.int32 or torch.int64")
        res = sample_host_batch(xyz, c, method=method, m=m, k=k, first=first, seed=seed,
                                seeds=seeds, sort=sort,
                                index_dtype=np.int64 if index_dtype == torch.int64 else np.int32,
                                return_sector=return_sector, index_base=index_base,
                                sector_base=sector_base)
        return tuple(torch.from_numpy(r) for r in res)
    x = _as_batch(xyz)
    perm = None
    if _perm is not None:
        if sort is not None:
            raise ValueError("sort and a permutation are exclusive")
        perm = _perm.to(device=x.device, dtype=torch.int32).contiguous()
        if tuple(perm.shape) != (x.shape[0], x.shape[1]):
            raise ValueError("perm must be (B, N)")
    if sort is not None:
        # the sort writes only the permutation; the sampler stages every
        # sector through it (no sorted copy of the clouds is made)
        perm = sort_perm(x, sort)
    B, N = x.shape[0], x.shape[1]
    dev = x.device
    if index_dtype not in (torch.int32, torch.int64):
        raise ValueError("index_dtype must be torch.int32 or torch.int64")
    idx = torch.empty((B, max(int(c), 0)), dtype=index_dtype, device=dev)
    stats = torch.empty((B, 4), dtype=torch.int64, device=dev)
    sector = torch.empty((B, max(int(c), 0)), dtype=torch.int32, device=dev) if return_sector else None
    seeds_ptr = 0
    if seeds is not None:
        seeds = seeds.to(device=dev, dtype=torch.int64).contiguous()
        if seeds.numel() != B:
            raise ValueError("seeds must hold one seed per cloud")
        seeds_ptr = seeds.data_ptr()
    _core.sample_device(METHODS[method], 1 if x.dtype == torch.float64 else 0, x.data_ptr(), B, N,
                        int(c), int(m), int(k) if k is not None else 0,
                        1 if first == "fixed" else 0, int(seed) & (2**64 - 1), seeds_ptr,
                        1 if index_dtype == torch.int64 else 0, idx.data_ptr(),
                        sector.data_ptr() if sector is not None else 0, stats.data_ptr(),
                        _stream_handle(dev), int(index_base), int(sector_base),
                        perm.data_ptr() if perm is not None else 0)
    out = [idx, stats]
    if return_sector:
        out.append(sector)
    if perm is not None and _perm is None:
        out.append(perm)
    return tuple(out)


def quality(xyz: torch.Tensor, idx: torch.Tensor):
    """Batched coverage_radius and separation (the reference's metrics,
    proj/src/metrics.cpp:16-52, bit-identical) of samples ``idx`` (B, c) in
    clouds ``xyz`` (B, N, 3), on the device. Returns two float64 (B,) tensors
    (NaN where an index is out of range; separation needs c >= 2)."""
    x = _as_batch(xyz)
    ix = idx.unsqueeze(0) if idx.dim() == 1 else idx
    ix = ix.to(device=x.device).contiguous()
    if ix.dtype not in (torch.int32, torch.int64):
        ix = ix.to(torch.int64)
    B, N, c = x.shape[0], x.shape[1], ix.shape[1]
    cov = torch.empty(B, dtype=torch.float64, device=x.device)
    sep = torch.full((B,), float("nan"), dtype=torch.float64, device=x.device)
    st = _stream_handle(x.device)
    cd, idt = (1 if x.dtype == torch.float64 else 0), (1 if ix.dtype == torch.int64 else 0)
    _core.metric_device(0, cd, x.data_ptr(), B, N, idt, ix.data_ptr(), c, cov.data_ptr(), st)
    if c >= 2:
        _core.metric_device(1, cd, x.data_ptr(), B, N, idt, ix.data_ptr(), c, sep.data_ptr(), st)
    return cov, sep


def kernel_family(method: str, n: int, m: int = 1, k: Optional[int] = None,
                  dtype: str = "float32", batch: int = 1, c: Optional[int] = None,
                  full: bool = False) -> str:
    """The sm_100a kernel :func:`sample` launches for this call shape -- the
    C++ dispatcher's own decision (``pcs_kernel_family``, csrc/sample_dispatch.cu
    run in plan mode; no device work). ``full`` keeps the template arguments,
    e.g. ``npdu_tmem_kernel<5,1024>``."""
    if method not in METHODS:
        raise ValueError(f"unknown method {method!r}")
    name = _core.kernel_family(METHODS[method], 1 if dtype == "float64" else 0, int(batch),
                               int(n), int(c if c is not None else n), int(m),
                               int(k) if k is not None else 0)
    return name if full else name.split("<", 1)[0]


def reload_knobs() -> None:
    """Re-read the PCS_* engine overrides (tests; they are read once per
    process otherwise)."""
    _core.reload_knobs()


def sample_host_batch(xyz, c: int, method: str = "afps", m: int = 1,
                      k: Optional[int] = None, first: str = "fixed", seed: int = 0,
                      sort: Optional[str] = None, device: Optional[str] = None,
                      index_dtype=np.int32, return_sector: bool = False, chunks: int = 0,
                      seeds=None, index_base: int = 0, sector_base: int = 0,
                      devices=None):
    """Host batch in, host results out, through the C-ABI host entry
    ``pcs_sample_host_batch`` (include/pcs_gpu.h): the per-cloud samplers
    over a batch in one native, pipelined call (H2D of a chunk overlaps the
    sort + sampling of the previous one). ``xyz``: (B, N, 3) float32/float64
    numpy array or CPU torch tensor (pin it -- ``tensor.pin_memory()`` -- for
    copy/compute overlap). Returns numpy ``(indices (B, c), stats (B, 4))``
    plus ``sector_of`` when ``return_sector`` and ``perm`` when ``sort``.

    ``devices`` (a list of CUDA ordinals, e.g. ``range(8)``) spreads the
    call over several GPUs from this one process (``pcs_sample_host_multi``):
    clouds split by cloud, or one AFPS / NPDU-AFPS cloud by sector run;
    results identical to the one-device call."""
    if method not in METHODS:
        raise ValueError(f"unknown method {method!r}")
    if first not in ("fixed", "random"):
        raise ValueError("first must be 'random' or 'fixed'")
    x = xyz if isinstance(xyz, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(xyz))
    if x.is_cuda:
        raise ValueError("sample_host_batch takes host memory; use sample() for CUDA tensors")
    x = x.unsqueeze(0) if x.dim() == 2 else x
    if x.dim() != 3 or x.shape[-1] != 3 or x.dtype not in (torch.float32, torch.float64):
        raise ValueError("expected a float32/float64 (B, N, 3) array")
    x = x.contiguous()
    B, N = x.shape[0], x.shape[1]
    idx64 = np.dtype(index_dtype) == np.int64
    pin = x.is_pinned()
    idx = torch.empty((B, max(int(c), 0)), dtype=torch.int64 if idx64 else torch.int32,
                      pin_memory=pin)
    stats = torch.empty((B, 4), dtype=torch.int64, pin_memory=pin)
    sec = torch.empty((B, max(int(c), 0)), dtype=torch.int32, pin_memory=pin) if return_sector else None
    perm = torch.empty((B, N), dtype=torch.int32, pin_memory=pin) if sort else None
    if sort is not None and sort not in _AXES:
        raise ValueError("axis must be x, y, or z")
    sd = None
    if seeds is not None:
        sd = torch.as_tensor(seeds).to(device="cpu", dtype=torch.int64).contiguous()
        if sd.numel() != B:
            raise ValueError("seeds must hold one seed per cloud")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    devs = [int(d.index if isinstance(d, torch.device) else d) for d in devices] if devices else []
    with torch.cuda.device(dev):
        _core.sample_host_ptr(METHODS[method], 1 if x.dtype == torch.float64 else 0,
                              x.data_ptr(), B, N, int(c), int(m), int(k) if k is not None else 0,
                              1 if first == "fixed" else 0, int(seed) & (2**64 - 1),
                              sd.data_ptr() if sd is not None else 0,
                              1 if idx64 else 0, idx.data_ptr(),
                              sec.data_ptr() if sec is not None else 0, stats.data_ptr(),
                              _AXES[sort] if sort is not None else -1,
                              perm.data_ptr() if perm is not None else 0, int(chunks),
                              int(index_base), int(sector_base), devs)
    out = [idx.numpy(), stats.numpy()]
    if return_sector:
        out.append(sec.numpy())
    if perm is not None:
        out.append(perm.numpy())
    return tuple(out)
