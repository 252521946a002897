"""Multi-GPU driver: one process per GPU, independent work split across ranks.

The sampling path shards with no data-path collective:

* a batch of clouds splits by cloud -- clouds are independent
  (proj/src/sampler.cpp keeps no cross-cloud state);
* one large cloud under AFPS / NPDU-AFPS splits by sector -- sectors are
  independent after the sort (sampler.cpp:48-79): rank r takes a contiguous
  run of sectors, i.e. a contiguous storage slice, and samples it with
  ``index_base`` / ``sector_base`` offsets so its indices, sector ids and
  per-sector seeds (seed ^ sector) are the global ones.

Results meet once, at the end (``gather_rows``). A contiguous run of the
reference's remainder-rule sectors, re-partitioned on its own, reproduces
exactly the same sector boundaries and quotas (the first ``total % m`` get
one extra), which is what makes the sector split exact.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def split(total: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of rank's share; the first total % world ranks get one more
    (the reference's partition_sectors rule, proj/src/sectors.cpp:9-24)."""
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


@dataclass
class SectorShard:
    sector_lo: int  # first global sector
    sector_hi: int
    point_lo: int   # storage slice [point_lo, point_hi)
    point_hi: int
    out_lo: int     # output slots [out_lo, out_hi) of the global index row
    out_hi: int

    @property
    def m(self):
        return self.sector_hi - self.sector_lo

    @property
    def n(self):
        return self.point_hi - self.point_lo

    @property
    def c(self):
        return self.out_hi - self.out_lo

    @property
    def empty(self):
        """More ranks than sectors: this rank has no sector to sample."""
        return self.m == 0


def _start(total: int, parts: int, s: int) -> int:
    base, rem = divmod(total, parts)
    return s * base + min(s, rem)


def sector_shard(n: int, c: int, m: int, world: int, rank: int) -> SectorShard:
    s0, s1 = split(m, world, rank)
    return SectorShard(s0, s1, _start(n, m, s0), _start(n, m, s1), _start(c, m, s0),
                       _start(c, m, s1))


def sample_sector_shard(sorted_xyz: torch.Tensor, sh: SectorShard, method: str, k=None,
                        first: str = "fixed", seed: int = 0):
    """Sample rank's run of sectors of the (already sorted) cloud(s)
    ``sorted_xyz`` (B, N, 3) on the device: global indices, sector ids and
    per-sector seeds. An empty shard (world > m) yields (B, 0) results, so
    it still takes part in ``gather_rows``. Returns (indices int32,
    stats int64 (B, 4), sector_of int32)."""
    from . import sample

    B = sorted_xyz.shape[0]
    if sh.empty:
        dev = sorted_xyz.device
        return (torch.zeros((B, 0), dtype=torch.int32, device=dev),
                torch.zeros((B, 4), dtype=torch.int64, device=dev),
                torch.zeros((B, 0), dtype=torch.int32, device=dev))
    return sample(sorted_xyz[:, sh.point_lo:sh.point_hi], sh.c, method=method, m=sh.m, k=k,
                  first=first, seed=seed, return_sector=True, index_base=sh.point_lo,
                  sector_base=sh.sector_lo)


def gather_rows(local: torch.Tensor, total_rows: int, world: int, group=None) -> torch.Tensor | None:
    """Concatenate every rank's rows (rank order) on rank 0; None elsewhere.
    One all_gather of padded shards -- the only collective, after sampling."""
    if world == 1:
        return local
    rows = torch.tensor([local.shape[0]], device=local.device)
    counts = [torch.zeros_like(rows) for _ in range(world)]
    dist.all_gather(counts, rows, group=group)
    pad = max(int(x.item()) for x in counts)
    buf = torch.zeros((pad,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    if dist.get_rank(group) != 0:
        return None
    out = torch.cat([p[: int(k.item())] for p, k in zip(parts, counts)])
    assert out.shape[0] == total_rows
    return out
