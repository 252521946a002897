// Sector-resident farthest point sampling kernels for sm_100a.
//
// Restates pcs::detail::local_fps (proj/src/sampler.cpp:85-167) for a whole
// batch of (cloud, sector) pairs at once, replacing the reference's
// per-sector std::thread pool (sampler.cpp:25-79) with one launch whose
// thread groups each own one sector:
//
//  * a group of W warps (T = 32*W threads) owns one sector; thread t owns
//    points j = s*T + t for slots s < P (interleaved, so loads coalesce and
//    an NPDU window spreads over all lanes);
//  * the sector's xyz is widened once to fp64 and staged in shared memory
//    (SoA); in the full-window kernel it is also held in registers, because
//    F2F.F64.F32 runs at ~1/4 of the DADD rate on B200 (tools/microbench);
//  * min-distances live in registers, in fp64, updated with the reference's
//    `dist <= d[j]` rule and counted for OpStats::dist_writes;
//  * the argmax is one fused pass: per-thread running max on the IEEE bits
//    of d (d >= 0, so bits order like values), then three redux.sync steps
//    (max hi word, max lo word, min index) per warp, then a double-buffered
//    shared-memory exchange with one named barrier per iteration across the
//    group's warps. No global-memory round trip per iteration.
//
// The reference's two-pass argmax (value max over everything, then first
// unsampled index holding it) equals one pass over (max d, min index)
// because every sampled point sits at distance exactly 0: it was a pivot
// inside its own window. When the max itself is 0 (all points coincide with
// samples) a second reduction picks the lowest unsampled index.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <initializer_list>
#include <string>

#include "device_common.cuh"
#include "internal.h"

namespace pcsk {

struct SampleParams {
  const void* xyz;
  // optional (B, N) sort permutation: sorted position -> storage index. When
  // set, the clouds are sampled in that order (sector point j of cloud b is
  // xyz[b, perm[b, begin + j]]): exact_sort's gather (proj/src/order.cpp:
  // 19-21) fused into the sampler's staging, so the sort writes only the
  // permutation and nobody writes / re-reads a sorted copy of the cloud.
  const int* perm;
  int f64;
  long long B, N, C, M, K;  // K == 0: full window
  int random_first;
  uint64_t seed;
  const uint64_t* seeds;
  void* out_idx;
  int idx64;
  long long index_base;   // added to every output index (ranges, shards)
  long long sector_base;  // added to sector ids (seed stream, sector_of)
  int* out_sector;
  unsigned long long* stats;
  double* trace;
  int nmax;  // smem capacity per group, points
  int G;     // sector groups per CTA
};

constexpr uint32_t kInfHi = 0x7ff00000u;

__device__ __forceinline__ void write_index(const SampleParams& p, long long b, int slot,
                                            long long v) {
  v += p.index_base;
  if (p.idx64)
    static_cast<long long*>(p.out_idx)[b * p.C + slot] = v;
  else
    static_cast<int*>(p.out_idx)[b * p.C + slot] = static_cast<int>(v);
}

// Global AoS (f32 or f64) -> shared SoA (CT). Widening f32 -> f64 is exact;
// CT = float is only ever used with f32 input.
template <typename Tin, typename CT>
__device__ __forceinline__ void stage_sector(const Tin* __restrict__ src, int n, CT* xs, CT* ys,
                                             CT* zs, int t, int nthreads) {
  auto put = [&](int e, Tin v) {
    const int q = e / 3, a = e - 3 * q;
    (a == 0 ? xs : (a == 1 ? ys : zs))[q] = static_cast<CT>(v);
  };
  int e0 = 0;
  if constexpr (sizeof(Tin) == 4) {
    // 16-byte loads, four in flight per thread: a sector is a few KB of
    // contiguous AoS, staging is load-latency bound otherwise
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
      const float4* s4 = reinterpret_cast<const float4*>(src);
      const int n4 = (3 * n) >> 2;
      int i = t;
      for (; i + 3 * nthreads < n4; i += 4 * nthreads) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldg(s4 + i + u * nthreads);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = 4 * (i + u * nthreads);
          put(e, v[u].x); put(e + 1, v[u].y); put(e + 2, v[u].z); put(e + 3, v[u].w);
        }
      }
      for (; i < n4; i += nthreads) {
        const float4 v = __ldg(s4 + i);
        const int e = 4 * i;
        put(e, v.x); put(e + 1, v.y); put(e + 2, v.z); put(e + 3, v.w);
      }
      e0 = 4 * n4;
    }
  }
  for (int e = e0 + t; e < 3 * n; e += nthreads) put(e, src[e]);
}

// Staging through the sort permutation: point j of the sector is storage
// point perm_sector[j] of `cloud` (the cloud's first point).
template <typename Tin, typename CT>
__device__ __forceinline__ void stage_sector_perm(const Tin* __restrict__ cloud,
                                                  const int* __restrict__ perm_sector, int n,
                                                  CT* xs, CT* ys, CT* zs, int t, int nthreads) {
  // four points in flight per thread: the permutation loads, then the
  // twelve coordinate loads (L2 gathers), then the stores
  int j = t;
  for (; j + 3 * nthreads < n; j += 4 * nthreads) {
    int i[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) i[u] = __ldg(perm_sector + j + u * nthreads);
    Tin v[4][3];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const Tin* q = cloud + 3LL * i[u];
      v[u][0] = __ldg(q);
      v[u][1] = __ldg(q + 1);
      v[u][2] = __ldg(q + 2);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int jj = j + u * nthreads;
      xs[jj] = static_cast<CT>(v[u][0]);
      ys[jj] = static_cast<CT>(v[u][1]);
      zs[jj] = static_cast<CT>(v[u][2]);
    }
  }
  for (; j < n; j += nthreads) {
    const Tin* q = cloud + 3LL * __ldg(perm_sector + j);
    const Tin x = __ldg(q), y = __ldg(q + 1), z = __ldg(q + 2);
    xs[j] = static_cast<CT>(x);
    ys[j] = static_cast<CT>(y);
    zs[j] = static_cast<CT>(z);
  }
}

// Stage a sector [begin, begin + n) of cloud b into shared SoA, in storage
// order or through p.perm.
template <typename Tin, typename CT>
__device__ __forceinline__ void stage_sector_of(const SampleParams& p, long long b,
                                                long long begin, int n, CT* xs, CT* ys, CT* zs,
                                                int t, int nthreads) {
  const Tin* cloud = static_cast<const Tin*>(p.xyz) + b * p.N * 3;
  if (p.perm)
    stage_sector_perm(cloud, p.perm + b * p.N + begin, n, xs, ys, zs, t, nthreads);
  else
    stage_sector(cloud + begin * 3, n, xs, ys, zs, t, nthreads);
}

template <int W>
__device__ __forceinline__ void group_sync(int gid) {
  if constexpr (W > 1)
    named_bar_sync(1 + gid, W * 32);
  else
    __syncwarp();
}

// Group-wide (max d, min index) across the W warps of a sector group.
template <int W>
__device__ __forceinline__ void group_argmax(uint32_t& hi, uint32_t& lo, uint32_t& j,
                                             uint4* cand, int& round, int gid, int lane,
                                             int warp) {
  warp_argmax(hi, lo, j);
  if constexpr (W > 1) {
    uint4* buf = cand + (round & 1) * W;
    if (lane == 0) buf[warp] = make_uint4(hi, lo, j, 0);
    named_bar_sync(1 + gid, W * 32);
    const uint4 v = lane < W ? buf[lane] : make_uint4(0, 0, kNoIndex, 0);
    hi = v.x;
    lo = v.y;
    j = v.z;
    warp_argmax(hi, lo, j);
  }
  ++round;
}

struct GroupSetup {
  long long b, s;
  SectorGeom g;
  double *xs, *ys, *zs;
  uint4* cand;
};

template <int W>
__device__ __forceinline__ bool setup_group(const SampleParams& p, unsigned char* smem, int gid,
                                            int t, GroupSetup& gs) {
  const long long flat = static_cast<long long>(blockIdx.x) * p.G + gid;
  if (flat >= p.B * p.M) return false;
  gs.b = flat / p.M;
  gs.s = flat % p.M;
  gs.g = sector_geom(p.N, p.C, p.M, gs.s);
  const size_t group_bytes = size_t(24) * p.nmax + 32 * W;
  unsigned char* base = smem + gid * group_bytes;
  gs.xs = reinterpret_cast<double*>(base);
  gs.ys = gs.xs + p.nmax;
  gs.zs = gs.ys + p.nmax;
  gs.cand = reinterpret_cast<uint4*>(base + size_t(24) * p.nmax);
  if (p.f64)
    stage_sector_of<double>(p, gs.b, gs.g.begin, gs.g.n, gs.xs, gs.ys, gs.zs, t, W * 32);
  else
    stage_sector_of<float>(p, gs.b, gs.g.begin, gs.g.n, gs.xs, gs.ys, gs.zs, t, W * 32);
  if (p.out_sector)
    for (int i = t; i < gs.g.quota; i += W * 32)
      p.out_sector[gs.b * p.C + gs.g.out_off + i] = static_cast<int>(gs.s + p.sector_base);
  return true;
}

__device__ __forceinline__ int first_point(const SampleParams& p, const GroupSetup& gs) {
  if (!p.random_first) return 0;
  const uint64_t seed =
      (p.seeds ? p.seeds[gs.b] : p.seed) ^ static_cast<uint64_t>(gs.s + p.sector_base);
  return static_cast<int>(splitmix_below(seed, static_cast<uint64_t>(gs.g.n)));
}

template <int W>
__device__ __forceinline__ void flush_stats(const SampleParams& p, const GroupSetup& gs, int t,
                                            unsigned writes, unsigned long long evals) {
  const unsigned ws = __reduce_add_sync(kFull, writes);
  if (p.stats == nullptr) return;
  unsigned long long* st = p.stats + gs.b * 4;
  if ((t & 31) == 0 && ws) atomicAdd(st + 1, static_cast<unsigned long long>(ws));
  if (t == 0) {
    const unsigned long long iters = static_cast<unsigned long long>(gs.g.quota - 1);
    atomicAdd(st + 0, evals);
    atomicAdd(st + 2, iters * static_cast<unsigned long long>(gs.g.n));
    atomicAdd(st + 3, iters);
  }
}

// Lowest unsampled index of the group (the reference's index pass when every
// remaining distance is 0, sampler.cpp:148-154).
template <int P, int W>
__device__ __forceinline__ uint32_t lowest_unsampled(unsigned vmask, unsigned smask, int t,
                                                     uint4* cand, int& round, int gid, int lane,
                                                     int warp) {
  uint32_t jm = kNoIndex;
#pragma unroll
  for (int k = P - 1; k >= 0; --k)
    if (((vmask & ~smask) >> k) & 1u) jm = static_cast<uint32_t>(k * W * 32 + t);
  uint32_t hi = jm != kNoIndex ? 1u : 0u, lo = 0, j = jm;
  group_argmax<W>(hi, lo, j, cand, round, gid, lane, warp);
  return j;
}

constexpr size_t kMaxSmem = 227 * 1024;
// windowed batches of at most this many sectors (one per SM) take
// npdu_wide_kernel: cfg4 sectors (1024 points, k=129) at 32-128 sectors
// 0.117 vs 0.142 ms; at 256 sectors the one-warp TMEM kernel wins again
// (0.141 vs 0.152 ms) and at 512 by 2x (tools/npdu_wide_ab.py)
constexpr long long kNpduWideMax = 148;

// Plan mode (pcs_kernel_family): while set, the launchers store the name of
// the kernel they would launch here and return cudaSuccess without touching
// the device. The check sits right before each launch, after every fit
// test, so the plan is the dispatch decision itself.
extern thread_local std::string* g_plan;
std::string kname(const char* base, std::initializer_list<long long> args);
inline bool plan(const char* base, std::initializer_list<long long> args) {
  if (!g_plan) return false;
  *g_plan = kname(base, args);
  return true;
}

// Launchers (one per translation unit). They return cudaErrorNotSupported
// when the sector does not fit the kernel family.
cudaError_t run_full_any(SampleParams p, long long nmax_sector, cudaStream_t st);
cudaError_t run_npdu_any(SampleParams p, long long nmax_sector, cudaStream_t st);
cudaError_t run_npdu_wide_any(SampleParams p, long long nmax_sector, cudaStream_t st);
cudaError_t run_rows_any(SampleParams p, long long nmax_sector, bool windowed, cudaStream_t st);
cudaError_t run_morton_any(SampleParams p, long long nmax_sector, cudaStream_t st);
cudaError_t run_morton_tmem_any(SampleParams p, long long nmax_sector, cudaStream_t st);
cudaError_t run_stream_any(SampleParams p, long long nmax_sector, cudaStream_t st);
cudaError_t run_cluster_any(SampleParams p, long long nmax_sector, cudaStream_t st);
cudaError_t run_tiny_any(SampleParams p, long long nmax_sector, cudaStream_t st);
// a thread per sector (fps_tiny_kernel) from this many sectors on
constexpr long long kTinyMinSectors = 2048;

}  // namespace pcsk
