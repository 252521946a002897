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
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>

#include "device_common.cuh"
#include "internal.h"

namespace pcsk {

struct SampleParams {
  const void* xyz;
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

template <typename Tin>
__device__ __forceinline__ void stage_sector(const Tin* __restrict__ src, int n, double* xs,
                                             double* ys, double* zs, int t, int nthreads) {
  for (int e = t; e < 3 * n; e += nthreads) {
    const double v = static_cast<double>(src[e]);
    const int q = e / 3, a = e - 3 * q;
    (a == 0 ? xs : (a == 1 ? ys : zs))[q] = v;
  }
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
  const long long off = (gs.b * p.N + gs.g.begin) * 3;
  if (p.f64)
    stage_sector(static_cast<const double*>(p.xyz) + off, gs.g.n, gs.xs, gs.ys, gs.zs, t, W * 32);
  else
    stage_sector(static_cast<const float*>(p.xyz) + off, gs.g.n, gs.xs, gs.ys, gs.zs, t, W * 32);
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

// ---------------------------------------------------------------- full window
// FPS / AFPS: every iteration updates the whole sector (sampler.cpp:115-129
// with window == sector). REGC: sector xyz also cached in registers.
template <int P, int W, bool REGC>
__global__ void __launch_bounds__(W * 32 * (W >= 8 ? 1 : (8 / W)))
    fps_full_kernel(const SampleParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int T = W * 32;
  const int gid = threadIdx.x / T, t = threadIdx.x % T, lane = t & 31, warp = t >> 5;
  GroupSetup gs;
  if (!setup_group<W>(p, smem, gid, t, gs)) return;
  const int n = gs.g.n;
  group_sync<W>(gid);

  double x[REGC ? P : 1], y[REGC ? P : 1], z[REGC ? P : 1], d[P];
  unsigned vmask = 0;
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const int j = k * T + t;
    const bool valid = j < n;
    vmask |= valid ? (1u << k) : 0u;
    if constexpr (REGC) {
      x[k] = valid ? gs.xs[j] : 0.0;
      y[k] = valid ? gs.ys[j] : 0.0;
      z[k] = valid ? gs.zs[j] : 0.0;
    }
    d[k] = valid ? __longlong_as_double(0x7ff0000000000000LL) : 0.0;
  }

  int cur = first_point(p, gs);
  if (t == 0) write_index(p, gs.b, gs.g.out_off, gs.g.begin + cur);
  unsigned smask = (cur % T == t) ? (1u << (cur / T)) : 0u;
  unsigned writes = 0;
  int round = 0;

  for (int it = 1; it < gs.g.quota; ++it) {
    const double px = gs.xs[cur], py = gs.ys[cur], pz = gs.zs[cur];
    unsigned long long best = 0;
    int bs = -1;
    // Branch-free over the slots so independent slots interleave (ILP).
    // Padding slots (j >= n) hold d = 0 and finite coordinates: they never
    // win the argmax (best starts at 0 with a strict >) and their writes are
    // masked out of the count.
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const int j = k * T + t;
      const double xx = REGC ? x[REGC ? k : 0] : gs.xs[min(j, n - 1)];
      const double yy = REGC ? y[REGC ? k : 0] : gs.ys[min(j, n - 1)];
      const double zz = REGC ? z[REGC ? k : 0] : gs.zs[min(j, n - 1)];
      const double dist = dist2(xx, yy, zz, px, py, pz);
      const bool lower = dist <= d[k];
      writes += (lower && ((vmask >> k) & 1u)) ? 1u : 0u;
      d[k] = lower ? dist : d[k];
      const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(d[k]));
      if (bits > best) {
        best = bits;
        bs = k;
      }
    }
    if (p.trace) {
#pragma unroll
      for (int k = 0; k < P; ++k)
        if ((vmask >> k) & 1u) p.trace[static_cast<long long>(it - 1) * n + k * T + t] = d[k];
    }
    uint32_t hi = static_cast<uint32_t>(best >> 32), lo = static_cast<uint32_t>(best);
    uint32_t j = bs >= 0 ? static_cast<uint32_t>(bs * T + t) : kNoIndex;
    group_argmax<W>(hi, lo, j, gs.cand, round, gid, lane, warp);
    if ((hi | lo) == 0u)
      j = lowest_unsampled<P, W>(vmask, smask, t, gs.cand, round, gid, lane, warp);
    cur = static_cast<int>(j);
    if (t == 0) write_index(p, gs.b, gs.g.out_off + it, gs.g.begin + cur);
    if (cur % T == t) smask |= 1u << (cur / T);
  }
  const unsigned long long evals =
      static_cast<unsigned long long>(gs.g.quota - 1) * static_cast<unsigned long long>(n);
  flush_stats<W>(p, gs, t, writes, evals);
}

// ---------------------------------------------------------------- NPDU window
// NPDU-FPS / NPDU-AFPS: the update touches only update_window(sector, idx, k)
// (proj/src/sectors.cpp:53-61). One warp owns one sector; xyz (fp64) and the
// min-distances d[] live in shared memory, so the rows of 32 points that a
// window touches can be addressed with a runtime row index. The argmax still
// ranges over the whole sector (as the reference's does), but
// incrementally: each row's (max d, min index) is cached in registers --
// lane l holds rows l, l+32, ... -- and only rows the window touched are
// re-reduced (3 redux each). d only decreases, so untouched rows keep valid
// maxima, and the per-iteration cost is O(k/32 + rows/32) instead of O(n).
// Shared memory per NPDU warp: xyz + d (fp64) and the sampled bitmap,
// rounded to 16 B so every warp's doubles stay aligned.
__host__ __device__ __forceinline__ size_t npdu_warp_bytes(int nmax) {
  return (size_t(32) * nmax + 4 * (nmax / 32 + 1) + 15) & ~size_t(15);
}

template <int RPL>
__global__ void __launch_bounds__(128) npdu_warp_kernel(const SampleParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int gid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long flat = static_cast<long long>(blockIdx.x) * p.G + gid;
  if (flat >= p.B * p.M) return;
  const long long b = flat / p.M, s = flat % p.M;
  const SectorGeom g = sector_geom(p.N, p.C, p.M, s);
  const int n = g.n, nmax = p.nmax;
  unsigned char* base = smem + static_cast<size_t>(gid) * npdu_warp_bytes(nmax);
  double* xs = reinterpret_cast<double*>(base);
  double* ys = xs + nmax;
  double* zs = ys + nmax;
  double* d = zs + nmax;
  unsigned* sampled = reinterpret_cast<unsigned*>(d + nmax);
  const long long off = (b * p.N + g.begin) * 3;
  if (p.f64)
    stage_sector(static_cast<const double*>(p.xyz) + off, n, xs, ys, zs, lane, 32);
  else
    stage_sector(static_cast<const float*>(p.xyz) + off, n, xs, ys, zs, lane, 32);
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  for (int j = lane; j < n; j += 32) d[j] = kInf;
  const int rows = (n + 31) >> 5;
  for (int w = lane; w < rows; w += 32) sampled[w] = 0u;
  if (p.out_sector)
    for (int i = lane; i < g.quota; i += 32)
      p.out_sector[b * p.C + g.out_off + i] = static_cast<int>(s + p.sector_base);
  // row maxima: lane l caches row r = l + 32*i in slot i; initially every
  // point is +inf, so a row's winner is its first point
  uint32_t rm_hi[RPL], rm_lo[RPL], rm_j[RPL];
#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    const int r = lane + 32 * i;
    rm_hi[i] = r < rows ? kInfHi : 0u;
    rm_lo[i] = 0u;
    rm_j[i] = r < rows ? static_cast<uint32_t>(r * 32) : kNoIndex;
  }
  GroupSetup gs;
  gs.b = b;
  gs.s = s;
  gs.g = g;
  int cur = first_point(p, gs);
  if (lane == 0) {
    write_index(p, b, g.out_off, g.begin + cur);
    sampled[cur >> 5] |= 1u << (cur & 31);
  }
  __syncwarp();
  const long long K = p.K;
  const int half_down = static_cast<int>(K / 2), half_up = static_cast<int>((K + 1) / 2);
  unsigned writes = 0;
  unsigned long long evals = 0;

  for (int it = 1; it < g.quota; ++it) {
    const double px = xs[cur], py = ys[cur], pz = zs[cur];
    const int wb = cur >= half_down ? cur - half_down : 0;
    const int we = min(n, cur + half_up);
    evals += static_cast<unsigned long long>(we - wb);
    const int r_lo = wb >> 5, r_hi = (we - 1) >> 5;
#pragma unroll 2
    for (int r = r_lo; r <= r_hi; ++r) {
      const int j = (r << 5) + lane;
      double dj = j < n ? d[j] : 0.0;
      if (j >= wb && j < we) {
        const double dist = dist2(xs[j], ys[j], zs[j], px, py, pz);
        const bool lower = dist <= dj;
        writes += lower ? 1u : 0u;
        if (lower) {
          dj = dist;
          d[j] = dist;
        }
      }
      const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(dj));
      uint32_t hi = static_cast<uint32_t>(bits >> 32), lo = static_cast<uint32_t>(bits);
      uint32_t jj = j < n ? static_cast<uint32_t>(j) : kNoIndex;
      warp_argmax(hi, lo, jj);
#pragma unroll
      for (int i = 0; i < RPL; ++i)
        if ((r >> 5) == i && (r & 31) == lane) {
          rm_hi[i] = hi;
          rm_lo[i] = lo;
          rm_j[i] = jj;
        }
    }
    if (p.trace) {
      __syncwarp();
      for (int j = lane; j < n; j += 32) p.trace[static_cast<long long>(it - 1) * n + j] = d[j];
    }
    // whole-sector argmax from the cached row maxima; rows l + 32*i grow with
    // i, so a strict > keeps the lowest index among equal distances
    uint32_t hi = rm_hi[0], lo = rm_lo[0], j = rm_j[0];
#pragma unroll
    for (int i = 1; i < RPL; ++i) {
      const bool gt = rm_hi[i] > hi || (rm_hi[i] == hi && rm_lo[i] > lo);
      hi = gt ? rm_hi[i] : hi;
      lo = gt ? rm_lo[i] : lo;
      j = gt ? rm_j[i] : j;
    }
    warp_argmax(hi, lo, j);
    if ((hi | lo) == 0u) {
      // every distance is 0: lowest unsampled index (sampler.cpp:148-154)
      uint32_t jm = kNoIndex;
      for (int w = lane; w < rows && jm == kNoIndex; w += 32) {
        const unsigned free_bits = ~sampled[w];
        if (free_bits) {
          const uint32_t cand = static_cast<uint32_t>(w * 32 + __ffs(free_bits) - 1);
          if (cand < static_cast<uint32_t>(n)) jm = cand;
        }
      }
      j = __reduce_min_sync(kFull, jm);
    }
    cur = static_cast<int>(j);
    if (lane == 0) {
      write_index(p, b, g.out_off + it, g.begin + cur);
      sampled[cur >> 5] |= 1u << (cur & 31);
    }
    __syncwarp();
  }
  const unsigned ws = __reduce_add_sync(kFull, writes);
  if (p.stats && lane == 0) {
    unsigned long long* st = p.stats + b * 4;
    const unsigned long long iters = static_cast<unsigned long long>(g.quota - 1);
    if (ws) atomicAdd(st + 1, static_cast<unsigned long long>(ws));
    atomicAdd(st + 0, evals);
    atomicAdd(st + 2, iters * static_cast<unsigned long long>(n));
    atomicAdd(st + 3, iters);
  }
}

// ---------------------------------------------------------------- dispatch

constexpr size_t kMaxSmem = 227 * 1024;

template <typename Kern>
cudaError_t launch_groups(Kern kern, SampleParams p, int W, int G, cudaStream_t st) {
  const size_t group_bytes = size_t(24) * p.nmax + 32 * W;
  const size_t smem = group_bytes * G;
  if (smem > kMaxSmem) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  p.G = G;
  const long long sectors = p.B * p.M;
  const long long blocks = (sectors + G - 1) / G;
  kern<<<static_cast<unsigned>(blocks), G * W * 32, smem, st>>>(p);
  return cudaGetLastError();
}

// Groups per CTA: up to `max_threads` threads and ~110 KB of shared memory
// (two CTAs per SM), fewer when there are not enough sectors to fill the SMs.
int pick_groups(long long sectors, int W, int nmax, int max_threads) {
  const size_t group_bytes = size_t(24) * nmax + 32 * W;
  int G = std::max(1, max_threads / (W * 32));
  if (W > 1) G = std::min(G, 15);  // named barriers 1..15
  while (G > 1 && group_bytes * G > 110 * 1024) G /= 2;
  while (G > 1 && (sectors + G - 1) / G < 2 * 148) G /= 2;
  return G;
}

template <int P, int W, bool REGC>
cudaError_t run_full(SampleParams p, cudaStream_t st) {
  const int G = pick_groups(p.B * p.M, W, p.nmax, W >= 8 ? W * 32 : 256);
  return launch_groups(fps_full_kernel<P, W, REGC>, p, W, std::min(G, W >= 8 ? 1 : 8 / W), st);
}

template <int RPL>
cudaError_t run_npdu(SampleParams p, cudaStream_t st) {
  const size_t warp_bytes = npdu_warp_bytes(p.nmax);
  int G = 4;
  while (G > 1 && warp_bytes * G > 110 * 1024) G /= 2;
  while (G > 1 && (p.B * p.M + G - 1) / G < 2 * 148) G /= 2;
  const size_t smem = warp_bytes * G;
  if (smem > kMaxSmem) return cudaErrorNotSupported;
  auto kern = npdu_warp_kernel<RPL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  p.G = G;
  const long long blocks = (p.B * p.M + G - 1) / G;
  kern<<<static_cast<unsigned>(blocks), 32 * G, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t dispatch(SampleParams p, long long nmax_sector, bool windowed, cudaStream_t st,
                     std::string* msg) {
  p.nmax = static_cast<int>((nmax_sector + 1) & ~1LL);
  const long long n = nmax_sector;
  if (!windowed) {
    if (n <= 32) return run_full<1, 1, true>(p, st);
    if (n <= 64) return run_full<2, 1, true>(p, st);
    if (n <= 128) return run_full<4, 1, true>(p, st);
    if (n <= 256) return run_full<8, 1, true>(p, st);
    if (n <= 512) return run_full<16, 1, true>(p, st);
    if (n <= 1024) return run_full<16, 2, true>(p, st);
    if (n <= 2048) return run_full<16, 4, true>(p, st);
    if (n <= 4096) return run_full<16, 8, true>(p, st);
    if (n <= 8192) return run_full<8, 32, false>(p, st);
  } else {
    cudaError_t e = cudaErrorNotSupported;
    if (n <= 1024) e = run_npdu<1>(p, st);
    else if (n <= 2048) e = run_npdu<2>(p, st);
    else if (n <= 4096) e = run_npdu<4>(p, st);
    else if (n <= 7040) e = run_npdu<8>(p, st);
    if (e != cudaErrorNotSupported) return e;
  }
  if (msg) *msg = "sector of " + std::to_string(n) + " points exceeds the on-chip sampler (8192)";
  return cudaErrorNotSupported;
}

}  // namespace pcsk

namespace pcs_internal {

cudaError_t launch_sample(const pcs_gpu_args& a, cudaStream_t stream, std::string* msg) {
  const bool sectored = a.method == PCS_METHOD_AFPS || a.method == PCS_METHOD_NPDU_AFPS;
  const bool windowed = a.method == PCS_METHOD_NPDU_FPS || a.method == PCS_METHOD_NPDU_AFPS;
  const long long M = sectored ? a.m : 1;
  const long long nmax = (a.n + M - 1) / M;
  pcsk::SampleParams p{};
  p.xyz = a.xyz;
  p.f64 = a.coord_dtype == PCS_DTYPE_F64;
  p.B = a.batch;
  p.N = a.n;
  p.C = a.c;
  p.M = M;
  // A window that always covers the whole sector is the full update
  // (k >= 2*n-1 => update_window == sector for every pivot), and the
  // OpStats agree: every window then holds the sector's n points.
  p.K = (windowed && a.k < 2 * nmax - 1) ? a.k : 0;
  p.random_first = a.seed_policy == PCS_RANDOM_FIRST_POINT;
  p.seed = a.seed;
  p.seeds = a.seeds;
  p.out_idx = a.out_indices;
  p.idx64 = a.index_dtype == PCS_INDEX_I64;
  p.out_sector = a.out_sector;
  p.stats = reinterpret_cast<unsigned long long*>(a.out_stats);
  p.index_base = a.index_base;
  p.sector_base = a.sector_base;
  if (a.out_stats) {
    cudaError_t e = cudaMemsetAsync(a.out_stats, 0, sizeof(uint64_t) * 4 * a.batch, stream);
    if (e != cudaSuccess) return e;
  }
  return pcsk::dispatch(p, nmax, p.K > 0, stream, msg);
}

cudaError_t launch_local_fps(const double* xyz, int64_t n, int64_t sb, int64_t se,
                             int64_t quota, int64_t k, int random_first, uint64_t seed,
                             int64_t* out_idx, uint64_t* out_stats, double* trace,
                             cudaStream_t stream, std::string* msg) {
  (void)n;
  const long long len = se - sb;
  pcsk::SampleParams p{};
  p.xyz = xyz + 3 * sb;
  p.f64 = 1;
  p.B = 1;
  p.N = len;
  p.C = quota;
  p.M = 1;
  p.K = (k > 0 && k < 2 * len - 1) ? k : 0;
  p.random_first = random_first;
  p.seed = seed;
  p.out_idx = out_idx;
  p.idx64 = 1;
  p.index_base = sb;
  p.stats = reinterpret_cast<unsigned long long*>(out_stats);
  p.trace = trace;
  cudaError_t e = cudaMemsetAsync(out_stats, 0, sizeof(uint64_t) * 4, stream);
  if (e != cudaSuccess) return e;
  return pcsk::dispatch(p, len, p.K > 0, stream, msg);
}

}  // namespace pcs_internal
