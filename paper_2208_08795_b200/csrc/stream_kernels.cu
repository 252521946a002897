// Streaming sampler for sectors beyond every on-chip engine (FPS / AFPS /
// NPDU variants), sm_100a.
//
// One cooperative launch per sector over all SMs: d[] (fp64) lives in global
// memory (L2-resident up to several million points: 126 MB of L2), each CTA
// owns a contiguous chunk of the sector. One iteration of local_fps
// (proj/src/sampler.cpp:114-161) is
//   1. every CTA updates its chunk's part of the window (reference operation
//      order, `dist <= d`) and reduces its chunk to a (max d, min index) key;
//      a CTA whose chunk misses the window keeps its previous key (NPDU:
//      most CTAs do no work at all);
//   2. one grid-wide barrier; every CTA reduces the G keys (double-buffered
//      by iteration parity, so one barrier per iteration suffices);
//   3. all-zero maximum: the lowest unsampled index (bitmap in global memory,
//      a second barrier on that rare path).
// Results, OpStats and the trace are the reference's, exactly.
#include <cooperative_groups.h>

#include <algorithm>

#include "internal.h"
#include "sampler_common.cuh"

namespace cg = cooperative_groups;

namespace pcsk {

namespace {

constexpr int kStreamThreads = 512;

__device__ __forceinline__ bool key_greater(uint32_t h1, uint32_t l1, uint32_t j1, uint32_t h2,
                                            uint32_t l2, uint32_t j2) {
  return h1 > h2 || (h1 == h2 && (l1 > l2 || (l1 == l2 && j1 < j2)));
}

// CTA-wide (max key, min index) -> every thread
__device__ __forceinline__ void block_argmax(uint32_t& hi, uint32_t& lo, uint32_t& j,
                                             uint4* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int W = kStreamThreads / 32;
  warp_argmax(hi, lo, j);
  __syncthreads();  // red[] of the previous use is consumed
  if (lane == 0) red[warp] = make_uint4(hi, lo, j, 0);
  __syncthreads();
  const uint4 v = lane < W ? red[lane] : make_uint4(0, 0, kNoIndex, 0);
  hi = v.x;
  lo = v.y;
  j = v.z;
  warp_argmax(hi, lo, j);
}

template <typename T>
__device__ __forceinline__ double coord(const T* src, long long j, int a) {
  return static_cast<double>(src[3 * j + a]);  // exact for fp32
}

}  // namespace

template <typename T>
__global__ void __launch_bounds__(kStreamThreads)
    stream_sector_kernel(const SampleParams p, long long b, long long s, double* __restrict__ d,
                         unsigned* __restrict__ sampled, uint4* __restrict__ cand) {
  __shared__ uint4 red[kStreamThreads / 32];
  cg::grid_group grid = cg::this_grid();
  const SectorGeom g = sector_geom(p.N, p.C, p.M, s);
  const long long n = g.n;
  const T* src = static_cast<const T*>(p.xyz) + (b * p.N + g.begin) * 3;
  const int G = gridDim.x;
  const long long per = (n + G - 1) / G;
  const long long c0 = ::min(n, static_cast<long long>(blockIdx.x) * per), c1 = ::min(n, c0 + per);
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  for (long long j = c0 + threadIdx.x; j < c1; j += kStreamThreads) d[j] = kInf;
  for (long long w = (c0 >> 5) + threadIdx.x; w <= ((c1 - 1) >> 5) && c1 > c0; w += kStreamThreads)
    sampled[w] = 0u;  // words may straddle chunks: both owners write 0
  if (p.out_sector && blockIdx.x == 0)
    for (int i = threadIdx.x; i < g.quota; i += kStreamThreads)
      p.out_sector[b * p.C + g.out_off + i] = static_cast<int>(s + p.sector_base);
  GroupSetup gs;
  gs.b = b;
  gs.s = s;
  gs.g = g;
  long long cur = first_point(p, gs);
  const long long out_base = b * p.C + g.out_off;
  const long long index_off = g.begin + p.index_base;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (p.idx64) static_cast<long long*>(p.out_idx)[out_base] = index_off + cur;
    else static_cast<int*>(p.out_idx)[out_base] = static_cast<int>(index_off + cur);
  }
  grid.sync();  // d / bitmap initialised everywhere
  if (threadIdx.x == 0 && cur >= c0 && cur < c1) atomicOr(&sampled[cur >> 5], 1u << (cur & 31));
  const long long K = p.K;
  const long long half_down = K / 2, half_up = (K + 1) / 2;
  unsigned writes = 0;
  unsigned long long evals = 0;
  // this CTA's chunk key, valid while the chunk is untouched
  uint32_t kh = 0u, kl = 0u, kj = kNoIndex;
  bool fresh = false;
  for (int it = 1; it < g.quota; ++it) {
    const double px = coord(src, cur, 0), py = coord(src, cur, 1), pz = coord(src, cur, 2);
    long long wb = 0, we = n;
    if (K > 0) {
      wb = cur >= half_down ? cur - half_down : 0;
      we = ::min(n, cur + half_up);
    }
    evals += static_cast<unsigned long long>(we - wb);
    const long long u0 = ::max(c0, wb), u1 = ::min(c1, we);
    if (u0 < u1 || !fresh) {
      uint32_t hi = 0u, lo = 0u, jj = kNoIndex;
      for (long long j = c0 + threadIdx.x; j < c1; j += kStreamThreads) {
        double dj = d[j];
        if (j >= u0 && j < u1) {
          const double e = dist2(coord(src, j, 0), coord(src, j, 1), coord(src, j, 2), px, py, pz);
          if (e <= dj) {
            dj = e;
            d[j] = e;
            ++writes;
          }
        }
        if (p.trace) p.trace[static_cast<long long>(it - 1) * n + j] = dj;
        const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(dj));
        const uint32_t h = static_cast<uint32_t>(bits >> 32), l = static_cast<uint32_t>(bits);
        if (key_greater(h, l, static_cast<uint32_t>(j), hi, lo, jj)) {
          hi = h; lo = l; jj = static_cast<uint32_t>(j);
        }
      }
      block_argmax(hi, lo, jj, red);
      kh = hi; kl = lo; kj = jj;
      fresh = true;
    } else if (p.trace) {
      for (long long j = c0 + threadIdx.x; j < c1; j += kStreamThreads)
        p.trace[static_cast<long long>(it - 1) * n + j] = d[j];
    }
    uint4* buf = cand + (it & 1) * G;
    if (threadIdx.x == 0) buf[blockIdx.x] = make_uint4(kh, kl, kj, 0);
    grid.sync();
    // every CTA reduces the G chunk keys (warp 0 of each, then broadcast)
    uint32_t hi = 0u, lo = 0u, jj = kNoIndex;
    for (int c = threadIdx.x; c < G; c += kStreamThreads) {
      const uint4 v = buf[c];
      if (key_greater(v.x, v.y, v.z, hi, lo, jj)) { hi = v.x; lo = v.y; jj = v.z; }
    }
    block_argmax(hi, lo, jj, red);
    if ((hi | lo) == 0u) {
      // every distance is 0: lowest unsampled index (sampler.cpp:148-154)
      uint32_t jm = kNoIndex;
      for (long long j = c0 + threadIdx.x; j < c1; j += kStreamThreads)
        if (!((sampled[j >> 5] >> (j & 31)) & 1u)) { jm = static_cast<uint32_t>(j); break; }
      uint32_t one = jm != kNoIndex ? 1u : 0u, zero = 0u;
      uint32_t mh = 0u;
      // (min index among unsampled) as a max-key reduction: key (1, 0, j)
      block_argmax(one, zero, jm, red);
      mh = one;
      uint4* buf2 = cand + 2 * G + (it & 1) * G;
      if (threadIdx.x == 0) buf2[blockIdx.x] = make_uint4(mh, 0u, jm, 0);
      grid.sync();
      uint32_t h2 = 0u, l2 = 0u, j2 = kNoIndex;
      for (int c = threadIdx.x; c < G; c += kStreamThreads) {
        const uint4 v = buf2[c];
        if (key_greater(v.x, v.y, v.z, h2, l2, j2)) { h2 = v.x; l2 = v.y; j2 = v.z; }
      }
      block_argmax(h2, l2, j2, red);
      jj = j2;
    }
    cur = jj;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (p.idx64) static_cast<long long*>(p.out_idx)[out_base + it] = index_off + cur;
      else static_cast<int*>(p.out_idx)[out_base + it] = static_cast<int>(index_off + cur);
    }
    if (cur >= c0 && cur < c1) {
      if (threadIdx.x == 0) atomicOr(&sampled[cur >> 5], 1u << (cur & 31));
      fresh = false;  // the pivot's own chunk changes next iteration anyway
    }
  }
  const unsigned ws = __reduce_add_sync(kFull, writes);
  if (p.stats) {
    unsigned long long* st = p.stats + b * 4;
    if ((threadIdx.x & 31) == 0 && ws) atomicAdd(st + 1, static_cast<unsigned long long>(ws));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const unsigned long long iters = static_cast<unsigned long long>(g.quota - 1);
      atomicAdd(st + 0, evals);
      atomicAdd(st + 2, iters * static_cast<unsigned long long>(n));
      atomicAdd(st + 3, iters);
    }
  }
}

cudaError_t run_stream_any(SampleParams p, long long nmax, cudaStream_t st) {
  if (plan("stream_sector_kernel", {p.f64 ? 8 : 4})) return cudaSuccess;
  int dev = 0, sms = 0, per_sm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  auto kern = p.f64 ? reinterpret_cast<const void*>(stream_sector_kernel<double>)
                    : reinterpret_cast<const void*>(stream_sector_kernel<float>);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kStreamThreads, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorNotSupported;
  const int G = sms * std::min(per_sm, 2);
  const size_t words = static_cast<size_t>((nmax + 31) / 32);
  const size_t bytes = sizeof(double) * static_cast<size_t>(nmax) + 4 * words + 16 * 4 * G + 16;
  void* ws = nullptr;
  e = pcs_internal::workspace_alloc(&ws, bytes, st);
  if (e != cudaSuccess) return e;
  double* d = static_cast<double*>(ws);
  unsigned* sampled = reinterpret_cast<unsigned*>(d + nmax);
  uint4* cand = reinterpret_cast<uint4*>(
      (reinterpret_cast<uintptr_t>(sampled + words) + 15) & ~static_cast<uintptr_t>(15));
  for (long long b = 0; b < p.B && e == cudaSuccess; ++b)
    for (long long s = 0; s < p.M && e == cudaSuccess; ++s) {
      void* args[] = {&p, &b, &s, &d, &sampled, &cand};
      e = cudaLaunchCooperativeKernel(kern, dim3(G), dim3(kStreamThreads), args, 0, st);
    }
  const cudaError_t e2 = cudaFreeAsync(ws, st);
  return e != cudaSuccess ? e : e2;
}

}  // namespace pcsk
