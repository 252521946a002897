// Per-cloud stable axis sort for sm_100a: the B200 form of pcs::exact_sort
// (proj/src/order.cpp:11-24: std::stable_sort of storage indices by
// points[i][axis] with operator<, then a gather).
//
// Keys: the coordinate's IEEE bits mapped to an order-preserving unsigned
// integer, with -0.0 first folded onto +0.0 (operator< treats them as
// equal, so stability must keep their storage order). NaN is excluded by
// the reference's precondition (proj/src/point_cloud.cpp:43-50).
//
// * fp32, N <= 4096, and up to 37 clouds of <= 65536: the on-chip LSD radix
//   (radix_reg_kernel, end of this file; a cluster of CTAs for N > 4096);
//   148+ clouds of <= 32768: radix_cta_kernel (one CTA per cloud, or a
//   2-CTA cluster merging its sorted halves).
// * fp32, N <= 16384 otherwise: one CTA per cloud sorts packed (key << 32 | index)
//   words with a bitonic network in shared memory. Packing the storage index
//   into the low bits makes every word unique and orders ties by index, so an
//   unstable network yields exactly the stable order.
// * fp32, 16384 < N <= 262144: the same network over a thread-block cluster
//   of up to 16 CTAs (16384 words each in shared memory; cross-CTA steps
//   through DSMEM). Larger fp32 clouds: the network in global (L2) memory,
//   block-local steps in shared memory, one launch per global step.
// * fp64 keys (the drop-in path): one CTA per cloud runs an LSD
//   radix sort, 8-bit digits, over global ping-pong buffers (L2-resident),
//   with tile-ordered ranking (match.any + per-warp digit counts) so every
//   pass is stable. Passes whose digit is constant across the cloud are
//   skipped.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>

#include "device_common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace pcsk {

__device__ __forceinline__ uint32_t order_key(float v) {
  uint32_t b = __float_as_uint(v);
  if (b == 0x80000000u) b = 0;  // -0.0 == +0.0 under operator<
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ uint64_t order_key(double v) {
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
  if (b == 0x8000000000000000ull) b = 0;
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

template <typename T>
__device__ __forceinline__ void gather_point(const T* __restrict__ src, T* __restrict__ dst,
                                             long long i, long long from) {
  dst[3 * i] = src[3 * from];
  dst[3 * i + 1] = src[3 * from + 1];
  dst[3 * i + 2] = src[3 * from + 2];
}

constexpr int kSortThreads = 1024;

__global__ void __launch_bounds__(kSortThreads)
    bitonic_sort_kernel(const float* __restrict__ xyz, long long N, int axis, int npow2,
                        float* __restrict__ out_xyz, int* __restrict__ out_perm) {
  extern __shared__ __align__(16) unsigned long long words[];
  const long long b = blockIdx.x;
  const float* src = xyz + b * N * 3;
  for (int i = threadIdx.x; i < npow2; i += kSortThreads)
    words[i] = i < N ? (static_cast<unsigned long long>(order_key(src[3LL * i + axis])) << 32) |
                           static_cast<unsigned>(i)
                     : ~0ull;
  __syncthreads();
  const int half = npow2 >> 1;
  for (int k = 2; k <= npow2; k <<= 1) {
    for (int j = k >> 1, lj = __ffs(k) - 2; j > 0; j >>= 1, --lj) {
      for (int i = threadIdx.x; i < half; i += kSortThreads) {
        // j is a power of two: pair (lo, lo + j) without integer division
        const int lo = ((i >> lj) << (lj + 1)) | (i & (j - 1)), hi = lo + j;
        const unsigned long long a = words[lo], c = words[hi];
        const bool ascending = (lo & k) == 0;
        if ((a > c) == ascending) {
          words[lo] = c;
          words[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  float* dst = out_xyz + b * N * 3;
  for (int i = threadIdx.x; i < N; i += kSortThreads) {
    const int from = static_cast<int>(words[i] & 0xffffffffu);
    if (out_perm) out_perm[b * N + i] = from;
    if (out_xyz) gather_point(src, dst, i, from);
  }
}

// LSD radix, one CTA per cloud. KeyT is uint32_t (fp32) or uint64_t (fp64).
template <typename T, typename KeyT>
__global__ void __launch_bounds__(kSortThreads)
    radix_sort_kernel(const T* __restrict__ xyz, long long N, int axis, KeyT* keys_a,
                      KeyT* keys_b, uint32_t* idx_a, uint32_t* idx_b, T* __restrict__ out_xyz,
                      int* __restrict__ out_perm) {
  __shared__ unsigned hist[256];
  __shared__ unsigned base[256];
  __shared__ unsigned tile_total[256];
  __shared__ unsigned wcount[32][257];
  __shared__ int skip;
  const long long b = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const T* src = xyz + b * N * 3;
  KeyT* ks = keys_a + b * N;
  KeyT* kd = keys_b + b * N;
  uint32_t* is = idx_a + b * N;
  uint32_t* id = idx_b + b * N;
  for (long long i = t; i < N; i += kSortThreads) {
    ks[i] = order_key(src[3 * i + axis]);
    is[i] = static_cast<uint32_t>(i);
  }
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int shift = 0; shift < int(sizeof(KeyT) * 8); shift += 8) {
    if (t < 256) hist[t] = 0;
    __syncthreads();
    for (long long i = t; i < N; i += kSortThreads)
      atomicAdd(&hist[static_cast<unsigned>(ks[i] >> shift) & 255u], 1u);
    __syncthreads();
    if (t == 0) {
      unsigned run = 0;
      int constant = 0;
      for (int dgt = 0; dgt < 256; ++dgt) {
        base[dgt] = run;
        run += hist[dgt];
        constant |= hist[dgt] == static_cast<unsigned>(N);
      }
      skip = constant;
    }
    __syncthreads();
    if (skip) continue;  // every key shares this digit: the pass is the identity
    for (long long tile = 0; tile < N; tile += kSortThreads) {
      const long long i = tile + t;
      const bool valid = i < N;
      const KeyT key = valid ? ks[i] : KeyT(0);
      const uint32_t ix = valid ? is[i] : 0u;
      const unsigned dgt = valid ? (static_cast<unsigned>(key >> shift) & 255u) : 256u;
      for (int e = t; e < 32 * 257; e += kSortThreads) (&wcount[0][0])[e] = 0;
      __syncthreads();
      const unsigned peers = __match_any_sync(kFull, dgt);
      const unsigned wrank = __popc(peers & lt_mask);
      if (valid && (peers & lt_mask) == 0) wcount[warp][dgt] = __popc(peers);
      __syncthreads();
      if (t < 256) {
        unsigned run = 0;
        for (int w = 0; w < 32; ++w) {
          const unsigned c = wcount[w][t];
          wcount[w][t] = run;
          run += c;
        }
        tile_total[t] = run;
      }
      __syncthreads();
      if (valid) {
        const unsigned dst = base[dgt] + wcount[warp][dgt] + wrank;
        kd[dst] = key;
        id[dst] = ix;
      }
      __syncthreads();
      if (t < 256) base[t] += tile_total[t];
      __syncthreads();
    }
    KeyT* tk = ks; ks = kd; kd = tk;
    uint32_t* ti = is; is = id; id = ti;
  }
  T* dst = out_xyz ? out_xyz + b * N * 3 : nullptr;
  for (long long i = t; i < N; i += kSortThreads) {
    const uint32_t from = is[i];
    if (out_perm) out_perm[b * N + i] = static_cast<int>(from);
    if (dst) gather_point(src, dst, i, from);
  }
}


// Register-resident bitonic for 2048 <= npow2 <= 16384 (one CTA per cloud,
// 1024 threads, E = npow2 / 1024 words per thread in registers, blocked:
// thread t holds words t*E .. t*E+E-1). Steps with j < E run in registers,
// E <= j < 32E through warp shuffles, and only j >= 32E through shared
// memory with a block barrier -- 15 barrier steps for 16384 words instead of
// the 105 of the all-shared-memory network.
// CS > 1: the cloud spans a cluster of CS CTAs (global word index
// rank * NP + local); steps whose partner lives in another CTA (j >= NP) go
// through DSMEM with cluster barriers.
// shared-memory word index with one pad word per 32: the blocked register
// layout (thread t's words t*E .. t*E+E-1) would otherwise put all 32 lanes
// of a warp on the same banks when it spills to / reloads from shared memory
__device__ __forceinline__ int spad(int i) { return i + (i >> 5); }

template <int E, int CS>
__global__ void __launch_bounds__(kSortThreads)
    bitonic_reg_kernel(const float* __restrict__ xyz, long long N, int axis,
                       float* __restrict__ out_xyz, int* __restrict__ out_perm) {
  extern __shared__ __align__(16) unsigned long long words[];
  constexpr int NP = E * kSortThreads;
  const int rank = CS > 1 ? static_cast<int>(cg::this_cluster().block_rank()) : 0;
  const long long b = blockIdx.x / CS;
  const long long base = static_cast<long long>(rank) * NP;
  const int t = threadIdx.x, lane = t & 31;
  const float* src = xyz + b * N * 3;
  unsigned long long x[E];
  // vector path: whole thread block of points in range and 16-byte aligned
  const long long g0 = base + static_cast<long long>(t) * E;  // first global word
  const bool vec = E % 4 == 0 && g0 + E <= N && ((b * N) & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(xyz) & 15) == 0;
  if (vec) {
    // this thread's E points are 3E consecutive floats (16-byte aligned when
    // E is a multiple of 4): vector loads, then pick the axis
    float v[3 * E];
    const float* p = src + 3 * g0;
    if constexpr (E % 4 == 0) {
#pragma unroll
      for (int q = 0; q < 3 * E / 4; ++q) {
        const float4 f = reinterpret_cast<const float4*>(p)[q];
        v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 3 * E; ++q) v[q] = p[q];
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const float key = axis == 0 ? v[3 * e] : (axis == 1 ? v[3 * e + 1] : v[3 * e + 2]);
      x[e] = (static_cast<unsigned long long>(order_key(key)) << 32) | static_cast<unsigned>(g0 + e);
    }
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const long long i = g0 + e;
      x[e] = i < N ? (static_cast<unsigned long long>(order_key(src[3 * i + axis])) << 32) |
                         static_cast<unsigned>(i)
                   : ~0ull;
    }
  }
  for (long long k = 2; k <= static_cast<long long>(NP) * CS; k <<= 1) {
    long long j = k >> 1;
    if (j >= 32 * E) {
#pragma unroll
      for (int e = 0; e < E; ++e) words[spad(t * E + e)] = x[e];
      if constexpr (CS > 1) {
        if (j >= NP) {
          // cross-CTA steps: the lower CTA of each pair exchanges in place
          for (; j >= NP; j >>= 1) {
            cg::this_cluster().sync();
            const int partner = rank ^ static_cast<int>(j / NP);
            if (rank < partner) {
              unsigned long long* remote = cg::this_cluster().map_shared_rank(words, partner);
              for (int q = t; q < NP; q += kSortThreads) {
                const unsigned long long a = words[spad(q)], c = remote[spad(q)];
                if ((a > c) == (((base + q) & k) == 0)) {
                  words[spad(q)] = c;
                  remote[spad(q)] = a;
                }
              }
            }
          }
          cg::this_cluster().sync();
        }
      }
      __syncthreads();
      for (; j >= 32 * E; j >>= 1) {
        const int lj = __ffsll(j) - 1;
        for (int q = t; q < NP / 2; q += kSortThreads) {
          const int lo = ((q >> lj) << (lj + 1)) | (q & static_cast<int>(j - 1)), hi = lo + static_cast<int>(j);
          const unsigned long long a = words[spad(lo)], c = words[spad(hi)];
          if ((a > c) == (((base + lo) & k) == 0)) {
            words[spad(lo)] = c;
            words[spad(hi)] = a;
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = words[spad(t * E + e)];
      __syncthreads();
    }
    for (; j >= E; j >>= 1) {
      const int d = static_cast<int>(j / E);  // partner lane distance
      // j, k >= E: which half of the pair and the direction depend on the
      // thread only
      const bool keep_min = ((g0 & j) == 0) == ((g0 & k) == 0);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const unsigned long long o = __shfl_xor_sync(kFull, x[e], d);
        x[e] = (o < x[e]) == keep_min ? o : x[e];
      }
    }
#pragma unroll
    for (int jj = E / 2; jj > 0; jj >>= 1) {
      if (jj > (k >> 1)) continue;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (e & jj) continue;
        const long long i = g0 + e;
        const unsigned long long a = x[e], c = x[e + jj];
        if ((a > c) == ((i & k) == 0)) {
          x[e] = c;
          x[e + jj] = a;
        }
      }
    }
  }
  (void)lane;
  float* dst = out_xyz ? out_xyz + b * N * 3 : nullptr;
  if (vec && (reinterpret_cast<uintptr_t>(out_perm) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(out_xyz) & 15) == 0) {
    // E consecutive outputs: vector stores of the permutation and the points
    int from[E];
#pragma unroll
    for (int e = 0; e < E; ++e) from[e] = static_cast<int>(x[e] & 0xffffffffu);
    if (out_perm) {
      int4* pp = reinterpret_cast<int4*>(out_perm + b * N + g0);
#pragma unroll
      for (int q = 0; q < E / 4; ++q) pp[q] = make_int4(from[4 * q], from[4 * q + 1], from[4 * q + 2], from[4 * q + 3]);
    }
    if (dst) {
      float v[3 * E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        // the point's 12 bytes from two aligned 8-byte loads (16 bytes
        // starting at the even float index at or below 3 * from)
        const long long i0 = 3LL * from[e];
        if (from[e] == N - 1) {  // the 16 bytes could run past the cloud
          v[3 * e] = src[i0]; v[3 * e + 1] = src[i0 + 1]; v[3 * e + 2] = src[i0 + 2];
          continue;
        }
        const float2* q = reinterpret_cast<const float2*>(src + (i0 & ~1LL));
        const float2 a = __ldg(q), c = __ldg(q + 1);
        const bool odd = i0 & 1;
        v[3 * e] = odd ? a.y : a.x;
        v[3 * e + 1] = odd ? c.x : a.y;
        v[3 * e + 2] = odd ? c.y : c.x;
      }
      float4* dp = reinterpret_cast<float4*>(dst + 3 * g0);
#pragma unroll
      for (int q = 0; q < 3 * E / 4; ++q) dp[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    if constexpr (CS > 1) cg::this_cluster().sync();
    return;
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const long long i = g0 + e;
    if (i < N) {
      const int from = static_cast<int>(x[e] & 0xffffffffu);
      if (out_perm) out_perm[b * N + i] = from;
      if (dst) gather_point(src, dst, i, from);
    }
  }
  if constexpr (CS > 1) cg::this_cluster().sync();  // partners may still read our words
}

template <int E, int CS = 1>
cudaError_t launch_reg_sort(const float* xyz, long long batch, long long n, int axis,
                            float* out_xyz, int* out_perm, cudaStream_t st) {
  const size_t smem = sizeof(unsigned long long) * (E * kSortThreads + E * kSortThreads / 32);
  auto kern = bitonic_reg_kernel<E, CS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  if (CS > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(batch * CS));
  cfg.blockDim = dim3(kSortThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, xyz, n, axis, out_xyz, out_perm);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Cluster size unit of the register networks (launch_reg_sort<16, CS>):
// one CTA holds 16384 keys.
constexpr int kBlk = 16384;

// ---------------------------------------------------------------- device-wide radix
// Large clouds (fp32 > 256K points, fp64 >= 64K): LSD radix over many CTAs
// per cloud, 8-bit digits, three launches per pass -- per-tile digit
// histograms, one exclusive scan per cloud over (digit, tile), and a stable
// scatter. Tiles are kRadixTile consecutive keys; inside a tile, warp w owns
// the contiguous run [w*256, w*256+256) and ranks its keys in order with
// match.any, so the scatter preserves input order within each digit (stable,
// as std::stable_sort). Keys are the order-preserving images of the
// coordinates (order_key), values the storage indices.
constexpr int kRadixThreads = 512;
constexpr int kRadixPerThread = 8;
constexpr int kRadixTile = kRadixThreads * kRadixPerThread;  // 4096

template <typename T, typename KeyT, bool FIRST>
__device__ __forceinline__ KeyT rs_key(const T* __restrict__ xyz, const KeyT* __restrict__ keys,
                                       long long b, long long N, long long i, int axis) {
  if constexpr (FIRST)
    return order_key(xyz[(b * N + i) * 3 + axis]);
  else
    return keys[b * N + i];
}

template <typename T, typename KeyT, bool FIRST>
__global__ void __launch_bounds__(kRadixThreads) rs_hist_kernel(const T* __restrict__ xyz, int axis,
                                                                const KeyT* __restrict__ keys,
                                                                long long N, int shift,
                                                                uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  const long long b = blockIdx.y;
  const int tiles = gridDim.x, tile = blockIdx.x;
  if (threadIdx.x < 256) h[threadIdx.x] = 0;
  __syncthreads();
  const long long t0 = static_cast<long long>(tile) * kRadixTile;
#pragma unroll
  for (int e = 0; e < kRadixPerThread; ++e) {
    const long long i = t0 + e * kRadixThreads + threadIdx.x;
    if (i < N)
      atomicAdd(&h[static_cast<uint32_t>(rs_key<T, KeyT, FIRST>(xyz, keys, b, N, i, axis) >> shift) & 255u], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 256) hist[(b * 256 + threadIdx.x) * tiles + tile] = h[threadIdx.x];
}

// per (cloud, digit): exclusive scan of the digit's tile counts in place,
// and the digit's total into totals[b][d] (the scatter scans the 256 totals)
__global__ void __launch_bounds__(256) rs_scan_kernel(uint32_t* __restrict__ hist,
                                                      uint32_t* __restrict__ totals, int tiles) {
  __shared__ uint32_t wsum[8];
  __shared__ uint32_t carry;
  const long long b = blockIdx.y;
  const int d = blockIdx.x;
  uint32_t* h = hist + (b * 256 + d) * static_cast<long long>(tiles);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < tiles; base += 256) {
    const int i = base + threadIdx.x;
    const uint32_t v = i < tiles ? h[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, off);
      if (lane >= off) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    uint32_t before = carry;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    if (i < tiles) h[i] = before + x - v;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t c = carry;
      for (int w = 0; w < 8; ++w) c += wsum[w];
      carry = c;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[b * 256 + d] = carry;
}

// exclusive scan of 256 counters in shared memory by one warp (8 per lane)
__device__ __forceinline__ void rs_scan256(uint32_t* c256, int lane) {
  uint32_t c[8], sum = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) { c[q] = c256[lane * 8 + q]; sum += c[q]; }
  uint32_t x = sum;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, off);
    if (lane >= off) x += y;
  }
  uint32_t run = x - sum;
#pragma unroll
  for (int q = 0; q < 8; ++q) { c256[lane * 8 + q] = run; run += c[q]; }
}

template <typename KeyT>
constexpr size_t rs_scatter_smem() {
  return sizeof(uint32_t) * (kRadixThreads / 32) * 256 + sizeof(uint32_t) * 512 +
         (sizeof(KeyT) + sizeof(uint32_t)) * kRadixTile;
}

// Stable scatter of one tile: rank in order (match.any per warp), regroup
// the tile by digit in shared memory, then write each digit's run
// contiguously. FIRST reads the keys from the cloud (values = storage
// indices); LAST writes the permutation and the gathered cloud instead of
// keys/values.
template <typename T, typename KeyT, bool FIRST, bool LAST>
__global__ void __launch_bounds__(kRadixThreads) rs_scatter_kernel(
    const T* __restrict__ xyz, int axis, const KeyT* __restrict__ kin,
    const uint32_t* __restrict__ vin, long long N, int shift, const uint32_t* __restrict__ offs,
    const uint32_t* __restrict__ totals, KeyT* __restrict__ kout, uint32_t* __restrict__ vout,
    T* __restrict__ out_xyz, int* __restrict__ out_perm) {
  constexpr int W = kRadixThreads / 32;
  extern __shared__ __align__(16) unsigned char rsm[];
  KeyT* skey = reinterpret_cast<KeyT*>(rsm);
  uint32_t* sval = reinterpret_cast<uint32_t*>(skey + kRadixTile);
  uint32_t (*wcount)[256] = reinterpret_cast<uint32_t (*)[256]>(sval + kRadixTile);
  uint32_t* dbase = &wcount[W - 1][0] + 256;  // digit base in the cloud
  uint32_t* tbase = dbase + 256;               // digit base in the tile
  const long long b = blockIdx.y;
  const int tiles = gridDim.x, tile = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < W * 256; i += kRadixThreads) (&wcount[0][0])[i] = 0;
  if (threadIdx.x < 256) dbase[threadIdx.x] = totals[b * 256 + threadIdx.x];
  __syncthreads();
  if (warp == 0) rs_scan256(dbase, lane);
  const long long t0 = static_cast<long long>(tile) * kRadixTile;
  const long long w0 = t0 + warp * (32 * kRadixPerThread);
  const unsigned lt = (1u << lane) - 1u;
  KeyT key[kRadixPerThread];
  uint32_t val[kRadixPerThread], dg[kRadixPerThread], rk[kRadixPerThread];
#pragma unroll
  for (int r = 0; r < kRadixPerThread; ++r) {
    const long long i = w0 + r * 32 + lane;
    const bool valid = i < N;
    key[r] = valid ? rs_key<T, KeyT, FIRST>(xyz, kin, b, N, i, axis) : KeyT(0);
    val[r] = valid ? (FIRST ? static_cast<uint32_t>(i) : vin[b * N + i]) : 0u;
    dg[r] = valid ? (static_cast<uint32_t>(key[r] >> shift) & 255u) : 256u;
    const unsigned peers = __match_any_sync(kFull, dg[r]);
    const uint32_t before = valid ? wcount[warp][dg[r]] : 0u;
    rk[r] = before + __popc(peers & lt);
    __syncwarp();
    if (valid && (peers & lt) == 0) wcount[warp][dg[r]] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x < 256) {  // per digit: exclusive prefix over the warps, tile total
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t c = wcount[w][threadIdx.x];
      wcount[w][threadIdx.x] = run;
      run += c;
    }
    tbase[threadIdx.x] = run;
  }
  __syncthreads();
  if (warp == 0) rs_scan256(tbase, lane);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRadixPerThread; ++r) {
    if (dg[r] < 256u) {
      const uint32_t lp = tbase[dg[r]] + wcount[warp][dg[r]] + rk[r];
      skey[lp] = key[r];
      sval[lp] = val[r];
    }
  }
  __syncthreads();
  const int cnt = static_cast<int>(N - t0 < kRadixTile ? N - t0 : kRadixTile);
  const uint32_t* o = offs + b * 256LL * tiles;
  for (int i = threadIdx.x; i < cnt; i += kRadixThreads) {
    const uint32_t d = static_cast<uint32_t>(skey[i] >> shift) & 255u;
    const long long dst = static_cast<long long>(dbase[d]) + o[d * tiles + tile] + (i - tbase[d]);
    if constexpr (LAST) {
      const uint32_t from = sval[i];
      if (out_perm) out_perm[b * N + dst] = static_cast<int>(from);
      if (out_xyz) gather_point(xyz + b * N * 3, out_xyz + b * N * 3, dst, from);
    } else {
      kout[b * N + dst] = skey[i];
      vout[b * N + dst] = sval[i];
    }
  }
}

template <typename T, typename KeyT, bool FIRST, bool LAST>
cudaError_t rs_pass(const T* xyz, int axis, const KeyT* kin, const uint32_t* vin, long long n,
                    long long batch, long long tiles, int shift, uint32_t* hist, uint32_t* totals,
                    KeyT* kout, uint32_t* vout, T* out_xyz, int* out_perm, cudaStream_t st) {
  const dim3 tg(static_cast<unsigned>(tiles), static_cast<unsigned>(batch));
  rs_hist_kernel<T, KeyT, FIRST><<<tg, kRadixThreads, 0, st>>>(xyz, axis, kin, n, shift, hist);
  rs_scan_kernel<<<dim3(256, static_cast<unsigned>(batch)), 256, 0, st>>>(hist, totals,
                                                                        static_cast<int>(tiles));
  auto kern = rs_scatter_kernel<T, KeyT, FIRST, LAST>;
  constexpr size_t smem = rs_scatter_smem<KeyT>();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  kern<<<tg, kRadixThreads, smem, st>>>(xyz, axis, kin, vin, n, shift, hist, totals, kout, vout,
                                        out_xyz, out_perm);
  return cudaGetLastError();
}

template <typename T, typename KeyT>
cudaError_t launch_device_radix(const T* xyz, long long batch, long long n, int axis, T* out_xyz,
                                int* out_perm, cudaStream_t st) {
  const long long tiles = (n + kRadixTile - 1) / kRadixTile;
  const size_t count = static_cast<size_t>(batch) * static_cast<size_t>(n);
  const size_t bytes =
      count * (2 * sizeof(KeyT) + 8) + sizeof(uint32_t) * 256 * (tiles + 1) * batch;
  void* ws = nullptr;
  cudaError_t e = pcs_internal::workspace_alloc(reinterpret_cast<void**>(&ws), bytes, st);
  if (e != cudaSuccess) return e;
  char* p = static_cast<char*>(ws);
  KeyT* ka = reinterpret_cast<KeyT*>(p);
  KeyT* kb = ka + count;
  uint32_t* va = reinterpret_cast<uint32_t*>(kb + count);
  uint32_t* vb = va + count;
  uint32_t* hist = vb + count;
  uint32_t* totals = hist + 256 * tiles * batch;
  constexpr int passes = static_cast<int>(sizeof(KeyT));
  for (int q = 0; q < passes && e == cudaSuccess; ++q) {
    const int shift = 8 * q;
    if (q == 0)
      e = rs_pass<T, KeyT, true, false>(xyz, axis, nullptr, nullptr, n, batch, tiles, shift, hist,
                                        totals, kb, vb, nullptr, nullptr, st);
    else if (q == passes - 1)
      e = rs_pass<T, KeyT, false, true>(xyz, axis, ka, va, n, batch, tiles, shift, hist, totals,
                                        nullptr, nullptr, out_xyz, out_perm, st);
    else
      e = rs_pass<T, KeyT, false, false>(xyz, axis, ka, va, n, batch, tiles, shift, hist, totals,
                                         kb, vb, nullptr, nullptr, st);
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  const cudaError_t e2 = cudaFreeAsync(ws, st);
  return e != cudaSuccess ? e : e2;
}

// ------------------------------------------------------ on-chip radix sort
// Stable LSD radix (8-bit digits, 4 passes over the 32-bit order key) of a
// cloud held on chip: a CTA of NT threads keeps E keys + storage indices
// per thread in registers; CS > 1 spreads the cloud over a thread-block
// cluster (CS * NT * E points), exchanging digit totals and scattering
// through DSMEM. Layout: warp w of cluster rank r owns the contiguous
// segment g = (r * NT/32 + w) * 32E + e * 32 + lane (striped across lanes, so
// the order inside a warp is e-major, lane-minor). Per pass:
//   rank   per key: eight ballots on the digit give the lanes sharing it;
//          the warp's private count hist[w][d] before this key + the peers
//          at lower lanes = the key's rank inside the warp's digit run
//          (segment order = storage order, so every pass is stable);
//   scan   offsets[w][d] = keys with a smaller digit (whole cloud) + keys
//          with digit d in earlier CTAs + in earlier warps of this CTA;
//   scatter key/index to offsets[w][d] + rank (local or remote shared
//          memory), barrier, read back the striped segment.
// Passes whose digit is the same for every key are the identity: skipped.
// Padding slots (g >= N) carry the key 0xffffffff (a NaN pattern, excluded
// by the reference's precondition), so they stay behind every real key.
// lanes holding the same 8-bit digit: one ballot per bit (MATCH.ANY has a
// long, poorly pipelined latency -- it bounded the first version of this
// kernel, ncu short_scoreboard stalls on its consumers)
__device__ __forceinline__ unsigned digit_peers(uint32_t d) {
  // per bit: the bit as a predicate, its ballot, and the ballot or its
  // complement folded into the running AND (4 instructions; the plain C++
  // form compiled to ~7 per bit)
  unsigned peers = kFull;
#pragma unroll
  for (int bit = 0; bit < 8; ++bit) {
    asm("{\n\t.reg .pred p;\n\t.reg .b32 m;\n\t"
        "and.b32 m, %1, %2;\n\t"
        "setp.ne.u32 p, m, 0;\n\t"
        "vote.sync.ballot.b32 m, p, 0xffffffff;\n\t"
        "@!p not.b32 m, m;\n\t"
        "and.b32 %0, %0, m;\n\t}"
        : "+r"(peers) : "r"(d), "r"(1u << bit));
  }
  return peers;
}

// Rank of each of the warp's E x 32 keys (slot e of lane l = segment
// position 32 e + l) inside its digit run, packed two 16-bit ranks per rk
// word. The lanes sharing a digit (peers) take consecutive ranks; the warp's
// running count per digit in hw[] is advanced by one atomicAdd from the
// peers' leader lane. A warp's shared-memory atomics complete in program
// order, so slot e+1 sees slot e's counts and ranks follow storage order
// (stable) without a warp barrier between slots: the slots of a group are
// independent chains (ballots, then atomics, then the shuffles that
// broadcast each leader's old count), not one serial read-modify-write.
template <int E>
__device__ __forceinline__ void warp_rank(const uint32_t (&key)[E], int shift, uint32_t* hw,
                                          int lane, unsigned lt_mask, uint32_t (&rk)[E / 2]) {
  constexpr int G = E < 4 ? E : 4;
#pragma unroll
  for (int e0 = 0; e0 < E; e0 += G) {
    unsigned pm[G];
    uint32_t old[G];
    int ld[G];
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const uint32_t d = (key[e0 + u] >> shift) & 255u;
      pm[u] = digit_peers(d);
      ld[u] = __ffs(pm[u]) - 1;
      old[u] = 0;
      // leader lane only, predicated (no divergent branch)
      const uint32_t addr = static_cast<uint32_t>(__cvta_generic_to_shared(hw + d));
      asm volatile("{\n\t.reg .pred p;\n\t"
                   "setp.eq.s32 p, %1, %2;\n\t"
                   "@p atom.shared.add.u32 %0, [%3], %4;\n\t}"
                   : "+r"(old[u]) : "r"(lane), "r"(ld[u]), "r"(addr), "r"(__popc(pm[u]))
                   : "memory");
    }
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int e = e0 + u;
      const uint32_t r = __shfl_sync(kFull, old[u], ld[u]) + __popc(pm[u] & lt_mask);
      if (e & 1) rk[e >> 1] |= r << 16; else rk[e >> 1] = r;
    }
  }
}

template <int NT, int E, int CS, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    radix_reg_kernel(const float* __restrict__ xyz, long long N, int axis,
                     float* __restrict__ out_xyz, int* __restrict__ out_perm) {
  constexpr int NW = NT / 32, NP = NT * E, P = NT / 256;  // P threads per digit in the scan
  static_assert(NT % 256 == 0 && NW / P == 8, "scan layout: 8 warps per scan thread");
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* sk = smem;                 // NP keys
  uint32_t* si = smem + NP;            // NP indices
  uint32_t* hist = smem + 2 * NP;      // [NW][256]
  uint32_t* ctot = hist + 256 * NW;    // [2][256] this CTA's digit totals (cluster form),
                                       // double-buffered by pass parity
  uint32_t* wsum = ctot + 512;         // [NW]
  __shared__ int identity;
  const int rank = CS > 1 ? static_cast<int>(cg::this_cluster().block_rank()) : 0;
  const long long b = blockIdx.x / CS;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  uint32_t* hw = hist + w * 256;       // this warp's digit counts, then offsets
  const float* src = xyz + b * N * 3;
  const long long seg = (static_cast<long long>(rank) * NW + w) * (32 * E) + lane;
  constexpr long long T = static_cast<long long>(NP) * CS;

  uint32_t key[E], idx[E], rk[E / 2];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const long long g = seg + 32 * e;
    key[e] = g < N ? order_key(__ldg(src + 3 * g + axis)) : 0xffffffffu;
    idx[e] = static_cast<uint32_t>(g);
  }
  for (int shift = 0; shift < 32; shift += 8) {
    for (int i = t; i < 256 * NW; i += NT) hist[i] = 0;
    if (t == 0) identity = 0;
    __syncthreads();
    // rank inside the warp's digit run
    warp_rank<E>(key, shift, hw, lane, lt_mask, rk);
    __syncthreads();
    // scan: thread (d, q) owns warps 8q .. 8q+7 of digit d
    const int d = t / P, q = t % P;
    uint32_t* h = hist + 8 * q * 256 + d;
    uint32_t ex[8], s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { ex[i] = s; s += h[256 * i]; }
    uint32_t pre = s;  // inclusive over q inside the digit's P threads
#pragma unroll
    for (int o = 1; o < P; o <<= 1) {
      const uint32_t v = __shfl_up_sync(kFull, pre, o, P);
      if (q >= o) pre += v;
    }
    uint32_t tot = __shfl_sync(kFull, pre, P - 1, P);
    pre -= s;  // exclusive over q
    uint32_t rpre = 0;  // digit d in earlier CTAs of the cluster
    if constexpr (CS > 1) {
      uint32_t* ct = ctot + ((shift >> 3) & 1) * 256 + d;
      if (q == 0) *ct = tot;
      cg::this_cluster().sync();
      uint32_t g = 0;
#pragma unroll
      for (int r = 0; r < CS; ++r) {
        const uint32_t v = *cg::this_cluster().map_shared_rank(ct, r);
        rpre += r < rank ? v : 0u;
        g += v;
      }
      tot = g;
    }
    // digits with a smaller value: inclusive scan of tot over the digits
    uint32_t inc = tot;
#pragma unroll
    for (int o = P; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[w] = inc;
    if (q == 0 && tot == static_cast<uint32_t>(T)) identity = 1;
    __syncthreads();
    uint32_t wb = lane < NW ? wsum[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(kFull, wb, o);
      if (lane >= o) wb += v;
    }
    const uint32_t wbase = w > 0 ? __shfl_sync(kFull, wb, (w - 1) & 31) : 0u;
    const uint32_t dbase = wbase + inc - tot + rpre + pre;
#pragma unroll
    for (int i = 0; i < 8; ++i) h[256 * i] = dbase + ex[i];
    const int skip = identity;
    __syncthreads();
    if (skip) continue;
    if (CS == 1 && shift == 24) {
      // last pass of a one-CTA cloud: write the outputs at their sorted
      // positions directly
      float* dst = out_xyz ? out_xyz + b * N * 3 : nullptr;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t dd = (key[e] >> shift) & 255u;
        const uint32_t r = (e & 1) ? rk[e >> 1] >> 16 : rk[e >> 1] & 0xffffu;
        const uint32_t pos = hw[dd] + r;
        if (pos < N) {
          if (out_perm) out_perm[b * N + pos] = static_cast<int>(idx[e]);
          if (dst) gather_point(src, dst, pos, idx[e]);
        }
      }
      return;
    }
    // scatter
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t dd = (key[e] >> shift) & 255u;
      const uint32_t r = (e & 1) ? rk[e >> 1] >> 16 : rk[e >> 1] & 0xffffu;
      const uint32_t pos = hw[dd] + r;
      if constexpr (CS > 1) {
        const int dst = static_cast<int>(pos / NP);
        const uint32_t lp = pos % NP;
        *cg::this_cluster().map_shared_rank(sk + lp, dst) = key[e];
        *cg::this_cluster().map_shared_rank(si + lp, dst) = idx[e];
      } else {
        sk[pos] = key[e];
        si[pos] = idx[e];
      }
    }
    if constexpr (CS > 1) cg::this_cluster().sync(); else __syncthreads();
    const int lb = w * 32 * E + lane;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      key[e] = sk[lb + 32 * e];
      idx[e] = si[lb + 32 * e];
    }
  }
  float* dst = out_xyz ? out_xyz + b * N * 3 : nullptr;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const long long g = seg + 32 * e;
    if (g < N) {
      if (out_perm) out_perm[b * N + g] = static_cast<int>(idx[e]);
      if (dst) gather_point(src, dst, g, idx[e]);
    }
  }
  if constexpr (CS > 1) cg::this_cluster().sync();  // no CTA leaves while partners may read it
}

template <int NT, int E, int CS = 1, int MINB = 1>
cudaError_t launch_radix_reg(const float* xyz, long long batch, long long n, int axis,
                             float* out_xyz, int* out_perm, cudaStream_t st) {
  constexpr int NW = NT / 32;
  const size_t smem = sizeof(uint32_t) * (2 * NT * E + 256 * NW + 512 + NW);
  auto kern = radix_reg_kernel<NT, E, CS, MINB>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  if (CS > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(batch * CS));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, xyz, n, axis, out_xyz, out_perm);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// CTA-local digit offsets: hist[w][d] (per-warp digit counts) becomes the
// position of warp w's first key with digit d in the CTA's output order.
// Returns whether one digit holds all NP keys (the pass is the identity).
template <int NT>
__device__ __forceinline__ bool cta_digit_offsets(uint32_t* hist, uint32_t* wsum, int* flag,
                                                  uint32_t np) {
  constexpr int NW = NT / 32, P = NT / 256;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int d = t / P, q = t % P;
  uint32_t* h = hist + 8 * q * 256 + d;
  uint32_t ex[8], s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) { ex[i] = s; s += h[256 * i]; }
  uint32_t pre = s;
#pragma unroll
  for (int o = 1; o < P; o <<= 1) {
    const uint32_t v = __shfl_up_sync(kFull, pre, o, P);
    if (q >= o) pre += v;
  }
  const uint32_t tot = __shfl_sync(kFull, pre, P - 1, P);
  pre -= s;
  uint32_t inc = tot;
#pragma unroll
  for (int o = P; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) wsum[w] = inc;
  if (q == 0 && tot == np) *flag = 1;
  __syncthreads();
  uint32_t wb = lane < NW ? wsum[lane] : 0u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(kFull, wb, o);
    if (lane >= o) wb += v;
  }
  const uint32_t wbase = w > 0 ? __shfl_sync(kFull, wb, (w - 1) & 31) : 0u;
  const uint32_t dbase = wbase + inc - tot + pre;
#pragma unroll
  for (int i = 0; i < 8; ++i) h[256 * i] = dbase + ex[i];
  const bool skip = *flag != 0;
  __syncthreads();
  return skip;
}

// Large-cloud on-chip radix: one CTA sorts NP = NT * E points with only the
// keys in registers; the 16-bit storage indices stay in shared memory
// (double-buffered, moved by the scatter), so E = 16 fits the 64-register
// budget of a 1024-thread CTA (the register-resident form spills there).
// CS == 2: each CTA of a 2-CTA cluster sorts its half of the cloud, then both
// merge the two sorted halves (merge path on the unique (key, index) pairs,
// the partner's half read through DSMEM) and each writes NP outputs.
// Clouds up to 65536 points (16-bit indices).
template <int NT, int E, int CS, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    radix_cta_kernel(const float* __restrict__ xyz, long long N, int axis,
                     float* __restrict__ out_xyz, int* __restrict__ out_perm, int only_flagged) {
  constexpr int NW = NT / 32, NP = NT * E;
  static_assert(CS == 1 || CS == 2, "one CTA or a pair");
  static_assert(NP * CS <= 65536, "16-bit indices");
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* kb = smem;                                      // NP keys (exchange, then sorted)
  uint16_t* ib = reinterpret_cast<uint16_t*>(smem + NP);    // [2][NP] indices
  uint32_t* hist = smem + NP + NP;                          // [NW][256]
  uint32_t* wsum = hist + 256 * NW;                         // [NW]
  __shared__ int identity;
  const int rank = CS > 1 ? static_cast<int>(cg::this_cluster().block_rank()) : 0;
  const long long b = blockIdx.x / CS;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  uint32_t* hw = hist + w * 256;
  const float* src = xyz + b * N * 3;
  const int lb = w * 32 * E + lane;  // this thread's first slot (striped)
  const long long gbase = static_cast<long long>(rank) * NP;

  if (only_flagged) {
    // second launch after bucket_sort_kernel: only the clouds it flagged
    // (perm[0] = -1); both CTAs of a pair read the flag before either writes
    const int f = out_perm[b * N];
    if constexpr (CS > 1) cg::this_cluster().sync();
    if (f != -1) return;
  }
  uint32_t key[E], rk[E / 2];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const long long g = gbase + lb + 32 * e;
    key[e] = g < N ? order_key(__ldg(src + 3 * g + axis)) : 0xffffffffu;
    ib[lb + 32 * e] = static_cast<uint16_t>(g);
  }
  int cur = 0;
  for (int shift = 0; shift < 32; shift += 8) {
    for (int i = t; i < 256 * NW; i += NT) hist[i] = 0;
    if (t == 0) identity = 0;
    __syncthreads();
    warp_rank<E>(key, shift, hw, lane, lt_mask, rk);
    __syncthreads();
    if (cta_digit_offsets<NT>(hist, wsum, &identity, NP)) continue;
    const uint16_t* isrc = ib + cur * NP;
    uint16_t* idst = ib + (cur ^ 1) * NP;
    if (CS == 1 && shift == 24) {
      // last pass of a one-CTA cloud: the scatter position is the sorted
      // position -- write the outputs there directly (no shared-memory
      // round trip, no final pass over the buffer)
      float* dst = out_xyz ? out_xyz + b * N * 3 : nullptr;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t dd = (key[e] >> shift) & 255u;
        const uint32_t r = (e & 1) ? rk[e >> 1] >> 16 : rk[e >> 1] & 0xffffu;
        const uint32_t pos = hw[dd] + r;
        if (pos < N) {
          const int from = isrc[lb + 32 * e];
          if (out_perm) out_perm[b * N + pos] = from;
          if (dst) gather_point(src, dst, pos, from);
        }
      }
      return;
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t dd = (key[e] >> shift) & 255u;
      const uint32_t r = (e & 1) ? rk[e >> 1] >> 16 : rk[e >> 1] & 0xffffu;
      const uint32_t pos = hw[dd] + r;
      kb[pos] = key[e];
      idst[pos] = isrc[lb + 32 * e];
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) key[e] = kb[lb + 32 * e];
    cur ^= 1;
  }
  const uint16_t* is = ib + cur * NP;
  float* dst = out_xyz ? out_xyz + b * N * 3 : nullptr;
  if constexpr (CS == 1) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const long long g = lb + 32 * e;
      if (g < N) {
        const int from = is[lb + 32 * e];
        if (out_perm) out_perm[b * N + g] = from;
        if (dst) gather_point(src, dst, g, from);
      }
    }
  } else {
    // The halves hold storage indices [0, NP) and [NP, 2 NP): on equal keys
    // the first half's point comes first, so the merge compares keys only
    // (A wins ties). Each CTA copies the partner's sorted keys next to its
    // own (coalesced DSMEM reads), merges locally, then fetches the chosen
    // indices (the partner's through DSMEM, all loads independent).
    __shared__ int cur_sh;
    uint32_t* kp = hist + 256 * NW + NW;  // NP partner keys
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) kb[lb + 32 * e] = key[e];
    if (t == 0) cur_sh = cur;
    cg::this_cluster().sync();
    const int other = rank ^ 1;
    const uint4* rk4 = reinterpret_cast<const uint4*>(cg::this_cluster().map_shared_rank(kb, other));
    for (int i = t; i < NP / 4; i += NT) reinterpret_cast<uint4*>(kp)[i] = rk4[i];
    const int ocur = *cg::this_cluster().map_shared_rank(&cur_sh, other);
    const uint16_t* iown = ib + cur * NP;
    const uint16_t* ioth = cg::this_cluster().map_shared_rank(ib, other) + ocur * NP;
    const uint32_t* KA = rank == 0 ? kb : kp;
    const uint32_t* KZ = rank == 0 ? kp : kb;
    __syncthreads();
    const int dg = rank * NP + t * E;  // this thread's E outputs (blocked)
    int lo = dg > NP ? dg - NP : 0, hi = dg < NP ? dg : NP;
    while (lo < hi) {  // first i with A[i] after Z[dg - i - 1]
      const int mid = (lo + hi) >> 1;
      if (KA[mid] <= KZ[dg - mid - 1]) lo = mid + 1; else hi = mid;
    }
    int i = lo, j = dg - lo;
    uint32_t from[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const bool take_a = j >= NP || (i < NP && KA[i] <= KZ[j]);
      from[e] = take_a ? static_cast<uint32_t>(i) : (0x10000u | static_cast<uint32_t>(j));
      if (take_a) ++i; else ++j;
    }
    const uint16_t* IA = rank == 0 ? iown : ioth;
    const uint16_t* IZ = rank == 0 ? ioth : iown;
#pragma unroll
    for (int e = 0; e < E; ++e)
      from[e] = (from[e] & 0x10000u) ? IZ[from[e] & 0xffffu] : IA[from[e]];
    cg::this_cluster().sync();  // both CTAs done reading each other: reuse kb as staging
#pragma unroll
    for (int e = 0; e < E; ++e) kb[t * E + e] = from[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int p = lb + 32 * e;
      const long long g = gbase + p;
      if (g < N) {
        const int f = static_cast<int>(kb[p]);
        if (out_perm) out_perm[b * N + g] = f;
        if (dst) gather_point(src, dst, g, f);
      }
    }
  }
}

template <int NT, int E, int CS = 1, int MINB = 1>
cudaError_t launch_radix_cta(const float* xyz, long long batch, long long n, int axis,
                             float* out_xyz, int* out_perm, cudaStream_t st, int only_flagged = 0) {
  constexpr int NW = NT / 32;
  // keys, [2] 16-bit indices, per-warp digit counts, warp sums (+ the
  // partner's keys for the 2-CTA merge)
  const size_t smem = sizeof(uint32_t) * (2 * NT * E + 256 * NW + NW + (CS > 1 ? NT * E : 0));
  auto kern = radix_cta_kernel<NT, E, CS, MINB>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(batch * CS));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, xyz, n, axis, out_xyz, out_perm, only_flagged);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// ------------------------------------------------------ value-bucket sort
// Stable sort of one cloud per CTA without per-digit ranking passes. The
// (order key, storage index) pairs are unique and ordered exactly as the
// stable sort orders the points, so any placement that sorts them is the
// stable order -- no pass needs to be stable itself:
//   1. order keys; the cloud's min / max;
//   2. bucket = a monotone image of the value: fma(v, s, c) with
//      s = nb / (hi - lo), c = 2^23 - lo s, read as an integer (float bits
//      of [2^22, 2^24) are consecutive integers), clamped to [0, nb) -- a
//      correctly rounded fma never reverses an order, so the buckets
//      partition the sorted sequence; each key's slot inside its bucket is
//      the histogram atomicAdd's return value;
//   3. exclusive scan of the counts; scatter (key, index) to
//      start[bucket] + slot (any order inside a bucket);
//   4. each bucket sorted in place by one thread (insertion sort of the
//      pairs: ~1 + nb / N pairs per bucket on average);
//   5. the indices copied out coalesced.
// A bucket larger than `limit` (many equal or clustered keys) would make
// step 4 slow: the CTA flags the cloud (perm[0] = -1) and
// radix_cta_kernel (only_flagged) sorts it in a second launch; so do clouds
// with a non-finite key. Clouds whose keys are all equal take the identity.
// Shared memory: keys 4N | indices 2N | 16-bit bucket starts 2 nb; the
// 32-bit histogram lives in the key region until the scatter overwrites it.
// Clouds < 65536 points (16-bit indices and starts).
__device__ __forceinline__ float key_value(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

template <int NT, int E, bool KEEP, bool QUAD>
__global__ void __launch_bounds__(NT, NT >= 1024 ? (E <= 2 ? 2 : 1) : 1024 / NT) bucket_sort_kernel(const float* __restrict__ xyz,
                                                             long long N, int axis, int nb, int limit,
                                                             float* __restrict__ out_xyz,
                                                             int* __restrict__ out_perm) {
  constexpr int NW = NT / 32;
  // E > 16: the keys do not stay in registers between the histogram and the
  // scatter (1024 threads x 64 registers); the scatter re-reads them (L2)
  constexpr bool kKeep = KEEP;
  extern __shared__ __align__(16) uint32_t smem[];
  const int n = static_cast<int>(N);
  uint32_t* sk = smem;                                                  // n keys
  uint32_t* hist = smem;                                                // nb counts (before the scatter)
  uint16_t* si = reinterpret_cast<uint16_t*>(smem + ((n + 1) & ~1));   // n indices
  uint16_t* st = si + ((n + 1) & ~1);                                   // nb + 1 starts
  __shared__ uint32_t red[3][NW];
  const long long b = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const float* src = xyz + b * N * 3;
  int* perm = out_perm + b * N;
  float* dst = out_xyz ? out_xyz + b * N * 3 : nullptr;

  uint32_t key[E], pk[E];
  uint32_t kmin = 0xffffffffu, kmax = 0u;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int g = t + NT * e;
    key[e] = g < n ? order_key(__ldg(src + 3LL * g + axis)) : 0u;
    if (g < n) {
      kmin = min(kmin, key[e]);
      kmax = max(kmax, key[e]);
    }
  }
  for (int i = t; i < nb; i += NT) hist[i] = 0u;
  kmin = __reduce_min_sync(kFull, kmin);
  kmax = __reduce_max_sync(kFull, kmax);
  if (lane == 0) {
    red[0][w] = kmin;
    red[1][w] = kmax;
  }
  __syncthreads();
  kmin = __reduce_min_sync(kFull, lane < NW ? red[0][lane] : 0xffffffffu);
  kmax = __reduce_max_sync(kFull, lane < NW ? red[1][lane] : 0u);
  if (kmin == kmax) {
    // every key equal: storage order is the stable order
    for (int i = t; i < n; i += NT) {
      perm[i] = i;
      if (dst) gather_point(src, dst, i, i);
    }
    return;
  }
  const float vlo = key_value(kmin), vhi = key_value(kmax);
  const float sc = static_cast<float>(nb) / (vhi - vlo);
  const float c0 = __fsub_rn(8388608.0f, __fmul_rn(vlo, sc));
  const bool finite = isfinite(vlo) && isfinite(vhi) && isfinite(sc) && isfinite(c0);
  auto bucket = [&](uint32_t k) -> int {
    const int q = static_cast<int>(__float_as_uint(__fmaf_rn(key_value(k), sc, c0))) - 0x4B000000;
    return min(max(q, 0), nb - 1);
  };
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int g = t + NT * e;
    pk[e] = 0u;
    if (g < n) {
      const int bk = bucket(key[e]);
      pk[e] = (static_cast<uint32_t>(bk) << 16) | atomicAdd(&hist[bk], 1u);
    }
  }
  __syncthreads();
  // exclusive scan of the counts (thread t owns a contiguous run) and the
  // largest bucket
  const int per = (nb + NT - 1) / NT, i0 = min(t * per, nb), i1 = min(i0 + per, nb);
  uint32_t sum = 0u, big = 0u;
  for (int i = i0; i < i1; ++i) {
    const uint32_t c = hist[i];
    sum += c;
    big = max(big, c);
  }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += v;
  }
  big = __reduce_max_sync(kFull, big);
  if (lane == 31) red[2][w] = inc;
  if (lane == 0) red[0][w] = big;
  __syncthreads();
  uint32_t wb = lane < NW ? red[2][lane] : 0u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(kFull, wb, o);
    if (lane >= o) wb += v;
  }
  big = __reduce_max_sync(kFull, lane < NW ? red[0][lane] : 0u);
  uint32_t run = (w > 0 ? __shfl_sync(kFull, wb, (w - 1) & 31) : 0u) + inc - sum;
  for (int i = i0; i < i1; ++i) {
    st[i] = static_cast<uint16_t>(run);
    run += hist[i];
  }
  if (t == 0) st[nb] = static_cast<uint16_t>(n);
  if (big > static_cast<uint32_t>(limit) || !finite) {
    if constexpr (!QUAD) {
      // radix_cta_kernel sorts this cloud (second launch)
      if (t == 0) perm[0] = -1;
      return;
    } else {
      // small clouds (<= 4 keys per thread): rank every pair against the
      // whole cloud in place of the second launch (n^2 / NT compares per
      // thread, a rare path)
      static_assert(!QUAD || KEEP, "the quadratic fallback keeps the keys in registers");
      __syncthreads();  // the histogram (key region) has been read
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (t + NT * e < n) sk[t + NT * e] = key[e];
      __syncthreads();
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int g = t + NT * e;
        if (g < n) {
          const uint32_t k = key[e];
          uint32_t r = 0u;
#pragma unroll 4
          for (int j = 0; j < n; ++j) {
            const uint32_t kj = sk[j];
            r += (kj < k || (kj == k && j < g)) ? 1u : 0u;
          }
          si[r] = static_cast<uint16_t>(g);
        }
      }
      __syncthreads();
      for (int i = t; i < n; i += NT) {
        const int from = si[i];
        perm[i] = from;
        if (dst) gather_point(src, dst, i, from);
      }
      return;
    }
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int g = t + NT * e;
    if (g < n) {
      const uint32_t k = kKeep ? key[e] : order_key(__ldg(src + 3LL * g + axis));
      const uint32_t pos = st[pk[e] >> 16] + (pk[e] & 0xffffu);
      sk[pos] = k;
      si[pos] = static_cast<uint16_t>(g);
    }
  }
  __syncthreads();
  // rank by position: thread t takes the pairs at positions t + NT e (a
  // warp's lanes mostly share a bucket, so their scans have equal trip
  // counts)
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int p = t + NT * e;
    if (p < n) {
      const uint32_t k = sk[p], g = si[p];
      const int bk = bucket(k);
      const uint32_t beg = st[bk], end = st[bk + 1];
      uint32_t lt = 0u, eq = 0u, j = beg;
#pragma unroll 1
      for (; j + 1u < end; j += 2u) {
        const uint32_t a = sk[j], c = sk[j + 1];
        lt += static_cast<uint32_t>(a < k) + static_cast<uint32_t>(c < k);
        eq += static_cast<uint32_t>(a == k) + static_cast<uint32_t>(c == k);
      }
      if (j < end) {
        const uint32_t a = sk[j];
        lt += static_cast<uint32_t>(a < k);
        eq += static_cast<uint32_t>(a == k);
      }
      if (eq > 1u) {
        // key ties: storage order among them
#pragma unroll 1
        for (uint32_t j = beg; j < end; ++j) lt += (sk[j] == k && si[j] < g) ? 1u : 0u;
      }
      pk[e] = ((beg + lt) << 16) | g;
    }
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (t + NT * e < n) si[pk[e] >> 16] = static_cast<uint16_t>(pk[e] & 0xffffu);
  __syncthreads();
  for (int i = t; i < n; i += NT) {
    const int from = si[i];
    perm[i] = from;
    if (dst) gather_point(src, dst, i, from);
  }
}

template <int NT, int E, bool KEEP = (E <= 16), bool QUAD = false>
cudaError_t launch_bucket_sort(const float* xyz, long long batch, long long n, int axis,
                               float* out_xyz, int* out_perm, cudaStream_t st) {
  // buckets: N / 2 (N / 4 above 16K points) -- more buckets shorten the
  // rank scans but cost more in the histogram and its scan (r02 sweep,
  // 256 clouds: N/1, N/2, N/4 at 8K 0.040 / 0.034 / 0.034 ms, 16K 0.071 /
  // 0.058 / 0.060, 32K - / 0.124 / 0.114)
  const int nb = static_cast<int>(std::max<long long>(1, n > 16384 ? n / 4 : n / 2));
  const size_t smem = sizeof(uint32_t) * ((n + 1) & ~1LL) + sizeof(uint16_t) * (((n + 1) & ~1LL) + nb + 2);
  auto kern = bucket_sort_kernel<NT, E, KEEP, QUAD>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  kern<<<static_cast<unsigned>(batch), NT, smem, st>>>(xyz, n, axis, nb, 96, out_xyz, out_perm);
  return cudaGetLastError();
}

}  // namespace pcsk

namespace pcs_internal {

cudaError_t launch_sort(int coord_dtype, const void* xyz, int64_t batch, int64_t n, int axis,
                        void* out_xyz, int32_t* out_perm, cudaStream_t stream) {
  if (batch <= 0 || n <= 0) return cudaSuccess;
  // On-chip radix (radix_reg_kernel) where it beats the bitonic networks
  // (tools/sort_ab.py on a B200): every cloud of <= 4096 points (256 x 4K:
  // 0.051 -> 0.035 ms), and few larger clouds, spread over a cluster of
  // 2K-point (<= 16 clouds) or 4K-point (<= 37 clouds) CTAs: 4 x 32K 0.133 ->
  // 0.037 ms, 37 x 8K 0.047 -> 0.035 ms. Many large clouds keep the bitonic
  // network (one or two CTAs per cloud, no cross-CTA scatter): 64 x 16K
  // 0.064 vs 0.082, 256 x 32K 0.53 vs 0.63.
  const bool radix_off = !pcs_internal::knobs().sort_radix;

  // clouds of 1K-4K points (and <= 148 smaller ones), permutation
  // requested: the value-bucket sort in 1024-thread CTAs (1-4 keys per
  // thread, two CTAs per SM up to 2 keys; a cloud it cannot bucket falls
  // back to in-CTA all-pairs ranks, no second launch). r02 perm-only vs
  // radix_reg_kernel: 16 x 2K 0.0124 -> 0.0103 ms, 148 x 2K 0.0144 ->
  // 0.0103, 256 x 2K 0.0184 -> 0.0143, 512 x 2K 0.0246 -> 0.0205, 64 x 4K
  // 0.0184 -> 0.0123, 256 x 4K 0.0267 -> 0.0205 (256 x 1K equal: radix)
  if (coord_dtype == PCS_DTYPE_F32 && !radix_off && n <= 4096 && (n > 1024 || batch <= 148) &&
      out_perm && pcs_internal::knobs().sort_bucket) {
    const float* x = static_cast<const float*>(xyz);
    float* o = static_cast<float*>(out_xyz);
    if (n <= 1024) return pcsk::launch_bucket_sort<1024, 1, true, true>(x, batch, n, axis, o, out_perm, stream);
    if (n <= 2048) return pcsk::launch_bucket_sort<1024, 2, true, true>(x, batch, n, axis, o, out_perm, stream);
    return pcsk::launch_bucket_sort<1024, 4, true, true>(x, batch, n, axis, o, out_perm, stream);
  }
  if (coord_dtype == PCS_DTYPE_F32 && !radix_off && (n <= 4096 || (batch <= 37 && n <= 65536))) {
    const float* x = static_cast<const float*>(xyz);
    float* o = static_cast<float*>(out_xyz);
    // <= one CTA per SM of 2K-point clouds: 512 threads x 4 keys (shorter
    // per-warp rank chains) beat 256 x 8 (r02: 1x2048 and 16x2048 0.0143 ->
    // 0.0123 ms; at 148 clouds equal)
    if (n > 1024 && n <= 2048 && batch <= 148)
      return pcsk::launch_radix_reg<512, 4, 1, 2>(x, batch, n, axis, o, out_perm, stream);
    if (n <= 1024) return pcsk::launch_radix_reg<256, 4, 1, 4>(x, batch, n, axis, o, out_perm, stream);
    if (n <= 2048) return pcsk::launch_radix_reg<256, 8, 1, 4>(x, batch, n, axis, o, out_perm, stream);
    if (n <= 4096) return pcsk::launch_radix_reg<512, 8, 1, 2>(x, batch, n, axis, o, out_perm, stream);
    if (batch <= 16 && n <= 32768) {
      if (n <= 8192) return pcsk::launch_radix_reg<256, 8, 4, 4>(x, batch, n, axis, o, out_perm, stream);
      if (n <= 16384) return pcsk::launch_radix_reg<256, 8, 8, 4>(x, batch, n, axis, o, out_perm, stream);
      return pcsk::launch_radix_reg<256, 8, 16, 4>(x, batch, n, axis, o, out_perm, stream);
    }
    if (n <= 8192) return pcsk::launch_radix_reg<512, 8, 2, 2>(x, batch, n, axis, o, out_perm, stream);
    if (n <= 16384) return pcsk::launch_radix_reg<512, 8, 4, 2>(x, batch, n, axis, o, out_perm, stream);
    if (n <= 32768) return pcsk::launch_radix_reg<512, 8, 8, 2>(x, batch, n, axis, o, out_perm, stream);
    return pcsk::launch_radix_reg<512, 8, 16, 2>(x, batch, n, axis, o, out_perm, stream);
  }
  // more clouds (38+) of 4K-32K points, permutation requested: the value-
  // bucket sort, one CTA per cloud (r02 sweep, perm only: 256 x 8K 0.045 ->
  // 0.034 ms, 256 x 16K 0.096 -> 0.058, 256 x 32K 0.242 -> 0.116, 64 x 8K
  // 0.027 -> 0.026; clouds <= 4K stay on radix_reg_kernel: 256 x 2K 0.018
  // vs 0.022 bucketed), then radix_cta_kernel for the clouds it flagged.
  // Without a permutation output, 38+ clouds of <= 32K points: one
  // 16K-point CTA per cloud (or a
  // pair merging their halves), indices in shared memory (radix_cta_kernel).
  // With the leader-atomic ranking it beats the bitonic networks from 38
  // clouds on (perm only, r02 tools/sort_sweep.py: 64x8K 0.035 -> 0.031 ms,
  // 128x16K 0.094 -> 0.051, 48x32K 0.115 -> 0.064, 128x32K 0.223 -> 0.125)
  if (coord_dtype == PCS_DTYPE_F32 && !radix_off && n <= 32768 && out_perm &&
      pcs_internal::knobs().sort_bucket) {
    const float* x = static_cast<const float*>(xyz);
    float* o = static_cast<float*>(out_xyz);
    cudaError_t e;
    // 16 keys per thread (32 above 16K; fewer threads with more keys each
    // measured slower: 256 x 16K 0.058 -> 0.065 ms at 32 per thread)
    // (at most one cloud per SM: 8 keys per thread shorten each CTA's chain,
    // 64 x 8K 0.026 -> 0.022 ms; a full wave keeps 16: 256 x 8K 0.034 vs 0.036)
    if (n <= 8192 && batch <= 148) e = pcsk::launch_bucket_sort<1024, 8>(x, batch, n, axis, o, out_perm, stream);
    else if (n <= 8192) e = pcsk::launch_bucket_sort<512, 16>(x, batch, n, axis, o, out_perm, stream);
    else if (n <= 16384) e = pcsk::launch_bucket_sort<1024, 16>(x, batch, n, axis, o, out_perm, stream);
    else e = pcsk::launch_bucket_sort<1024, 32>(x, batch, n, axis, o, out_perm, stream);
    if (e != cudaSuccess) return e;
    const bool pair = batch * 2 <= 148;
    if (n <= 8192 && pair) return pcsk::launch_radix_cta<256, 16, 2, 4>(x, batch, n, axis, o, out_perm, stream, 1);
    if (n <= 8192) return pcsk::launch_radix_cta<512, 16, 1, 2>(x, batch, n, axis, o, out_perm, stream, 1);
    if (n <= 16384 && pair) return pcsk::launch_radix_cta<512, 16, 2, 2>(x, batch, n, axis, o, out_perm, stream, 1);
    if (n <= 16384) return pcsk::launch_radix_cta<1024, 16, 1, 1>(x, batch, n, axis, o, out_perm, stream, 1);
    return pcsk::launch_radix_cta<1024, 16, 2, 1>(x, batch, n, axis, o, out_perm, stream, 1);
  }
  if (coord_dtype == PCS_DTYPE_F32 && !radix_off && n <= 32768) {
    const float* x = static_cast<const float*>(xyz);
    float* o = static_cast<float*>(out_xyz);
    // at most half a wave of clouds: a CTA pair per cloud (each sorts half,
    // then both merge) puts twice the SMs on the batch (64x8K 0.031 ->
    // 0.027 ms, 64x16K 0.049 -> 0.037)
    const bool pair = batch * 2 <= 148;
    if (n <= 8192 && pair) return pcsk::launch_radix_cta<256, 16, 2, 4>(x, batch, n, axis, o, out_perm, stream);
    if (n <= 8192) return pcsk::launch_radix_cta<512, 16, 1, 2>(x, batch, n, axis, o, out_perm, stream);
    if (n <= 16384 && pair) return pcsk::launch_radix_cta<512, 16, 2, 2>(x, batch, n, axis, o, out_perm, stream);
    if (n <= 16384) return pcsk::launch_radix_cta<1024, 16, 1, 1>(x, batch, n, axis, o, out_perm, stream);
    return pcsk::launch_radix_cta<1024, 16, 2, 1>(x, batch, n, axis, o, out_perm, stream);
  }
  if (coord_dtype == PCS_DTYPE_F32 && n > 1024 && n <= 16384) {
    const float* x = static_cast<const float*>(xyz);
    float* o = static_cast<float*>(out_xyz);
    // few clouds: spread each over a cluster of 2-4 CTAs (the idle SMs
    // shorten each cloud's network); otherwise one CTA per cloud
    const bool spread = true;
    if (spread && n > 4096 && batch * 4 <= 148) {
      if (n <= 8192) return pcsk::launch_reg_sort<2, 4>(x, batch, n, axis, o, out_perm, stream);
      return pcsk::launch_reg_sort<4, 4>(x, batch, n, axis, o, out_perm, stream);
    }
    if (spread && n > 2048 && batch * 2 <= 148) {
      if (n <= 4096) return pcsk::launch_reg_sort<2, 2>(x, batch, n, axis, o, out_perm, stream);
      if (n <= 8192) return pcsk::launch_reg_sort<4, 2>(x, batch, n, axis, o, out_perm, stream);
      return pcsk::launch_reg_sort<8, 2>(x, batch, n, axis, o, out_perm, stream);
    }
    if (n <= 2048) return pcsk::launch_reg_sort<2>(x, batch, n, axis, o, out_perm, stream);
    if (n <= 4096) return pcsk::launch_reg_sort<4>(x, batch, n, axis, o, out_perm, stream);
    if (n <= 8192) return pcsk::launch_reg_sort<8>(x, batch, n, axis, o, out_perm, stream);
    return pcsk::launch_reg_sort<16>(x, batch, n, axis, o, out_perm, stream);
  }
  if (coord_dtype == PCS_DTYPE_F32 && n <= 16384) {
    int npow2 = 1;
    while (npow2 < n) npow2 <<= 1;
    if (npow2 < 2) npow2 = 2;
    const size_t smem = sizeof(unsigned long long) * npow2;
    cudaError_t e = cudaFuncSetAttribute(pcsk::bitonic_sort_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    pcsk::bitonic_sort_kernel<<<static_cast<unsigned>(batch), pcsk::kSortThreads, smem, stream>>>(
        static_cast<const float*>(xyz), n, axis, npow2, static_cast<float*>(out_xyz), out_perm);
    return cudaGetLastError();
  }
  if (coord_dtype == PCS_DTYPE_F32) {
    const float* x = static_cast<const float*>(xyz);
    float* o = static_cast<float*>(out_xyz);
    // register network across a cluster of 16384-word CTAs
    if (n <= 2 * pcsk::kBlk) return pcsk::launch_reg_sort<16, 2>(x, batch, n, axis, o, out_perm, stream);
    if (n <= 4 * pcsk::kBlk) return pcsk::launch_reg_sort<16, 4>(x, batch, n, axis, o, out_perm, stream);
    if (n <= 8 * pcsk::kBlk) return pcsk::launch_reg_sort<16, 8>(x, batch, n, axis, o, out_perm, stream);
    if (n <= 16 * pcsk::kBlk) return pcsk::launch_reg_sort<16, 16>(x, batch, n, axis, o, out_perm, stream);
    return pcsk::launch_device_radix<float, uint32_t>(x, batch, n, axis, o, out_perm, stream);
  }
  if (coord_dtype == PCS_DTYPE_F64 && n >= 65536)
    return pcsk::launch_device_radix<double, uint64_t>(static_cast<const double*>(xyz), batch, n,
                                                       axis, static_cast<double*>(out_xyz),
                                                       out_perm, stream);
  // fp64 keys (drop-in path): LSD radix
  const size_t key_bytes = coord_dtype == PCS_DTYPE_F64 ? 8 : 4;
  const size_t count = static_cast<size_t>(batch) * static_cast<size_t>(n);
  void* ws = nullptr;
  cudaError_t e = pcs_internal::workspace_alloc(reinterpret_cast<void**>(&ws), count * (2 * key_bytes + 8), stream);
  if (e != cudaSuccess) return e;
  char* p = static_cast<char*>(ws);
  void* ka = p;
  void* kb = p + count * key_bytes;
  uint32_t* ia = reinterpret_cast<uint32_t*>(p + 2 * count * key_bytes);
  uint32_t* ib = ia + count;
  if (coord_dtype == PCS_DTYPE_F64)
    pcsk::radix_sort_kernel<double, uint64_t><<<static_cast<unsigned>(batch), pcsk::kSortThreads, 0, stream>>>(
        static_cast<const double*>(xyz), n, axis, static_cast<uint64_t*>(ka),
        static_cast<uint64_t*>(kb), ia, ib, static_cast<double*>(out_xyz), out_perm);
  else
    pcsk::radix_sort_kernel<float, uint32_t><<<static_cast<unsigned>(batch), pcsk::kSortThreads, 0, stream>>>(
        static_cast<const float*>(xyz), n, axis, static_cast<uint32_t*>(ka),
        static_cast<uint32_t*>(kb), ia, ib, static_cast<float*>(out_xyz), out_perm);
  e = cudaGetLastError();
  cudaError_t e2 = cudaFreeAsync(ws, stream);
  return e != cudaSuccess ? e : e2;
}

}  // namespace pcs_internal
