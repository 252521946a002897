// Per-cloud stable axis sort for sm_100a: the B200 form of pcs::exact_sort
// (proj/src/order.cpp:11-24: std::stable_sort of storage indices by
// points[i][axis] with operator<, then a gather).
//
// Keys: the coordinate's IEEE bits mapped to an order-preserving unsigned
// integer, with -0.0 first folded onto +0.0 (operator< treats them as
// equal, so stability must keep their storage order). NaN is excluded by
// the reference's precondition (proj/src/point_cloud.cpp:43-50).
//
// * fp32, N <= 16384: one CTA per cloud sorts packed (key << 32 | index)
//   words with a bitonic network in shared memory. Packing the storage index
//   into the low bits makes every word unique and orders ties by index, so an
//   unstable network yields exactly the stable order.
// * otherwise (fp64 keys, or larger clouds): one CTA per cloud runs an LSD
//   radix sort, 8-bit digits, over global ping-pong buffers (L2-resident),
//   with tile-ordered ranking (match.any + per-warp digit counts) so every
//   pass is stable. Passes whose digit is constant across the cloud are
//   skipped.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_common.cuh"
#include "internal.h"

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
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < half; i += kSortThreads) {
        const int lo = 2 * j * (i / j) + (i % j), hi = lo + j;
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

}  // namespace pcsk

namespace pcs_internal {

cudaError_t launch_sort(int coord_dtype, const void* xyz, int64_t batch, int64_t n, int axis,
                        void* out_xyz, int32_t* out_perm, cudaStream_t stream) {
  if (batch <= 0 || n <= 0) return cudaSuccess;
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
  const size_t key_bytes = coord_dtype == PCS_DTYPE_F64 ? 8 : 4;
  const size_t count = static_cast<size_t>(batch) * static_cast<size_t>(n);
  void* ws = nullptr;
  cudaError_t e = cudaMallocAsync(&ws, count * (2 * key_bytes + 8), stream);
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
