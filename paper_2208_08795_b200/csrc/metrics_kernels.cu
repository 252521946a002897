// Sample-quality metrics on the GPU: the reference's
// coverage_radius and separation (proj/src/metrics.cpp:16-52), batched over
// clouds. Both are O(N * |S|) (O(|S|^2) for separation) exact scans in fp64
// with the reference's squared_dist (proj/include/pcs/point_cloud.hpp:51-56),
// so min / max are exact and the final sqrt is correctly rounded on both
// sides: results are bit-identical to the reference's.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_common.cuh"
#include "internal.h"

namespace pcsk {

constexpr int kMetThreads = 256;
constexpr int kTile = 1024;

template <typename T>
__device__ __forceinline__ void load_point(const T* __restrict__ xyz, long long i, double& x,
                                           double& y, double& z) {
  x = static_cast<double>(xyz[3 * i]);
  y = static_cast<double>(xyz[3 * i + 1]);
  z = static_cast<double>(xyz[3 * i + 2]);
}

template <typename I>
__device__ __forceinline__ long long sample_at(const I* idx, long long b, long long C, long long s) {
  return static_cast<long long>(idx[b * C + s]);
}

// coverage: out_bits[b] = max over points of (min over samples of d^2), as
// IEEE bits (values >= 0 order like their bits); all-ones = index error.
template <typename T, typename I>
__global__ void __launch_bounds__(kMetThreads)
    coverage_kernel(const T* __restrict__ xyz, long long N, const I* __restrict__ idx,
                    long long C, unsigned long long* __restrict__ out_bits) {
  __shared__ double sx[kTile], sy[kTile], sz[kTile];
  __shared__ int bad;
  const long long b = blockIdx.y;
  const T* cloud = xyz + b * N * 3;
  const long long i = static_cast<long long>(blockIdx.x) * kMetThreads + threadIdx.x;
  double px = 0, py = 0, pz = 0;
  if (i < N) load_point(cloud, i, px, py, pz);
  double best = __longlong_as_double(0x7ff0000000000000LL);
  if (threadIdx.x == 0) bad = 0;
  for (long long t0 = 0; t0 < C; t0 += kTile) {
    const int len = static_cast<int>(min(static_cast<long long>(kTile), C - t0));
    __syncthreads();
    for (int s = threadIdx.x; s < len; s += kMetThreads) {
      const long long si = sample_at(idx, b, C, t0 + s);
      if (si < 0 || si >= N) {
        bad = 1;
        sx[s] = sy[s] = sz[s] = 0;
      } else {
        load_point(cloud, si, sx[s], sy[s], sz[s]);
      }
    }
    __syncthreads();
    for (int s = 0; s < len; ++s) best = fmin(best, dist2(px, py, pz, sx[s], sy[s], sz[s]));
  }
  __syncthreads();
  unsigned long long bits = i < N ? static_cast<unsigned long long>(__double_as_longlong(best)) : 0ull;
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(kFull, bits, o);
    bits = v > bits ? v : bits;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out_bits + b, bad ? ~0ull : bits);
}

// separation: out_bits[b] = min over sample pairs (i < j) of d^2.
template <typename T, typename I>
__global__ void __launch_bounds__(kMetThreads)
    separation_kernel(const T* __restrict__ xyz, long long N, const I* __restrict__ idx,
                      long long C, unsigned long long* __restrict__ out_bits) {
  __shared__ double sx[kTile], sy[kTile], sz[kTile];
  const long long b = blockIdx.y;
  const T* cloud = xyz + b * N * 3;
  const long long i = static_cast<long long>(blockIdx.x) * kMetThreads + threadIdx.x;
  double px = 0, py = 0, pz = 0;
  bool ok = i < C;
  if (ok) {
    const long long si = sample_at(idx, b, C, i);
    ok = si >= 0 && si < N;
    if (ok) load_point(cloud, si, px, py, pz);
  }
  double best = __longlong_as_double(0x7ff0000000000000LL);
  // pairs (i, j) with j > i: tiles from this block's first index on
  const long long first = static_cast<long long>(blockIdx.x) * kMetThreads;
  for (long long t0 = first; t0 < C; t0 += kTile) {
    const int len = static_cast<int>(min(static_cast<long long>(kTile), C - t0));
    __syncthreads();
    for (int s = threadIdx.x; s < len; s += kMetThreads) {
      const long long si = sample_at(idx, b, C, t0 + s);
      if (si >= 0 && si < N) load_point(cloud, si, sx[s], sy[s], sz[s]);
      else sx[s] = sy[s] = sz[s] = 0;
    }
    __syncthreads();
    if (ok)
      for (int s = 0; s < len; ++s)
        if (t0 + s > i) best = fmin(best, dist2(px, py, pz, sx[s], sy[s], sz[s]));
  }
  unsigned long long bits = ok ? static_cast<unsigned long long>(__double_as_longlong(best))
                               : 0x7ff0000000000000ull;
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(kFull, bits, o);
    bits = v < bits ? v : bits;
  }
  if ((threadIdx.x & 31) == 0) atomicMin(out_bits + b, bits);
}

__global__ void fill_kernel(unsigned long long* bits, long long B, unsigned long long v) {
  const long long b = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b < B) bits[b] = v;
}

// bits of d^2 -> sqrt(d^2) (correctly rounded, as std::sqrt); index errors
// (all-ones) become NaN.
__global__ void finish_kernel(const unsigned long long* bits, double* out, long long B) {
  const long long b = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b < B)
    out[b] = bits[b] == ~0ull ? __longlong_as_double(0x7ff8000000000000LL)
                              : __dsqrt_rn(__longlong_as_double(static_cast<long long>(bits[b])));
}

template <typename T, typename I>
cudaError_t run_metric(int which, const void* xyz, long long B, long long N, const void* idx,
                       long long C, double* out, cudaStream_t st) {
  unsigned long long* bits = nullptr;
  cudaError_t e = pcs_internal::workspace_alloc(reinterpret_cast<void**>(&bits), sizeof(unsigned long long) * B, st);
  if (e != cudaSuccess) return e;
  // coverage starts at 0 (max), separation at +inf (min)
  fill_kernel<<<static_cast<unsigned>((B + 127) / 128), 128, 0, st>>>(
      bits, B, which == 0 ? 0ull : 0x7ff0000000000000ull);
  e = cudaGetLastError();
  if (e == cudaSuccess) {
    const T* x = static_cast<const T*>(xyz);
    const I* ix = static_cast<const I*>(idx);
    if (which == 0) {
      const dim3 grid(static_cast<unsigned>((N + kMetThreads - 1) / kMetThreads), static_cast<unsigned>(B));
      coverage_kernel<T, I><<<grid, kMetThreads, 0, st>>>(x, N, ix, C, bits);
    } else {
      const dim3 grid(static_cast<unsigned>((C + kMetThreads - 1) / kMetThreads), static_cast<unsigned>(B));
      separation_kernel<T, I><<<grid, kMetThreads, 0, st>>>(x, N, ix, C, bits);
    }
    finish_kernel<<<static_cast<unsigned>((B + 127) / 128), 128, 0, st>>>(bits, out, B);
    e = cudaGetLastError();
  }
  const cudaError_t e2 = cudaFreeAsync(bits, st);
  return e != cudaSuccess ? e : e2;
}

}  // namespace pcsk

namespace pcs_internal {

cudaError_t launch_metric(int which, int coord_dtype, const void* xyz, int64_t batch, int64_t n,
                          int index_dtype, const void* idx, int64_t c, double* out,
                          cudaStream_t stream) {
  if (batch <= 0) return cudaSuccess;
  const bool f64 = coord_dtype == PCS_DTYPE_F64, i64 = index_dtype == PCS_INDEX_I64;
  if (f64 && i64) return pcsk::run_metric<double, long long>(which, xyz, batch, n, idx, c, out, stream);
  if (f64) return pcsk::run_metric<double, int>(which, xyz, batch, n, idx, c, out, stream);
  if (i64) return pcsk::run_metric<float, long long>(which, xyz, batch, n, idx, c, out, stream);
  return pcsk::run_metric<float, int>(which, xyz, batch, n, idx, c, out, stream);
}

}  // namespace pcs_internal
