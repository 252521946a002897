// Pipe-throughput microbenchmarks for the FP64 sampler roofline.
// Measures, on the whole chip with CUDA events: DADD, DMUL, DFMA, F2F.F64.F32
// (+DADD), DSETP+SEL, FFMA, 64-bit integer compare+select, and the latency of
// a dependent redux.sync chain. Prints one JSON line.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void k_dadd(double* out, double c) {
  double a[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) a[i] = __dadd_rn(a[i], c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += a[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void k_dmul(double* out, double c) {
  double a[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) a[i] = __dmul_rn(a[i], c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += a[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void k_dfma(double* out, double c) {
  double a[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) a[i] = __fma_rn(a[i], c, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += a[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// F2F.F64.F32 followed by DADD: compare against k_dadd to isolate the convert.
__global__ void k_f2f(double* out, float c) {
  double a[kChains];
  float f[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) { a[i] = 0; f[i] = threadIdx.x * 1e-3f + i; }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) { a[i] = __dadd_rn(a[i], (double)f[i]); f[i] = __fadd_rn(f[i], c); }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += a[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void k_ffma(float* out, float c) {
  float a[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) a[i] = __fmaf_rn(a[i], c, c);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += a[i];
  if (s == 12345.678f) out[threadIdx.x] = s;
}

// min-update as DSETP + 2xSEL, chained per register.
__global__ void k_dmin(double* out, double c) {
  double a[kChains], b[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) { a[i] = threadIdx.x * 1e-3 + i; b[i] = a[i] * 0.5; }
  unsigned cnt = 0;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      const bool lower = b[i] <= a[i];
      cnt += lower;
      a[i] = lower ? b[i] : a[i];
      b[i] = b[i] + c;
    }
  }
  double s = cnt;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += a[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void k_redux_lat(unsigned* out, long long* cycles) {
  unsigned v = threadIdx.x * 2654435761u;
  long long t0 = clock64();
  for (int it = 0; it < 1024; ++it) {
    unsigned m;
    asm volatile("redux.sync.max.u32 %0, %1, 0xffffffff;" : "=r"(m) : "r"(v));
    v = v ^ m ^ it;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cycles[0] = t1 - t0; out[0] = v; }
}

__global__ void k_shfl_lat(unsigned* out, long long* cycles) {
  unsigned v = threadIdx.x * 2654435761u;
  long long t0 = clock64();
  for (int it = 0; it < 1024; ++it) {
    v = __shfl_xor_sync(0xffffffffu, v, 1) + it;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cycles[0] = t1 - t0; out[0] = v; }
}

template <typename K, typename... A>
float time_kernel(K k, int grid, int block, A... args) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<grid, block>>>(args...);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<<<grid, block>>>(args...);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a); cudaEventDestroy(b);
  return ms / 5;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double* dbuf; float* fbuf; unsigned* ubuf; long long* cyc;
  CK(cudaMalloc(&dbuf, 1 << 20)); CK(cudaMalloc(&fbuf, 1 << 20));
  CK(cudaMalloc(&ubuf, 1 << 20)); CK(cudaMalloc(&cyc, 64));
  const int block = 256, grid = sms * 8;
  const double ops = double(grid) * block * kChains * kIters;
  float t_dadd = time_kernel(k_dadd, grid, block, dbuf, 1.0000001);
  float t_dmul = time_kernel(k_dmul, grid, block, dbuf, 1.0000001);
  float t_dfma = time_kernel(k_dfma, grid, block, dbuf, 1.0000001);
  float t_f2f = time_kernel(k_f2f, grid, block, dbuf, 1.0f);
  float t_ffma = time_kernel(k_ffma, grid, block, fbuf, 1.0000001f);
  float t_dmin = time_kernel(k_dmin, grid, block, dbuf, 1e-9);
  CK(cudaDeviceSynchronize());
  k_redux_lat<<<1, 32>>>(ubuf, cyc);
  long long rc = 0; CK(cudaMemcpy(&rc, cyc, 8, cudaMemcpyDeviceToHost));
  k_shfl_lat<<<1, 32>>>(ubuf, cyc);
  long long sc = 0; CK(cudaMemcpy(&sc, cyc, 8, cudaMemcpyDeviceToHost));
  CK(cudaGetLastError());
  auto g = [&](float ms) { return ops / (ms * 1e-3) / 1e9; };  // Gop/s (per-lane ops)
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d, "
         "\"dadd_gops\": %.1f, \"dmul_gops\": %.1f, \"dfma_gops\": %.1f, "
         "\"f2f_plus_dadd_gops\": %.1f, \"ffma_gops\": %.1f, \"dmin_update_gops\": %.1f, "
         "\"redux_dep_cycles\": %.1f, \"shfl_dep_cycles\": %.1f}\n",
         p.name, sms, clk_khz, g(t_dadd), g(t_dmul), g(t_dfma), g(t_f2f), g(t_ffma),
         g(t_dmin), rc / 1024.0, sc / 1024.0);
  return 0;
}
