// Second pipe probe: compare/select primitives used by the FPS argmax and
// min-update. Each op is chained per register (8 chains/thread).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int kChains = 8, kIters = 4096;

// DSETP + predicated count only (values do not change -> pure compare cost)
__global__ void k_dsetp(double* out, double c) {
  double a[kChains]; unsigned cnt[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) { a[i] = threadIdx.x * 1e-3 + i; cnt[i] = 0; }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) { cnt[i] += (a[i] <= c); a[i] = __longlong_as_double(__double_as_longlong(a[i]) ^ it); }
  }
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += cnt[i];
  if (s == 12345) out[threadIdx.x] = s;
}
// same loop body but integer u64 compare of the bit patterns
__global__ void k_isetp64(double* out, double c) {
  unsigned long long a[kChains]; unsigned cnt[kChains];
  unsigned long long cc = __double_as_longlong(c);
#pragma unroll
  for (int i = 0; i < kChains; ++i) { a[i] = threadIdx.x * 1000 + i; cnt[i] = 0; }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) { cnt[i] += (a[i] <= cc); a[i] ^= it; }
  }
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += cnt[i];
  if (s == 12345) out[threadIdx.x] = s;
}
// baseline: just the xor + count
__global__ void k_base(double* out, double c) {
  unsigned long long a[kChains]; unsigned cnt[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) { a[i] = threadIdx.x * 1000 + i; cnt[i] = 0; }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) { cnt[i] += (unsigned)a[i]; a[i] ^= it; }
  }
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += cnt[i];
  if (s == 12345) out[threadIdx.x] = s;
}
// fp32 filter body: 3 FADD, FMUL, 2 FFMA, FMUL, FSETP
__global__ void k_filter(float* out, float c) {
  float px = 0.1f, py = 0.2f, pz = 0.3f; unsigned cnt[kChains];
  float x[kChains], y[kChains], z[kChains], dh[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) { x[i] = threadIdx.x * 1e-3f + i; y[i] = x[i] * 0.5f; z[i] = x[i] * 0.25f; dh[i] = 0.5f; cnt[i] = 0; }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      float dx = x[i] - px, dy = y[i] - py, dz = z[i] - pz;
      float d = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, dx * dx));
      cnt[i] += (d * 0.999f > dh[i]);
    }
    px += c; py += c; pz += c;
  }
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += cnt[i];
  if (s == 12345) out[threadIdx.x] = s;
}
// exact fp64 distance from double coords, DSETP min-update and write count
__global__ void k_exact(double* out, double c) {
  double px = 0.1, py = 0.2, pz = 0.3; unsigned cnt = 0;
  double x[kChains], y[kChains], z[kChains], d[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) { x[i] = threadIdx.x * 1e-3 + i; y[i] = x[i] * 0.5; z[i] = x[i] * 0.25; d[i] = 1e30; }
  for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      double dx = __dsub_rn(x[i], px), dy = __dsub_rn(y[i], py), dz = __dsub_rn(z[i], pz);
      double dist = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      bool lower = dist <= d[i]; cnt += lower; d[i] = lower ? dist : d[i];
    }
    px += c; py -= c; pz += c;
  }
  double s = cnt;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += d[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}
// same with u64 integer compare (d >= 0)
__global__ void k_exact_int(double* out, double c) {
  double px = 0.1, py = 0.2, pz = 0.3; unsigned cnt = 0;
  double x[kChains], y[kChains], z[kChains]; unsigned long long d[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) { x[i] = threadIdx.x * 1e-3 + i; y[i] = x[i] * 0.5; z[i] = x[i] * 0.25; d[i] = 0x7ff0000000000000ull; }
  for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      double dx = __dsub_rn(x[i], px), dy = __dsub_rn(y[i], py), dz = __dsub_rn(z[i], pz);
      unsigned long long dist = __double_as_longlong(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
      bool lower = dist <= d[i]; cnt += lower; d[i] = lower ? dist : d[i];
    }
    px += c; py -= c; pz += c;
  }
  double s = cnt;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += __longlong_as_double(d[i]);
  if (s == 12345.678) out[threadIdx.x] = s;
}
template <typename K, typename... A>
float tk(K k, int grid, int block, A... args) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<grid, block>>>(args...); cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<<<grid, block>>>(args...);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / 5;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int block = 256, grid = p.multiProcessorCount * 8;
  double* db; float* fb; cudaMalloc(&db, 1 << 20); cudaMalloc(&fb, 1 << 20);
  const double ops = double(grid) * block * kChains * kIters;
  auto g = [&](float ms, double o) { return o / (ms * 1e-3) / 1e9; };
  float t0 = tk(k_base, grid, block, db, 1.0), t1 = tk(k_dsetp, grid, block, db, 1.0);
  float t2 = tk(k_isetp64, grid, block, db, 1.0), t3 = tk(k_filter, grid, block, fb, 1e-7f);
  float t4 = tk(k_exact, grid, block, db, 1e-9), t5 = tk(k_exact_int, grid, block, db, 1e-9);
  printf("{\"base_xor_count_gops\": %.1f, \"dsetp_body_gops\": %.1f, \"isetp64_body_gops\": %.1f, "
         "\"fp32_filter_pts_g\": %.1f, \"exact_dsetp_pts_g\": %.1f, \"exact_int_pts_g\": %.1f, \"err\": \"%s\"}\n",
         g(t0, ops), g(t1, ops), g(t2, ops), g(t3, ops), g(t4, ops / 4), g(t5, ops / 4),
         cudaGetErrorString(cudaGetLastError()));
}
