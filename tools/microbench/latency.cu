// Dependent-chain latencies (cycles/op) of the ops on the sampler's critical
// path, with asm volatile so the chains cannot be folded or hoisted.
#include <cstdio>
#include <cuda_runtime.h>
#define N 256
__device__ __forceinline__ long long clk() { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t) :: "memory"); return t; }
// clock read that cannot issue before `dep` is available
__device__ __forceinline__ long long clkd(double dep) { long long t; asm volatile("{.reg .f64 z; mov.f64 z, %1; mov.u64 %0, %%clock64;}" : "=l"(t) : "d"(dep) : "memory"); return t; }
__device__ __forceinline__ long long clku(unsigned dep) { long long t; asm volatile("{.reg .u32 z; mov.u32 z, %1; mov.u64 %0, %%clock64;}" : "=l"(t) : "r"(dep) : "memory"); return t; }
__global__ void lat(double* dout, long long* cyc, float fin, double din) {
  __shared__ double sd[64];
  __shared__ float sf[64];
  if (threadIdx.x < 64) { sd[threadIdx.x] = 0; sf[threadIdx.x] = 0; }
  __syncwarp();
  double a = din; float f = fin; unsigned u = threadIdx.x; unsigned idx = 0;
  long long t0, t1;
  t0 = clk(); a += (double)(t0 >> 62); for (int i = 0; i < N; ++i) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(a) : "d"(din)); t1 = clkd(a); cyc[0] = t1 - t0; dout[100 + threadIdx.x] = a;
  t0 = clk(); a += (double)(t0 >> 62); for (int i = 0; i < N; ++i) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(a) : "d"(din)); t1 = clkd(a); cyc[1] = t1 - t0; dout[200 + threadIdx.x] = a;
  t0 = clk(); for (int i = 0; i < N; ++i) { asm volatile("cvt.f64.f32 %0, %1;" : "=d"(a) : "f"(f)); asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f) : "d"(a)); } t1 = clk(); cyc[2] = t1 - t0;
  t0 = clk(); for (int i = 0; i < N; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f) : "f"(fin)); t1 = clk(); cyc[3] = t1 - t0;
  t0 = clk(); a += (double)(t0 >> 62); for (int i = 0; i < N; ++i) asm volatile("{.reg .pred p; setp.le.f64 p, %0, %1; selp.f64 %0, %0, %1, p;}" : "+d"(a) : "d"(din)); t1 = clkd(a); cyc[4] = t1 - t0; dout[300 + threadIdx.x] = a;
  t0 = clk(); for (int i = 0; i < N; ++i) asm volatile("redux.sync.max.u32 %0, %0, 0xffffffff;" : "+r"(u)); t1 = clk(); cyc[5] = t1 - t0;
  t0 = clk(); for (int i = 0; i < N; ++i) asm volatile("ld.shared.u32 %0, [%0];" : "+r"(idx)); t1 = clk(); cyc[6] = t1 - t0;
  t0 = clk(); f += (float)(t0 >> 62); for (int i = 0; i < N; ++i) { asm volatile("cvt.f64.f32 %0, %1;" : "=d"(a) : "f"(f)); f = __int_as_float(__float_as_int(f) ^ (int)(__double_as_longlong(a) & 1)); } t1 = clkd(a); cyc[7] = t1 - t0; dout[400 + threadIdx.x] = a;
  t0 = clk(); a += (double)(t0 >> 62); for (int i = 0; i < N; ++i) asm volatile("{.reg .f64 t; cvt.f64.f32 t, %1; add.rn.f64 %0, %0, t;}" : "+d"(a) : "f"(f)); t1 = clkd(a); cyc[8] = t1 - t0;
  dout[threadIdx.x] = a + f + u + idx + sd[0] + sf[0];
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 4096); cudaMalloc(&c, 64 * 8);
  lat<<<1, 32>>>(d, c, 1.5f, 1.0000001); lat<<<1, 32>>>(d, c, 1.5f, 1.0000001);
  long long h[9]; cudaMemcpy(h, c, 72, cudaMemcpyDeviceToHost);
  const char* names[] = {"dadd", "dmul", "f2f_f64_f32_then_f32_f64", "ffma", "dsetp_selp", "redux", "lds32", "f2f_then_xor_dep", "f2f_plus_dadd_dep"};
  printf("{");
  for (int i = 0; i < 9; ++i) printf("\"%s\": %.1f%s", names[i], h[i] / double(N), i < 8 ? ", " : "}\n");
  return 0;
}
