// Throughput (whole chip, per-lane Gops) of warp-collective and conversion
// ops: redux.sync, shfl, vote, F2F.F64.F32, and the integer widening path.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kIt = 2048;
__global__ void k_redux(unsigned* o) {
  unsigned a = threadIdx.x, b = a * 3, c = a * 5, d = a * 7;
  for (int i = 0; i < kIt; ++i) {
    a = __reduce_max_sync(0xffffffffu, a) ^ i; b = __reduce_max_sync(0xffffffffu, b) ^ i;
    c = __reduce_min_sync(0xffffffffu, c) ^ i; d = __reduce_min_sync(0xffffffffu, d) ^ i;
  }
  if ((a ^ b ^ c ^ d) == 12345) o[0] = a;
}
__global__ void k_shfl(unsigned* o) {
  unsigned a = threadIdx.x, b = a * 3, c = a * 5, d = a * 7;
  for (int i = 0; i < kIt; ++i) {
    a = __shfl_xor_sync(0xffffffffu, a, 1) ^ i; b = __shfl_xor_sync(0xffffffffu, b, 2) ^ i;
    c = __shfl_xor_sync(0xffffffffu, c, 4) ^ i; d = __shfl_xor_sync(0xffffffffu, d, 8) ^ i;
  }
  if ((a ^ b ^ c ^ d) == 12345) o[0] = a;
}
__global__ void k_vote(unsigned* o) {
  unsigned a = threadIdx.x, b = a * 3, c = a * 5, d = a * 7;
  for (int i = 0; i < kIt; ++i) {
    a = __ballot_sync(0xffffffffu, a & 1) ^ i; b = __ballot_sync(0xffffffffu, b & 2) ^ i;
    c = __ballot_sync(0xffffffffu, c & 4) ^ i; d = __ballot_sync(0xffffffffu, d & 8) ^ i;
  }
  if ((a ^ b ^ c ^ d) == 12345) o[0] = a;
}
__global__ void k_f2f(unsigned* o, float s) {
  float f0 = threadIdx.x, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3; double acc = 0;
  for (int i = 0; i < kIt; ++i) {
    acc += (double)f0; acc += (double)f1; acc += (double)f2; acc += (double)f3;
    f0 += s; f1 += s; f2 += s; f3 += s;
  }
  if (acc == 12345.0) o[0] = 1;
}
// exact float -> double widening with integer ops (normal floats and zero)
__device__ __forceinline__ double widen(float f) {
  const unsigned b = __float_as_uint(f), m = b & 0x7fffffffu;
  const unsigned hi = m ? (((m >> 3) + 0x38000000u) | (b & 0x80000000u)) : (b & 0x80000000u);
  return __hiloint2double(hi, b << 29);
}
__global__ void k_iwiden(unsigned* o, float s) {
  float f0 = threadIdx.x, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3; double acc = 0;
  for (int i = 0; i < kIt; ++i) {
    acc += widen(f0); acc += widen(f1); acc += widen(f2); acc += widen(f3);
    f0 += s; f1 += s; f2 += s; f3 += s;
  }
  if (acc == 12345.0) o[0] = 1;
}
__global__ void k_daddonly(unsigned* o, float s) {
  double f0 = threadIdx.x, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3; double acc = 0;
  for (int i = 0; i < kIt; ++i) {
    acc += f0; acc += f1; acc += f2; acc += f3;
    f0 += s; f1 += s; f2 += s; f3 += s;
  }
  if (acc == 12345.0) o[0] = 1;
}
template <typename K, typename... A>
float tk(K k, A... a) {
  cudaEvent_t x, y; cudaEventCreate(&x); cudaEventCreate(&y);
  k<<<148 * 8, 256>>>(a...); cudaEventRecord(x);
  for (int r = 0; r < 3; ++r) k<<<148 * 8, 256>>>(a...);
  cudaEventRecord(y); cudaEventSynchronize(y); float ms; cudaEventElapsedTime(&ms, x, y); return ms / 3;
}
int main() {
  unsigned* o; cudaMalloc(&o, 64);
  const double ops = 148.0 * 8 * 256 * kIt * 4;
  auto g = [&](float ms) { return ops / (ms * 1e-3) / 1e9; };
  printf("{\"redux_gops\": %.0f, \"shfl_gops\": %.0f, \"vote_gops\": %.0f, \"f2f_plus_dadd_gops\": %.0f, "
         "\"intwiden_plus_dadd_gops\": %.0f, \"dadd_only_gops\": %.0f, \"err\": \"%s\"}\n",
         g(tk(k_redux, o)), g(tk(k_shfl, o)), g(tk(k_vote, o)), g(tk(k_f2f, o, 1.0f)),
         g(tk(k_iwiden, o, 1.0f)), g(tk(k_daddonly, o, 1.0f)), cudaGetErrorString(cudaGetLastError()));
}
