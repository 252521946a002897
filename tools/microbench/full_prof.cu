// Per-phase cycle profile of the full-window kernel (instrumented build).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DPCS_PROF
//      -I include -I paper_2208_08795_b200/csrc tools/microbench/full_prof.cu -o tools/microbench/full_prof
// usage: full_prof N B M C   (uniform cube, AFPS with M sectors, C samples)
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../paper_2208_08795_b200/csrc/full_kernels.cu"

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 2048;
  const int B = argc > 2 ? atoi(argv[2]) : 16;
  const int M = argc > 3 ? atoi(argv[3]) : 8;
  const int C = argc > 4 ? atoi(argv[4]) : 512;
  std::vector<float> h(static_cast<size_t>(B) * N * 3);
  std::mt19937 rng(1);
  std::uniform_real_distribution<float> u(-1.f, 1.f);
  for (auto& v : h) v = u(rng);
  float* dx;
  long long* di;
  unsigned long long* dst;
  cudaMalloc(&dx, h.size() * 4);
  cudaMalloc(&di, static_cast<size_t>(B) * C * 8);
  cudaMalloc(&dst, B * 32);
  cudaMemcpy(dx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  pcsk::SampleParams p{};
  p.xyz = dx; p.f64 = 0; p.B = B; p.N = N; p.C = C; p.M = M; p.K = 0;
  p.out_idx = di; p.idx64 = 1; p.stats = dst;
  const long long nmax = (N + M - 1) / M;
  p.nmax = static_cast<int>((nmax + 1) & ~1LL);
  for (int rep = 0; rep < 2; ++rep) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_fprof, z, sizeof(z));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t e = pcsk::run_full_any(p, nmax, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long r[8];
    cudaMemcpyFromSymbol(r, g_fprof, sizeof(r));
    const double it = static_cast<double>(r[3]);
    printf("N=%d B=%d M=%d C=%d err=%d ms=%.3f | cycles/iter: pivot+slots %.0f argmax %.0f tail %.0f\n",
           N, B, M, C, static_cast<int>(e), ms, r[0] / it, r[1] / it, r[2] / it);
  }
  return 0;
}
