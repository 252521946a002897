// Per-phase cycle profile of npdu_wide_kernel (instrumented build, -DPCS_PROF).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DPCS_PROF
//      -I include -I paper_2208_08795_b200/csrc tools/microbench/wide_prof.cu -o tools/microbench/wide_prof
// usage: wide_prof N B M C K   (uniform cube sorted-free, NPDU-AFPS)
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../paper_2208_08795_b200/csrc/full_kernels.cu"

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 32768;
  const int B = argc > 2 ? atoi(argv[2]) : 1;
  const int M = argc > 3 ? atoi(argv[3]) : 32;
  const int C = argc > 4 ? atoi(argv[4]) : 8192;
  const int K = argc > 5 ? atoi(argv[5]) : 129;
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
  p.xyz = dx; p.f64 = 0; p.B = B; p.N = N; p.C = C; p.M = M; p.K = K;
  p.out_idx = di; p.idx64 = 1; p.stats = dst;
  const long long nmax = (N + M - 1) / M;
  p.nmax = static_cast<int>((nmax + 1) & ~1LL);
  for (int rep = 0; rep < 2; ++rep) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_fprof, z, sizeof(z));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t e = pcsk::run_npdu_wide_any(p, nmax, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long r[8];
    cudaMemcpyFromSymbol(r, g_fprof, sizeof(r));
    const double it = static_cast<double>(r[4]);
    printf("N=%d B=%d M=%d C=%d K=%d err=%d ms=%.4f | cycles/iter: slots %.0f warpmax %.0f "
           "exchange %.0f warpmax2 %.0f (iters %.0f)\n",
           N, B, M, C, K, static_cast<int>(e), ms, r[0] / it, r[1] / it, r[2] / it, r[3] / it, it);
  }
  return 0;
}
