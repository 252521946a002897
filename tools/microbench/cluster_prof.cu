// Per-phase cycle profile of the cluster-spread full-window kernel
// (instrumented build; links the library for the host-side helpers).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DPCS_PROF
//      -I include -I paper_2208_08795_b200/csrc tools/microbench/cluster_prof.cu
//      -L paper_2208_08795_b200/lib -lpcs_gpu -Xlinker -rpath,paper_2208_08795_b200/lib
//      -o tools/microbench/cluster_prof
// usage: cluster_prof N C CS   (one uniform cube cloud, FPS)
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../paper_2208_08795_b200/csrc/cluster_kernels.cu"

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 2048;
  const int C = argc > 2 ? atoi(argv[2]) : 512;
  std::vector<float> h(static_cast<size_t>(N) * 3);
  std::mt19937 rng(1);
  std::uniform_real_distribution<float> u(-1.f, 1.f);
  for (auto& v : h) v = u(rng);
  float* dx;
  long long* di;
  unsigned long long* dst;
  cudaMalloc(&dx, h.size() * 4);
  cudaMalloc(&di, static_cast<size_t>(C) * 8);
  cudaMalloc(&dst, 32);
  cudaMemcpy(dx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  pcsk::SampleParams p{};
  p.xyz = dx; p.f64 = 0; p.B = 1; p.N = N; p.C = C; p.M = 1; p.K = 0;
  p.out_idx = di; p.idx64 = 1; p.stats = dst;
  for (int rep = 0; rep < 3; ++rep) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_cprof, z, sizeof(z));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t e = pcsk::run_cluster_any(p, N, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long r[8];
    cudaMemcpyFromSymbol(r, g_cprof, sizeof(r));
    const double it = static_cast<double>(r[4]);
    printf("N=%d C=%d err=%d ms=%.3f | cycles/iter: update %.0f warp_argmax %.0f send+wait %.0f "
           "reduce %.0f (iters %.0f)\n", N, C, static_cast<int>(e), ms, r[0] / it, r[1] / it,
           r[2] / it, r[3] / it, it);
  }
  return 0;
}
