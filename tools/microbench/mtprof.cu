// Per-phase cycle profile of the TMEM Morton-row sampler (instrumented build).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DPCS_PROF
//      -I include -I paper_2208_08795_b200/csrc tools/microbench/mtprof.cu -o tools/microbench/mtprof
// usage: mtprof N B   (uniform cube, x-sorted, FPS C = N/4)
#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../paper_2208_08795_b200/csrc/morton_tmem_kernels.cu"

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 8192;
  const int B = argc > 2 ? atoi(argv[2]) : 148;
  std::vector<float> h(static_cast<size_t>(B) * N * 3);
  std::mt19937 rng(1);
  std::uniform_real_distribution<float> u(-1.f, 1.f);
  for (int b = 0; b < B; ++b) {
    std::vector<std::array<float, 3>> pts(N);
    for (auto& q : pts) q = {u(rng), u(rng), u(rng)};
    std::stable_sort(pts.begin(), pts.end(), [](auto& a, auto& c) { return a[0] < c[0]; });
    for (int i = 0; i < N; ++i)
      for (int a = 0; a < 3; ++a) h[(static_cast<size_t>(b) * N + i) * 3 + a] = pts[i][a];
  }
  float* dx;
  long long* di;
  unsigned long long* dst;
  cudaMalloc(&dx, h.size() * 4);
  cudaMalloc(&di, static_cast<size_t>(B) * N / 4 * 8);
  cudaMalloc(&dst, B * 32);
  cudaMemcpy(dx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  pcsk::SampleParams p{};
  p.xyz = dx; p.f64 = 0; p.B = B; p.N = N; p.C = N / 4; p.M = 1; p.K = 0;
  p.out_idx = di; p.idx64 = 1; p.stats = dst;
  for (int rep = 0; rep < 2; ++rep) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_tprof, z, sizeof(z));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t e = pcsk::run_morton_tmem_any(p, N, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long r[8];
    cudaMemcpyFromSymbol(r, g_tprof, sizeof(r));
    const int rows = (N + 31) / 32;
    int CS = 1;
    while ((rows + CS - 1) / CS > 512) CS *= 2;
    const int lr = (rows + CS - 1) / CS;
    const int W = lr <= 128 ? 4 : lr <= 256 ? 8 : 16;
    const double it = static_cast<double>(B) * (N / 4 - 1) * W * CS;  // warp-iterations
    printf("N=%d B=%d CS=%d W=%d err=%d ms=%.3f | cycles per warp-iter: process %.0f warp_red %.0f exch %.0f tail %.0f | cand rows/iter/CTA %.1f pairs/iter/warp %.2f\n",
           N, B, CS, W, static_cast<int>(e), ms, r[0] / it, r[1] / it, r[2] / it, r[3] / it,
           r[4] / (it / W), r[5] / it);
  }
  return 0;
}
