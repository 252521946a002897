// Batched sampler entry: picks the kernel family per sector size and window.
#include <algorithm>
#include <initializer_list>

#include "sampler_common.cuh"

namespace pcsk {

// Full-window sectors above kMortonMin take the Morton-row engine first; the
// register-resident full kernel wins below it when the SMs hold few sectors
// (r01: cfg5 FPS 256 x 2K full 0.37 ms vs Morton 0.58 ms; 256 x 4K full 1.70
// vs Morton 1.24 ms). With many sectors (>= 4 per SM) of more than 1024
// points the Morton TMEM form wins already (its CTAs are small: 8 sectors
// of 2K per SM against 2 for the register kernel): AFPS M=16 at 32K 5.13 ->
// 3.18 ms, M=4 at 8K 1.33 -> 1.03 ms.
constexpr long long kMortonMin = 3072;
constexpr long long kMortonMinBusy = 1024;
constexpr long long kBusySectors = 4 * 148;

thread_local std::string* g_plan = nullptr;

std::string kname(const char* base, std::initializer_list<long long> args) {
  std::string s(base);
  s += '<';
  bool first = true;
  for (long long a : args) {
    if (!first) s += ',';
    s += std::to_string(a);
    first = false;
  }
  return s + '>';
}

cudaError_t dispatch(SampleParams p, long long nmax_sector, bool windowed, cudaStream_t st,
                     std::string* msg) {
  p.nmax = static_cast<int>((nmax_sector + 1) & ~1LL);
  const pcs_internal::Knobs& kn = pcs_internal::knobs();
  // PCS_SAMPLER=rows forces the pruned-row engine, =stream the streaming
  // engine (tests, A/B)
  const bool rows = kn.sampler == 1;
  if (kn.sampler == 2) return run_stream_any(p, nmax_sector, st);
  // full-window sectors: Morton rows beyond the register kernels' sweet
  // spot (PCS_MORTON=0 selects the storage-order rows, PCS_MORTON_MIN moves
  // the crossover)
  const bool use_morton = !windowed && kn.morton;
  const long long morton_min = kn.morton_min >= 0 ? kn.morton_min : kMortonMin;
  // fp32 input: the TMEM form first (per-point state in tensor memory, half
  // the shared memory per point); PCS_MORTON_TMEM=0 keeps it in shared memory
  const bool morton_tmem = !p.f64 && kn.morton_tmem;
  auto morton_any = [&]() {
    cudaError_t r = morton_tmem ? run_morton_tmem_any(p, nmax_sector, st) : cudaErrorNotSupported;
    return r == cudaErrorNotSupported ? run_morton_any(p, nmax_sector, st) : r;
  };
  const bool busy = p.B * p.M >= kBusySectors && nmax_sector > kMortonMinBusy && kn.morton_min < 0;
  cudaError_t e = cudaErrorNotSupported;
  // few full-window fp32 sectors (one wave of clusters): each spread over a
  // cluster of up to 8 SMs (cluster_kernels.cu)
  if (!rows) e = run_tiny_any(p, nmax_sector, st);
  if (e == cudaErrorNotSupported && !windowed && !rows && kn.cluster && nmax_sector <= 8192)
    e = run_cluster_any(p, nmax_sector, st);
  if (e == cudaErrorNotSupported && use_morton &&
      (rows || nmax_sector > morton_min || (busy && morton_tmem)))
    e = morton_any();
  // windowed sectors past the TMEM NPDU kernel (> 4096 points, fp32): the
  // TMEM row engine in storage order, rows restricted to the window
  // (PCS_NPDU_BIG=0 keeps the warp / shared-memory row kernels)
  if (e == cudaErrorNotSupported && !rows && windowed && !p.f64 && nmax_sector > 4096 &&
      kn.npdu_big)
    e = run_morton_tmem_any(p, nmax_sector, st);
  if (e == cudaErrorNotSupported && !rows)
    e = windowed ? run_npdu_any(p, nmax_sector, st) : run_full_any(p, nmax_sector, st);
  if (e == cudaErrorNotSupported && use_morton) e = morton_any();
  if (e == cudaErrorNotSupported) e = run_rows_any(p, nmax_sector, windowed, st);
  // beyond every on-chip engine: d[] in global memory (L2), one cooperative
  // launch per sector
  if (e == cudaErrorNotSupported && !rows) e = run_stream_any(p, nmax_sector, st);
  if (e == cudaErrorNotSupported && msg)
    *msg = "sector of " + std::to_string(nmax_sector) + " points: no sampler of this build fits";
  return e;
}

}  // namespace pcsk

namespace pcsk {

// xyz[b, perm[b, i]] -> out[b, i]: the sorted copy, for the engines that
// re-read coordinates from global memory (rows, Morton rows in shared
// memory, streaming) instead of staging them once.
template <typename T>
__global__ void gather_sorted_kernel(const T* __restrict__ xyz, const int* __restrict__ perm,
                                     long long N, long long total, T* __restrict__ out) {
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < total; i += 256LL * gridDim.x) {
    const long long b = i / N;
    const T* q = xyz + 3 * (b * N + __ldg(perm + i));
    out[3 * i] = q[0];
    out[3 * i + 1] = q[1];
    out[3 * i + 2] = q[2];
  }
}

}  // namespace pcsk

namespace pcs_internal {

namespace {

pcsk::SampleParams params_of(const pcs_gpu_args& a, long long* nmax) {
  const bool sectored = a.method == PCS_METHOD_AFPS || a.method == PCS_METHOD_NPDU_AFPS;
  const bool windowed = a.method == PCS_METHOD_NPDU_FPS || a.method == PCS_METHOD_NPDU_AFPS;
  const long long M = sectored ? a.m : 1;
  *nmax = (a.n + M - 1) / M;
  pcsk::SampleParams p{};
  p.xyz = a.xyz;
  p.perm = a.perm;
  p.f64 = a.coord_dtype == PCS_DTYPE_F64;
  p.B = a.batch;
  p.N = a.n;
  p.C = a.c;
  p.M = M;
  // A window that always covers the whole sector is the full update
  // (k >= 2*n-1 => update_window == sector for every pivot), and the
  // OpStats agree: every window then holds the sector's n points.
  p.K = (windowed && a.k < 2 * *nmax - 1) ? a.k : 0;
  p.random_first = a.seed_policy == PCS_RANDOM_FIRST_POINT;
  p.seed = a.seed;
  p.seeds = a.seeds;
  p.out_idx = a.out_indices;
  p.idx64 = a.index_dtype == PCS_INDEX_I64;
  p.out_sector = a.out_sector;
  p.stats = reinterpret_cast<unsigned long long*>(a.out_stats);
  p.index_base = a.index_base;
  p.sector_base = a.sector_base;
  return p;
}

}  // namespace

cudaError_t launch_sample(const pcs_gpu_args& a, cudaStream_t stream, std::string* msg) {
  long long nmax = 0;
  pcsk::SampleParams p = params_of(a, &nmax);
  if (a.out_stats) {
    cudaError_t e = cudaMemsetAsync(a.out_stats, 0, sizeof(uint64_t) * 4 * a.batch, stream);
    if (e != cudaSuccess) return e;
  }
  if (!p.perm) return pcsk::dispatch(p, nmax, p.K > 0, stream, msg);
  // The staging engines gather through the permutation themselves; the
  // engines that re-read coordinates from global memory get a sorted copy.
  std::string fam;
  {
    pcsk::g_plan = &fam;
    const cudaError_t pe = pcsk::dispatch(p, nmax, p.K > 0, nullptr, msg);
    pcsk::g_plan = nullptr;
    if (pe != cudaSuccess) return pe;
  }
  const bool stages = fam.rfind("fps_full_kernel", 0) == 0 || fam.rfind("npdu_", 0) == 0 ||
                      fam.rfind("morton_tmem_kernel", 0) == 0 ||
                      fam.rfind("fps_cluster_kernel", 0) == 0;
  if (stages) return pcsk::dispatch(p, nmax, p.K > 0, stream, msg);
  const size_t csize = p.f64 ? 8 : 4;
  const long long total = p.B * p.N;
  void* ws = nullptr;
  cudaError_t e = workspace_alloc(&ws, csize * 3 * static_cast<size_t>(total), stream);
  if (e != cudaSuccess) return e;
  const unsigned grid = static_cast<unsigned>(std::min<long long>(148 * 8, (total + 255) / 256));
  if (p.f64)
    pcsk::gather_sorted_kernel<double><<<grid, 256, 0, stream>>>(
        static_cast<const double*>(p.xyz), p.perm, p.N, total, static_cast<double*>(ws));
  else
    pcsk::gather_sorted_kernel<float><<<grid, 256, 0, stream>>>(
        static_cast<const float*>(p.xyz), p.perm, p.N, total, static_cast<float*>(ws));
  e = cudaGetLastError();
  p.xyz = ws;
  p.perm = nullptr;
  if (e == cudaSuccess) e = pcsk::dispatch(p, nmax, p.K > 0, stream, msg);
  const cudaError_t e2 = cudaFreeAsync(ws, stream);
  return e != cudaSuccess ? e : e2;
}

int plan_sample(const pcs_gpu_args& a, std::string* name, std::string* msg) {
  long long nmax = 0;
  const pcsk::SampleParams p = params_of(a, &nmax);
  pcsk::g_plan = name;
  const cudaError_t e = pcsk::dispatch(p, nmax, p.K > 0, nullptr, msg);
  pcsk::g_plan = nullptr;
  return e == cudaSuccess ? 0 : -1;
}

cudaError_t launch_local_fps(const double* xyz, int64_t n, int64_t sb, int64_t se,
                             int64_t quota, int64_t k, int random_first, uint64_t seed,
                             int64_t* out_idx, uint64_t* out_stats, double* trace,
                             cudaStream_t stream, std::string* msg) {
  (void)n;
  const long long len = se - sb;
  pcsk::SampleParams p{};
  p.xyz = xyz + 3 * sb;
  p.f64 = 1;
  p.B = 1;
  p.N = len;
  p.C = quota;
  p.M = 1;
  p.K = (k > 0 && k < 2 * len - 1) ? k : 0;
  p.random_first = random_first;
  p.seed = seed;
  p.out_idx = out_idx;
  p.idx64 = 1;
  p.index_base = sb;
  p.stats = reinterpret_cast<unsigned long long*>(out_stats);
  p.trace = trace;
  cudaError_t e = cudaMemsetAsync(out_stats, 0, sizeof(uint64_t) * 4, stream);
  if (e != cudaSuccess) return e;
  return pcsk::dispatch(p, len, p.K > 0, stream, msg);
}

}  // namespace pcs_internal
