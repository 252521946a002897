// Full-window FPS / AFPS for batches of few sectors: one sector spread over a
// thread-block cluster of CS CTAs (one SM each) so that each iteration's
// update (sampler.cpp:115-129 over the whole sector) is split CS ways.
//
// A lone 2048-point sector on one SM is issue-bound (r01/r02 ncu: cfg1
// fps_full_kernel<8,8,1>, 1889 warp instructions per iteration at IPC 2.0 =
// ~950 cycles per iteration); spread over 8 SMs each CTA updates 256 points
// and the iteration becomes the exchange latency instead.
//
// Layout: CTA r of the cluster holds the sector's contiguous chunk
// [r*chunk, r*chunk + chunk); thread t of the CTA owns chunk slots k*T + t
// (P slots) with fp64 coordinates and d in registers. Per iteration:
//   update -> per-thread best -> warp (max d, min index) -> every warp
//   st.async's its candidate (key + fp32 coordinates, 32 B) into every CTA's
//   mailbox with mbarrier::complete_tx -> each warp waits on its CTA's
//   mbarrier and reduces the W*CS candidates itself (no CTA barrier, no
//   cluster barrier) -> the winner is the next pivot everywhere.
// Mailboxes are double-buffered by iteration parity: a CTA can only start
// writing round i+2 after receiving every warp's round i+1 message, which
// each warp sends after it has finished reading round i.
//
// Exactness is the full kernel's: keys are (IEEE bits of d, index), the
// reference's value max + first index (sampler.cpp:137-154); when the max is
// 0 (every remaining point coincides with a sample) a second exchange
// picks the lowest unsampled index. fp32 input only (widened exactly).
#include <cooperative_groups.h>

#include "rows_common.cuh"
#include "sampler_common.cuh"

namespace cg = cooperative_groups;

#ifdef PCS_PROF
__device__ unsigned long long g_cprof[8];
#define CPROF_T(v) v = clock64()
#else
#define CPROF_T(v)
#endif

namespace pcsk {

namespace {

struct alignas(16) CMsg {
  uint32_t hi, lo, j, pad;
  float x, y, z, pad2;
};

template <int P, int W, int CS>
__global__ void __launch_bounds__(W * 32) fps_cluster_kernel(const SampleParams p) {
  constexpr int T = W * 32;
  extern __shared__ __align__(16) unsigned char smem[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int rank = static_cast<int>(cg::this_cluster().block_rank());
  const long long flat = static_cast<long long>(blockIdx.x) / CS;  // (cloud, sector)
  const long long b = flat / p.M, s = flat % p.M;
  const SectorGeom g = sector_geom(p.N, p.C, p.M, s);
  const int n = g.n;
  const int chunk = (n + CS - 1) / CS;
  const int lo_r = rank * chunk;
  const int m_r = max(0, min(chunk, n - lo_r));  // points of this CTA

  // shared: fp32 chunk coordinates, mailboxes [2][CS*W], two mbarriers
  float* xs = reinterpret_cast<float*>(smem);
  float* ys = xs + P * T;
  float* zs = ys + P * T;
  CMsg* mbox = reinterpret_cast<CMsg*>(zs + P * T);
  uint64_t* bar = reinterpret_cast<uint64_t*>(mbox + 2 * CS * W);

  const float* cloud = static_cast<const float*>(p.xyz) + b * p.N * 3;
  const int* perm_s = p.perm ? p.perm + b * p.N + g.begin : nullptr;
  auto pt = [&](int j) -> const float* {
    return cloud + 3LL * (perm_s ? static_cast<long long>(__ldg(perm_s + j)) : g.begin + j);
  };
  for (int l = t; l < m_r; l += T) {
    const float* q = pt(lo_r + l);
    xs[l] = __ldg(q);
    ys[l] = __ldg(q + 1);
    zs[l] = __ldg(q + 2);
  }
  if (t == 0) {
    rows::mbar_init(&bar[0], 1);
    rows::mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (p.out_sector && rank == 0)
    for (int i = t; i < g.quota; i += T)
      p.out_sector[b * p.C + g.out_off + i] = static_cast<int>(s + p.sector_base);
  // every CTA's mbarriers exist before any partner can st.async into them
  cg::this_cluster().sync();

  double x[P], y[P], z[P], d[P];
  unsigned vmask = 0;
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const int l = k * T + t;
    const bool valid = l < m_r;
    vmask |= valid ? (1u << k) : 0u;
    // padding slots: NaN coordinates never write (NaN compares false) and
    // d = 0 never wins (best starts at 0 with a strict >)
    const double kNaN = __longlong_as_double(0x7ff8000000000000LL);
    x[k] = valid ? static_cast<double>(xs[l]) : kNaN;
    y[k] = valid ? static_cast<double>(ys[l]) : kNaN;
    z[k] = valid ? static_cast<double>(zs[l]) : kNaN;
    d[k] = valid ? __longlong_as_double(0x7ff0000000000000LL) : 0.0;
  }
  GroupSetup gs;
  gs.b = b;
  gs.s = s;
  gs.g = g;
  int cur = first_point(p, gs);
  double px, py, pz;
  {
    const float* q = pt(cur);
    px = static_cast<double>(__ldg(q));
    py = static_cast<double>(__ldg(q + 1));
    pz = static_cast<double>(__ldg(q + 2));
  }
  auto mark = [&](int c, unsigned& sm) {
    const int l = c - lo_r;
    if (l >= 0 && l < m_r && l % T == t) sm |= 1u << (l / T);
  };
  unsigned smask = 0;
  mark(cur, smask);
  // outputs buffered in rank 0's warp 0 (sample i in lane i % 32)
  const bool writer = rank == 0 && warp == 0;
  const long long obase = b * p.C + g.out_off;
  const long long ioff = g.begin + p.index_base;
  int ob = cur;
  auto flush = [&](int i0, int cnt) {
    if (writer && lane < cnt) {
      if (p.idx64) static_cast<long long*>(p.out_idx)[obase + i0 + lane] = ioff + ob;
      else static_cast<int*>(p.out_idx)[obase + i0 + lane] = static_cast<int>(ioff + ob);
    }
  };
  unsigned writes = 0;
  int round = 0;
  const int nmsg = CS * W;
#ifdef PCS_PROF
  long long c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0;
  unsigned long long pacc[5] = {0, 0, 0, 0, 0};
#endif

  // one cluster-wide (max key, min index) over every warp's candidate; the
  // winner's coordinates ride along
  auto exchange = [&](uint32_t hi, uint32_t lo, uint32_t j, float fx, float fy, float fz,
                      uint32_t& wh, uint32_t& wl, uint32_t& wj, float& wx, float& wy, float& wz) {
    const int buf = round & 1;
    CMsg* mb = mbox + buf * nmsg;
    if (lane < CS) {
      const uint32_t rs = rows::mapa(mb + rank * W + warp, lane);
      const uint32_t rb = rows::mapa(&bar[buf], lane);
      rows::st_async_v4(rs, rb, hi, lo, j, 0u);
      rows::st_async_v4(rs + 16, rb, __float_as_uint(fx), __float_as_uint(fy),
                        __float_as_uint(fz), 0u);
    }
    if (t == 0) rows::mbar_arrive_expect_tx(&bar[buf], nmsg * 32u);
    rows::mbar_wait(&bar[buf], (round >> 1) & 1);
    CPROF_T(c3);
    uint32_t bh = 0u, bl = 0u, bj = kNoIndex;
    float cx = 0.f, cy = 0.f, cz = 0.f;
#pragma unroll
    for (int e0 = 0; e0 < CS * W; e0 += 32) {
      const int e = e0 + lane;
      if (e < nmsg) {
        const uint4 k = *reinterpret_cast<const uint4*>(mb + e);
        const float4 c = *reinterpret_cast<const float4*>(&mb[e].x);
        if (rows::key_gt(k.x, k.y, k.z, bh, bl, bj)) {
          bh = k.x; bl = k.y; bj = k.z; cx = c.x; cy = c.y; cz = c.z;
        }
      }
    }
    uint32_t h2 = bh, l2 = bl, j2 = bj;
    warp_argmax(h2, l2, j2);
    const unsigned who = __ballot_sync(kFull, bh == h2 && bl == l2 && bj == j2);
    const int src = __ffs(who) - 1;
    wh = h2; wl = l2; wj = j2;
    wx = __shfl_sync(kFull, cx, src);
    wy = __shfl_sync(kFull, cy, src);
    wz = __shfl_sync(kFull, cz, src);
    ++round;
  };

  for (int it = 1; it < g.quota; ++it) {
    CPROF_T(c0);
    unsigned long long best = 0;
    int bs = -1;
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const double dist = dist2(x[k], y[k], z[k], px, py, pz);
      const bool lower = dist <= d[k];
      writes += lower ? 1u : 0u;
      d[k] = lower ? dist : d[k];
      const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(d[k]));
      if (bits > best) {
        best = bits;
        bs = k;
      }
    }
    uint32_t hi = static_cast<uint32_t>(best >> 32), lo = static_cast<uint32_t>(best);
    uint32_t j = bs >= 0 ? static_cast<uint32_t>(lo_r + bs * T + t) : kNoIndex;
    CPROF_T(c1);
    warp_argmax(hi, lo, j);
    CPROF_T(c2);
    // the warp winner's coordinates (its chunk slot, broadcast LDS)
    const int wl_ = j != kNoIndex ? static_cast<int>(j) - lo_r : 0;
    uint32_t wh, wlo, wj;
    float fx, fy, fz;
    exchange(hi, lo, j, xs[wl_], ys[wl_], zs[wl_], wh, wlo, wj, fx, fy, fz);
    if ((wh | wlo) == 0u) {
      // every remaining distance is 0: the lowest unsampled index
      uint32_t jm = kNoIndex;
#pragma unroll
      for (int k = P - 1; k >= 0; --k)
        if (((vmask & ~smask) >> k) & 1u) jm = static_cast<uint32_t>(lo_r + k * T + t);
      uint32_t h1 = jm != kNoIndex ? 1u : 0u, l1 = 0u, j1 = jm;
      warp_argmax(h1, l1, j1);
      const int ll = j1 != kNoIndex ? static_cast<int>(j1) - lo_r : 0;
      exchange(h1, l1, j1, xs[ll], ys[ll], zs[ll], wh, wlo, wj, fx, fy, fz);
    }
    CPROF_T(c4);
#ifdef PCS_PROF
    pacc[0] += c1 - c0; pacc[1] += c2 - c1; pacc[2] += c3 - c2; pacc[3] += c4 - c3; pacc[4] += 1;
#endif
    cur = static_cast<int>(wj);
    px = static_cast<double>(fx);
    py = static_cast<double>(fy);
    pz = static_cast<double>(fz);
    mark(cur, smask);
    if (lane == (it & 31)) ob = cur;
    if ((it & 31) == 31) flush(it - 31, 32);
  }
  if (((g.quota - 1) & 31) != 31) flush((g.quota - 1) & ~31, ((g.quota - 1) & 31) + 1);
#ifdef PCS_PROF
  if (t == 0 && rank == 0)
    for (int q = 0; q < 5; ++q) atomicAdd(&g_cprof[q], pacc[q]);
#endif
  // stats: writes from every CTA; the rest once per sector
  const unsigned ws = __reduce_add_sync(kFull, writes);
  if (p.stats) {
    unsigned long long* st = p.stats + b * 4;
    if (lane == 0 && ws) atomicAdd(st + 1, static_cast<unsigned long long>(ws));
    if (rank == 0 && t == 0) {
      const unsigned long long iters = static_cast<unsigned long long>(g.quota - 1);
      atomicAdd(st + 0, iters * static_cast<unsigned long long>(n));
      atomicAdd(st + 2, iters * static_cast<unsigned long long>(n));
      atomicAdd(st + 3, iters);
    }
  }
  // no CTA may exit while a partner can still st.async into its mailbox:
  // every message of the last round has been received by now, but remote
  // arrivals of that round target this CTA's barrier -- wait for all CTAs
  cg::this_cluster().sync();
}

template <int P, int W, int CS>
cudaError_t launch_cluster(SampleParams p, cudaStream_t st) {
  constexpr int T = W * 32;
  const size_t smem = size_t(12) * P * T + 2 * CS * W * sizeof(CMsg) + 2 * sizeof(uint64_t);
  if (plan("fps_cluster_kernel", {P, W, CS})) return cudaSuccess;
  auto kern = fps_cluster_kernel<P, W, CS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  if (CS > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(p.B * p.M * CS));
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int CS>
cudaError_t launch_cluster_p(SampleParams p, long long n, cudaStream_t st) {
  // 4 warps per CTA; slots per thread from the chunk size
  const long long chunk = (n + CS - 1) / CS;
  if (chunk <= 128) return launch_cluster<1, 4, CS>(p, st);
  if (chunk <= 256) return launch_cluster<2, 4, CS>(p, st);
  if (chunk <= 512) return launch_cluster<4, 4, CS>(p, st);
  if (chunk <= 1024) return launch_cluster<8, 4, CS>(p, st);
  return cudaErrorNotSupported;
}

}  // namespace

// Few full-window fp32 sectors of >= 2048 points: the largest cluster (<= 8
// CTAs) that leaves each CTA >= 256 points and the batch on at most half
// the SMs (r02 tools/cluster_ab.py: FPS 1x2048 0.268 -> 0.238 ms at CS=8,
// 1x4096 0.778 -> 0.472, 1x8192 1.516 -> 1.144, AFPS 1x8192 M=4 0.269 ->
// 0.234; 16x2048 at CS=8 no gain, CS=4 0.243; 1024-point sectors slower).
cudaError_t run_cluster_any(SampleParams p, long long n, cudaStream_t st) {
  if (p.f64 || p.trace || p.K > 0 || n < 2048) return cudaErrorNotSupported;
  const long long sectors = p.B * p.M;
  int cs = pcs_internal::knobs().cluster_cs;
  while (cs > 1 && (sectors * cs * 2 > 148 || n < 256LL * cs)) cs >>= 1;
  if (cs < 2) return cudaErrorNotSupported;
  if (cs == 8) return launch_cluster_p<8>(p, n, st);
  if (cs == 4) return launch_cluster_p<4>(p, n, st);
  return launch_cluster_p<2>(p, n, st);
}

}  // namespace pcsk
