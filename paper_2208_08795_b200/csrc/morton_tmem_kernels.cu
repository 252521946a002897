// Morton-row sampler with the per-point state in tensor memory (fp32 input,
// full window: FPS / AFPS sectors of 4K-125K points), sm_100a.
//
// The algorithm is morton_rows_kernel's (see morton_kernels.cu): per CTA, the
// points regrouped into rows of 32 Morton-consecutive slots, exact box
// pruning, lazy row keys, warp -> CTA / cluster argmax. What moves: each
// slot's fp64 min-distance d and its sector index live in TMEM -- row r of
// warp w is the column quad (d lo, d hi, index, -) of w's lane quarter, slot
// position = TMEM lane -- and shared memory keeps only the fp32 coordinates
// (12 B per point instead of 24). Consequences: an 8K-point sector fits in
// 96 KB (two clouds per SM instead of one), a 16K-point sector fits one SM
// (no cluster), a 32K-point sector needs a cluster of 2 instead of 4.
//
// TMEM is private to the warp that owns a lane quarter, so every access to a
// row's d/index is made by the row's owner warp; rows are only ever touched
// by their owner (row r -> warp r % W), as in the shared-memory engine.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "internal.h"
#include "rows_common.cuh"
#include "tmem.cuh"

namespace cg = cooperative_groups;

#ifdef PCS_PROF
__device__ unsigned long long g_tprof[8];
#define TPROF_T(v) long long v = clock64()
#else
#define TPROF_T(v)
#endif

namespace pcsk {

using namespace rows;

namespace {

// Z-order cells of ~8 points for the slot bucketing: 2^bits cells, 32 to
// 4096 (a multiple of 32 for the one-warp scan)
#ifndef MORTON_CELL_PTS
#define MORTON_CELL_PTS 8
#endif
__host__ __device__ __forceinline__ int morton_cell_bits(int np) {
  int b = 5;
  while (b < 12 && (1 << b) * MORTON_CELL_PTS < np) ++b;
  return b;
}

// four-row update steps for 4-warp CTAs with 3+ candidate rows (A/B: -DMORTON_QUAD=0)
#ifndef MORTON_QUAD
#define MORTON_QUAD 1
#endif
constexpr bool kQuadRows = MORTON_QUAD != 0;


__device__ __forceinline__ void tm_row_ld(uint32_t a, double& d, uint32_t& orig) {
  uint32_t r[4];
  tm_ld(a, r);
  tm_wait_ld();
  d = __hiloint2double(static_cast<int>(r[1]), static_cast<int>(r[0]));
  orig = r[2];
}

}  // namespace

// Slot i (row i / 32, position i % 32) -- rows interleaved over warps: local
// row r belongs to warp r % W as its row l = r / W, stored at TMEM columns
// tm + 4l .. 4l+3 of the warp's quarter. One row per lane for the row
// metadata (box, max high word), as in the shared-memory engine.
// WIN (NPDU variants, update_window, proj/src/sectors.cpp:53-61): slots
// keep storage order (windows are storage ranges) and only rows meeting the
// window are candidates; the rest of the engine is unchanged.
template <int W, int CS, bool WIN>
__global__ void __launch_bounds__(W * 32) morton_tmem_kernel(const SampleParams p, int tm_cols) {
  static_assert(W % 4 == 0, "whole lane quarters");
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t tm_base_sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int T = W * 32;
  const bool dense = gridDim.x >= 148u;  // a CTA or more per SM
  const int rank = CS > 1 ? static_cast<int>(cg::this_cluster().block_rank()) : 0;
  const long long flat = static_cast<long long>(blockIdx.x) / CS;
  const long long b = flat / p.M, s = flat % p.M;
  const SectorGeom g = sector_geom(p.N, p.C, p.M, s);
  const int n = g.n;
  const int srows = (n + 31) >> 5;
  const int srows_local = srows > rank ? (srows - rank + CS - 1) / CS : 0;
  const int np = p.nmax;  // slot capacity: rows_cap * 32, rows_cap = W * rpw
  const int rpw = (np >> 5) / W;  // rows per warp (capacity)
  float* xs = reinterpret_cast<float*>(smem);
  float* ys = xs + np;
  float* zs = ys + np;
  unsigned* sampled = reinterpret_cast<unsigned*>(zs + np);
  uint4* cand = reinterpret_cast<uint4*>(sampled + (np >> 5) + 4 - ((np >> 5) & 3));
  Msg* xbuf = reinterpret_cast<Msg*>(cand + 2 * W);                               // [2][CS * W]
  uint64_t* xbar = reinterpret_cast<uint64_t*>(xbuf + (CS > 1 ? 2 * CS * W : 0));  // [2]
  int* scratch = reinterpret_cast<int*>(xbar + 2);                                 // [8]
  uint32_t* hist = reinterpret_cast<uint32_t*>(scratch + 8);  // [1 << morton_cell_bits]
  if (p.f64) __trap();
  auto to_sector = [&](int jl) { return (((jl >> 5) * CS + rank) << 5) + (jl & 31); };

  if (warp == 0) tm_alloc(&tm_base_sh, tm_cols);
  if (threadIdx.x < 6) scratch[threadIdx.x] = (threadIdx.x & 1) ? INT_MIN : INT_MAX;
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tm = tm_base_sh + ((static_cast<uint32_t>(warp & 3) * 32u) << 16) +
                      static_cast<uint32_t>((warp >> 2) * 4 * rpw);
  int held = 0;
  if (srows_local > 0) {
    const int last_R = (srows_local - 1) * CS + rank;
    held = (srows_local - 1) * 32 + min(32, n - last_R * 32);
  }
  // sector point j: storage order, or through the sort permutation
  const float* cloud_b = static_cast<const float*>(p.xyz) + b * p.N * 3;
  const int* perm_s = p.perm ? p.perm + b * p.N + g.begin : nullptr;
  auto pt = [&](long long j) -> const float* {
    return cloud_b + 3LL * (perm_s ? static_cast<long long>(__ldg(perm_s + j)) : g.begin + j);
  };

  // ---- 1. bounding box of the CTA's points (read from global / L2)
  {
    float x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY, z0 = INFINITY,
          z1 = -INFINITY;
    for (int jl = threadIdx.x; jl < np; jl += T) {
      const int gj = to_sector(jl);
      if ((jl >> 5) < srows_local && gj < n) {
        const float* q = pt(gj);
        const float x = q[0], y = q[1], z = q[2];
        x0 = fminf(x0, x); x1 = fmaxf(x1, x);
        y0 = fminf(y0, y); y1 = fmaxf(y1, y);
        z0 = fminf(z0, z); z1 = fmaxf(z1, z);
      }
    }
    const int v[6] = {f2ord(x0), f2ord(x1), f2ord(y0), f2ord(y1), f2ord(z0), f2ord(z1)};
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      const int r = (a & 1) ? __reduce_max_sync(kFull, v[a]) : __reduce_min_sync(kFull, v[a]);
      if (lane == 0) {
        if (a & 1) atomicMax(&scratch[a], r);
        else atomicMin(&scratch[a], r);
      }
    }
  }
  __syncthreads();
  // ---- 2./3. slot order: storage order (WIN) or a Z-order bucketing --
  //         counting sort of the points by the top bits of their Morton
  //         code (cells of ~8 points; order inside a cell is whatever the
  //         shared-memory atomics give -- any order is exact, only the row
  //         boxes' compactness depends on it)
  uint32_t* src_slot = reinterpret_cast<uint32_t*>(zs);
  if constexpr (WIN) {
    for (int i = threadIdx.x; i < np; i += T) src_slot[i] = static_cast<uint32_t>(i);
  } else {
    const int cb = morton_cell_bits(np);
    const int cells = 1 << cb;
    uint32_t* rank_of = reinterpret_cast<uint32_t*>(xs);
    uint32_t* cell_of = reinterpret_cast<uint32_t*>(ys);
    for (int i = threadIdx.x; i < cells; i += T) hist[i] = 0u;
    __syncthreads();
    const float bx0 = ord2f(scratch[0]), by0 = ord2f(scratch[2]), bz0 = ord2f(scratch[4]);
    const float ext = fmaxf(fmaxf(ord2f(scratch[1]) - bx0, ord2f(scratch[3]) - by0),
                            ord2f(scratch[5]) - bz0);
    const float sc = (ext > 0.f && ext < INFINITY) ? 1023.0f / ext : 0.f;
    for (int jl = threadIdx.x; jl < np; jl += T) {
      const int gj = to_sector(jl);
      uint32_t cell = kNoIndex;
      if ((jl >> 5) < srows_local && gj < n) {
        const float* q = pt(gj);
        auto qz = [&](float c, float c0) {
          const float t = fminf(fmaxf((c - c0) * sc, 0.f), 1023.f);
          return spread3(static_cast<uint32_t>(t));
        };
        const uint32_t code = qz(q[0], bx0) | (qz(q[1], by0) << 1) | (qz(q[2], bz0) << 2);
        cell = code >> (30 - cb);
        rank_of[jl] = atomicAdd(&hist[cell], 1u);
      }
      cell_of[jl] = cell;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the cell counts (cells / 32 per lane)
      const int per = cells >> 5;
      uint32_t sum = 0;
      for (int i = 0; i < per; ++i) sum += hist[lane * per + i];
      uint32_t x = sum;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, off);
        if (lane >= off) x += y;
      }
      uint32_t run = x - sum;
      for (int i = 0; i < per; ++i) {
        const uint32_t c = hist[lane * per + i];
        hist[lane * per + i] = run;
        run += c;
      }
    }
    __syncthreads();
    for (int jl = threadIdx.x; jl < np; jl += T) {
      const uint32_t cell = cell_of[jl];
      if (cell != kNoIndex) src_slot[hist[cell] + rank_of[jl]] = static_cast<uint32_t>(jl);
    }
  }
  __syncthreads();
  // ---- 4. each warp gathers its rows' coordinates (from L2) and writes
  //         d / index to TMEM
  {
    for (int l = 0; l < rpw; ++l) {
      const int i = ((warp + W * l) << 5) + lane;
      const uint32_t jl = src_slot[i];
      const bool valid = i < held;
      float x = 0.f, y = 0.f, z = 0.f;
      uint32_t o = kNoIndex;
      if (valid) {
        const int gj = to_sector(static_cast<int>(jl));
        const float* q = pt(gj);
        x = q[0]; y = q[1]; z = q[2];
        o = static_cast<uint32_t>(gj);
      }
      xs[i] = x; ys[i] = y; zs[i] = z;  // zs[i] overwrites src_slot[i]: same thread
      const uint32_t w4[4] = {0u, valid ? 0x7ff00000u : 0u, o, 0u};  // d = +inf / 0
      tm_st(tm + 4 * l, w4);
    }
    tm_wait_st();
  }
  for (int w = threadIdx.x; w < (np >> 5); w += T) sampled[w] = 0u;
  if (p.out_sector && rank == 0)
    for (int i = threadIdx.x; i < g.quota; i += T)
      p.out_sector[b * p.C + g.out_off + i] = static_cast<int>(s + p.sector_base);
  bool sub_local = false;
  if (CS > 1 && threadIdx.x == 0) {
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < held; i += T)
    sub_local |= is_subnormal_f32(xs[i]) || is_subnormal_f32(ys[i]) || is_subnormal_f32(zs[i]);
  const bool any_sub = __syncthreads_or(sub_local) != 0;
  if constexpr (CS > 1) cg::this_cluster().sync();

  // ---- 5. per-lane row metadata: box + exact max of the high words
  const int rows = (held + 31) >> 5;
  const int r = warp + W * lane;  // this lane's row (the warp's row l = lane)
  float bx0, bx1, by0, by1, bz0, bz1;
  uint32_t rmh;
  {
    float x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY, z0 = INFINITY,
          z1 = -INFINITY;
    if (r < rows) {
      const int e = min(32, held - r * 32);
      for (int q = 0; q < e; ++q) {
        const int i = r * 32 + q;
        x0 = fminf(x0, xs[i]); x1 = fmaxf(x1, xs[i]);
        y0 = fminf(y0, ys[i]); y1 = fmaxf(y1, ys[i]);
        z0 = fminf(z0, zs[i]); z1 = fmaxf(z1, zs[i]);
      }
    }
    bx0 = x0; bx1 = x1; by0 = y0; by1 = y1; bz0 = z0; bz1 = z1;
    rmh = r < rows ? kInfHi : 0u;
  }

  GroupSetup gs;
  gs.b = b;
  gs.s = s;
  gs.g = g;
  int cur = first_point(p, gs);  // sector-local
  const float* pc = pt(cur);
  float pfx = pc[0], pfy = pc[1], pfz = pc[2];
  double px = pfx, py = pfy, pz = pfz;
  const long long out_base = b * p.C + g.out_off;
  const long long index_off = g.begin + p.index_base;
  if (rank == 0 && threadIdx.x == 0) {
    if (p.idx64) static_cast<long long*>(p.out_idx)[out_base] = index_off + cur;
    else static_cast<int*>(p.out_idx)[out_base] = static_cast<int>(index_off + cur);
  }
  for (int l = 0; l < rpw; ++l) {  // mark the first point (its unique slot)
    double dv;
    uint32_t o;
    tm_row_ld(tm + 4 * l, dv, o);
    const int i = ((warp + W * l) << 5) + lane;
    if (o == static_cast<uint32_t>(cur)) sampled[i >> 5] |= 1u << (i & 31);
  }
  unsigned writes = 0;
  int round = 0;
#ifdef PCS_PROF
  unsigned long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif

  const long long K = p.K;
  const int half_down = static_cast<int>(K / 2), half_up = static_cast<int>((K + 1) / 2);
  unsigned long long evals = 0;
  auto iterate = [&](auto f2f_tag) {
  constexpr bool F2F = decltype(f2f_tag)::value;
  for (int it = 1; it < g.quota; ++it) {
    TPROF_T(t0);
    [[maybe_unused]] int wb = 0, we = n;
    if constexpr (WIN) {
      wb = cur >= half_down ? cur - half_down : 0;
      we = min(n, cur + half_up);
      evals += static_cast<unsigned long long>(we - wb);
    }
    bool need = r < rows;
    if constexpr (WIN) {
      const int R = r * CS + rank;  // this lane's row in sector order
      need = need && (R << 5) < we && (R << 5) + 32 > wb;
    }
    if (need) {
      const float lb = __fadd_rd(__fadd_rd(gap2(bx0, bx1, pfx, pfx), gap2(by0, by1, pfy, pfy)),
                                 gap2(bz0, bz1, pfz, pfz));
      need = !(f32_as_f64_hi_lb(__fmul_rd(lb, 0.99999904f)) > rmh);
    }
    unsigned todo = __ballot_sync(kFull, need);
#ifdef PCS_PROF
    pacc[4] += __popc(todo);
#endif
    tm_wait_st();  // last iteration's row stores land before rows are re-read
    // candidate rows, NR per step (independent distance chains overlap).
    // 4-warp CTAs (many rows per warp) take 3+ candidates four at a time
    // (AFPS M=16 at 32K 2.98 -> 2.92 ms, M=4 at 8K 1.094 -> 1.067); with 8 or
    // 16 warps the four-row step measured 3-7% slower
    // (profiles/r02_morton_quad_ab.log). Missing rows repeat the first one
    // and store its final value again
    auto update_rows = [&](auto nr_tag) {
      constexpr int NR = decltype(nr_tag)::value;
      int l[NR];
      l[0] = __ffs(todo) - 1;
      todo &= todo - 1;
#pragma unroll
      for (int q = 1; q < NR; ++q) {
        l[q] = todo ? __ffs(todo) - 1 : l[0];
        todo &= todo - 1;
      }
      uint32_t r4[NR][4];
#pragma unroll
      for (int q = 0; q < NR; ++q) tm_ld(tm + 4 * l[q], r4[q]);
      double e[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const int j = ((warp + W * l[q]) << 5) + lane;
        e[q] = dist2(to_f64<F2F>(xs[j]), to_f64<F2F>(ys[j]), to_f64<F2F>(zs[j]), px, py, pz);
      }
      tm_wait_ld();
      double d[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        d[q] = __hiloint2double(static_cast<int>(r4[q][1]), static_cast<int>(r4[q][0]));
        bool w = (q == 0 || l[q] != l[0]) && r4[q][2] != kNoIndex && e[q] <= d[q];
        if constexpr (WIN)
          w = w && static_cast<int>(r4[q][2]) >= wb && static_cast<int>(r4[q][2]) < we;
        writes += w ? 1u : 0u;
        d[q] = w ? e[q] : d[q];
      }
#pragma unroll
      for (int q = 1; q < NR; ++q) d[q] = l[q] == l[0] ? d[0] : d[q];
      uint32_t h[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const uint32_t sd[2] = {static_cast<uint32_t>(__double2loint(d[q])),
                                static_cast<uint32_t>(__double2hiint(d[q]))};
        tm_st(tm + 4 * l[q], sd);
        h[q] = __reduce_max_sync(kFull, sd[1]);
      }
#pragma unroll
      for (int q = NR - 1; q >= 0; --q)
        if (lane == l[q]) rmh = h[q];
    };
    while (todo) {
#ifdef PCS_PROF
      pacc[5] += 1;
#endif
      if (kQuadRows && (W == 4 || (W == 8 && dense)) && __popc(todo) > 2) update_rows(std::integral_constant<int, 4>{});
      else update_rows(std::integral_constant<int, 2>{});
    }
    tm_wait_st();
    TPROF_T(t1);
    // warp argmax: rows with the largest high word, exact key from TMEM
    uint32_t hi = __reduce_max_sync(kFull, rmh), lo = 0u, j = kNoIndex, pos = 0u;
    {
      unsigned tied = __ballot_sync(kFull, r < rows && rmh == hi);
      while (tied) {
        const int L = __ffs(tied) - 1;
        tied &= tied - 1;
        double dv;
        uint32_t o;
        tm_row_ld(tm + 4 * L, dv, o);
        const uint32_t h0 = static_cast<uint32_t>(__double2hiint(dv));
        const uint32_t l0 = static_cast<uint32_t>(__double2loint(dv));
        const uint32_t l = __reduce_max_sync(kFull, h0 == hi ? l0 : 0u);
        const uint32_t m = __reduce_min_sync(
            kFull, (h0 == hi && l0 == l && o != kNoIndex) ? (o << 5) | lane : kNoIndex);
        if (l > lo || (l == lo && m < j)) {
          lo = l; j = m; pos = (static_cast<uint32_t>(warp + W * L) << 5) | (m & 31u);
        }
      }
      j = j == kNoIndex ? kNoIndex : j >> 5;
    }
    TPROF_T(t2);
    auto take_local = [&](uint32_t i) {
      pfx = xs[i]; pfy = ys[i]; pfz = zs[i];
      px = to_f64<F2F>(pfx); py = to_f64<F2F>(pfy); pz = to_f64<F2F>(pfz);
    };
    constexpr unsigned kMsg = 32u;
    auto exchange = [&](uint32_t h, uint32_t l, uint32_t jj, uint32_t at, bool& mine_out) {
      Msg* mb = xbuf + (round & 1) * (CS * W);
      if (lane < CS) {
        const int i = jj == kNoIndex ? 0 : static_cast<int>(at);
        const uint32_t rs = mapa(mb + rank * W + warp, lane), rb = mapa(&xbar[round & 1], lane);
        st_async_v4(rs, rb, h, l, jj, at);
        st_async_v4(rs + 16, rb, __float_as_uint(xs[i]), __float_as_uint(ys[i]),
                    __float_as_uint(zs[i]), 0u);
      }
      if (threadIdx.x == 0) mbar_arrive_expect_tx(&xbar[round & 1], CS * W * kMsg);
      mbar_wait(&xbar[round & 1], (round >> 1) & 1);
      uint32_t bh = 0u, bl = 0u, bj = kNoIndex;
      int be = 0;
#pragma unroll
      for (int e0 = 0; e0 < CS * W; e0 += 32) {
        const int e = e0 + lane;
        if (e < CS * W) {
          const uint4 k = *reinterpret_cast<const uint4*>(mb + e);
          if (key_gt(k.x, k.y, k.z, bh, bl, bj)) { bh = k.x; bl = k.y; bj = k.z; be = e; }
        }
      }
      uint32_t h2 = bh, l2 = bl, j2 = bj;
      warp_argmax(h2, l2, j2);
      const unsigned who = __ballot_sync(kFull, bh == h2 && bl == l2 && bj == j2);
      const int e = __shfl_sync(kFull, be, __ffs(who) - 1);
      const Msg& w = mb[e];
      pfx = __uint_as_float(w.c[0]); pfy = __uint_as_float(w.c[1]); pfz = __uint_as_float(w.c[2]);
      px = to_f64<F2F>(pfx); py = to_f64<F2F>(pfy); pz = to_f64<F2F>(pfz);
      mine_out = e / W == rank;
      pos = w.pos;
      hi = h2; lo = l2; j = j2;
      ++round;
    };
    bool mine = true;
    if constexpr (CS > 1) {
      exchange(hi, lo, j, pos, mine);
    } else {
      uint4* buf = cand + (round & 1) * W;
      if (lane == 0) buf[warp] = make_uint4(hi, lo, j, pos);
      __syncthreads();
      const uint4 v = lane < W ? buf[lane] : make_uint4(0, 0, kNoIndex, 0);
      hi = v.x; lo = v.y; j = v.z;
      warp_argmax(hi, lo, j);
      const unsigned who = __ballot_sync(kFull, lane < W && v.x == hi && v.y == lo && v.z == j);
      pos = buf[who ? __ffs(who) - 1 : 0].w;
      ++round;
      if ((hi | lo) != 0u) take_local(pos);
    }
    TPROF_T(t3);
    if ((hi | lo) == 0u) {
      // every distance is 0: lowest unsampled index (sampler.cpp:148-154);
      // each warp scans its own rows, then the CTA combines
      uint32_t jm = kNoIndex, at = 0u;
      for (int l = 0; l < rpw; ++l) {
        double dv;
        uint32_t o;
        tm_row_ld(tm + 4 * l, dv, o);
        const int i = ((warp + W * l) << 5) + lane;
        const bool free_slot = i < held && !((sampled[i >> 5] >> (i & 31)) & 1u);
        if (free_slot && o < jm) { jm = o; at = static_cast<uint32_t>(i); }
      }
      const uint32_t wm = __reduce_min_sync(kFull, jm);
      const unsigned who = __ballot_sync(kFull, jm == wm);
      at = __shfl_sync(kFull, at, __ffs(who) - 1);
      uint4* buf = cand + (round & 1) * W;
      if (lane == 0) buf[warp] = make_uint4(wm, at, 0, 0);
      __syncthreads();
      const uint4 v = lane < W ? buf[lane] : make_uint4(kNoIndex, 0, 0, 0);
      jm = __reduce_min_sync(kFull, v.x);
      const unsigned who2 = __ballot_sync(kFull, lane < W && v.x == jm);
      at = __shfl_sync(kFull, v.y, __ffs(who2) - 1);
      ++round;
      if constexpr (CS > 1) {
        exchange(jm != kNoIndex ? 1u : 0u, 0u, jm, at, mine);
      } else {
        j = jm;
        pos = at;
        take_local(at);
      }
    }
    cur = static_cast<int>(j);
    if (rank == 0 && threadIdx.x == 0) {
      if (p.idx64) static_cast<long long*>(p.out_idx)[out_base + it] = index_off + cur;
      else static_cast<int*>(p.out_idx)[out_base + it] = static_cast<int>(index_off + cur);
    }
    if (mine && threadIdx.x == 0) sampled[pos >> 5] |= 1u << (pos & 31);
#ifdef PCS_PROF
    TPROF_T(t4);
    pacc[0] += t1 - t0; pacc[1] += t2 - t1; pacc[2] += t3 - t2; pacc[3] += t4 - t3;
#endif
  }
  };
  // fp32 -> fp64 of the candidate rows' coordinates: F2F (XU pipe; always
  // exact) or integer widening (exact without subnormals). r02 s4 A/B
  // (profiles/r02_morton_f2f_ab.log): F2F is faster in 16-warp CTAs (FPS 16K
  // 6.94 -> 6.38 ms, 32K 34.7 -> 31.8) and in 4-warp CTAs (AFPS M=16 at 32K
  // 2.91 -> 2.49); 8-warp CTAs take it, with four-row steps, when every SM
  // has a CTA (`dense`: FPS 8K 2.11 -> 2.02, 4K 1.06 -> 1.03) and keep the
  // integer form and row pairs below that (cfg3 FPS, 64 CTAs: 1.49 vs 1.53)
  if (any_sub || W != 8 || dense)
    iterate(std::true_type{});
  else
    iterate(std::false_type{});
#ifdef PCS_PROF
  if (lane == 0)
    for (int q = 0; q < 6; ++q) atomicAdd(&g_tprof[q], pacc[q]);
#endif
  const unsigned ws = __reduce_add_sync(kFull, writes);
  if (p.stats) {
    unsigned long long* st = p.stats + b * 4;
    if (lane == 0 && ws) atomicAdd(st + 1, static_cast<unsigned long long>(ws));
    if (rank == 0 && threadIdx.x == 0) {
      const unsigned long long iters = static_cast<unsigned long long>(g.quota - 1);
      atomicAdd(st + 0, WIN ? evals : iters * static_cast<unsigned long long>(n));
      atomicAdd(st + 2, iters * static_cast<unsigned long long>(n));
      atomicAdd(st + 3, iters);
    }
  }
  tm_wait_st();
  tm_fence_before();
  __syncthreads();
  if (warp == 0) tm_dealloc(tm_base_sh, tm_cols);
  if constexpr (CS > 1) cg::this_cluster().sync();
}

namespace {

size_t morton_tmem_smem(int np, int W, int CS) {
  size_t bytes = static_cast<size_t>(np) * 12;
  bytes += ((np >> 5) + 4 - ((np >> 5) & 3)) * 4;
  bytes += 2 * W * sizeof(uint4);
  bytes += CS > 1 ? 2 * CS * W * sizeof(Msg) : 0;
  bytes += 2 * sizeof(uint64_t) + 8 * sizeof(int);
  bytes += sizeof(uint32_t) << morton_cell_bits(np);  // bucketing histogram
  return bytes;
}

template <int W, int CS, bool WIN>
cudaError_t launch_morton_tmem(SampleParams p, int rows, cudaStream_t st) {
  const int rpw = (rows + W - 1) / W;
  const int np = rpw * W * 32;
  p.nmax = np;
  const size_t smem = morton_tmem_smem(np, W, CS);
  if (smem > kMaxSmem) return cudaErrorNotSupported;
  int cols = 32;
  while (cols < W * rpw) cols *= 2;  // W/4 warps per quarter x 4 columns x rpw rows
  if (cols > 512) return cudaErrorNotSupported;
  if (plan("morton_tmem_kernel", {W, CS, WIN})) return cudaSuccess;
  auto kern = morton_tmem_kernel<W, CS, WIN>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  if (CS > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(p.B * p.M * CS));
  cfg.blockDim = dim3(W * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, p, cols);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// Warps per CTA: the fewest that give one row per lane, except that CTAs
// of 65-128 rows get 8 warps when the SMs hold about two sectors or fewer
// (r01: 256 x 4K FPS 1.24 -> 1.13 ms; with ~7 sectors per SM the smaller
// CTAs win: AFPS M=4 at 8K 1.09 vs 1.37 ms).
int morton_tmem_w(int rows, long long sectors) {
  const int forced = pcs_internal::knobs().morton_w;
  if ((forced == 4 || forced == 8 || forced == 16) && rows <= 32 * forced) return forced;
  int w = rows <= 128 ? 4 : rows <= 256 ? 8 : 16;
  if (w == 4 && rows > 64 && sectors <= 2 * 148) w = 8;
  return w;
}

template <int CS>
cudaError_t launch_morton_tmem_w(SampleParams p, int rows, cudaStream_t st) {
  // one row per lane: W >= rows / 32, a multiple of 4 (whole lane quarters)
  const int w = morton_tmem_w(rows, p.B * p.M);
  if (rows > 512) return cudaErrorNotSupported;
  if (p.K > 0) {
    if (w <= 4) return launch_morton_tmem<4, CS, true>(p, rows, st);
    if (w <= 8) return launch_morton_tmem<8, CS, true>(p, rows, st);
    return launch_morton_tmem<16, CS, true>(p, rows, st);
  }
  if (w <= 4) return launch_morton_tmem<4, CS, false>(p, rows, st);
  if (w <= 8) return launch_morton_tmem<8, CS, false>(p, rows, st);
  return launch_morton_tmem<16, CS, false>(p, rows, st);
}

}  // namespace

// Smallest cluster whose per-CTA share fits (<= 512 rows and shared memory).
// (Spreading few sectors over larger clusters than capacity needs measured
// slower everywhere but a lone 32K cloud.)
cudaError_t run_morton_tmem_any(SampleParams p, long long n, cudaStream_t st) {
  // fp32 batches; distance traces come from the fp64 drop-in (other engines)
  if (p.f64 || p.trace) return cudaErrorNotSupported;
  const long long srows = (n + 31) / 32;
  const int cs_min = 1;
  for (int CS = cs_min; CS <= 16; CS *= 2) {
    const int rows = static_cast<int>((srows + CS - 1) / CS);
    if (rows > 512) continue;
    const int W = morton_tmem_w(rows, p.B * p.M);
    const int rpw = (rows + W - 1) / W;
    if (morton_tmem_smem(rpw * W * 32, W, CS) > kMaxSmem) continue;
    switch (CS) {
      case 1: return launch_morton_tmem_w<1>(p, rows, st);
      case 2: return launch_morton_tmem_w<2>(p, rows, st);
      case 4: return launch_morton_tmem_w<4>(p, rows, st);
      case 8: return launch_morton_tmem_w<8>(p, rows, st);
      default: return launch_morton_tmem_w<16>(p, rows, st);
    }
  }
  return cudaErrorNotSupported;
}

}  // namespace pcsk
