// NPDU-FPS / NPDU-AFPS kernels for sm_100a.
//
// The update touches only update_window(sector, idx, k) (proj/src/
// sectors.cpp:53-61): the k storage neighbours of the pivot. One warp owns
// one sector. xyz and the fp64 min-distances d[] live in shared memory, so
// the rows of 32 points a window touches are addressed with a runtime row
// index; fp32 inputs stay fp32 there (widened exactly on use), which halves
// the footprint and doubles the sectors resident per SM.
//
// The argmax still ranges over the whole sector, as the reference's does
// (sampler.cpp:137-154), but incrementally: each row's (max d, min index) is
// cached in registers -- lane l holds rows l, l+32, ... -- and only rows the
// window touched are re-reduced. d only decreases, so untouched rows keep
// valid maxima; an iteration costs O(k/32 + rows/32) instead of O(n).
//
// Shared arrays are padded with whole rows past the sector end (d = 0,
// xyz = 0): the window's rows are processed branch-free and unclamped, pad
// lanes never write (the window ends inside the sector) and never win the
// argmax (their d = 0 can only tie a max of 0, which takes the lowest-
// unsampled path).
#include <cstdlib>
#include <type_traits>

#include "sampler_common.cuh"
#include "rows_common.cuh"
#include "tmem.cuh"

namespace pcsk {

// Rows of padding after the sector: the RMAX-unrolled path reads up to
// RMAX-1 rows past the window's last row; the runtime loop reads one.
__host__ __device__ constexpr int npdu_pad_rows(int rmax) { return rmax > 2 ? rmax : 2; }

__host__ __device__ __forceinline__ int npdu_padded(int nmax, int rmax) {
  return (((nmax + 31) >> 5) + npdu_pad_rows(rmax)) << 5;
}

// GC: xyz stays in global memory (L1/L2-resident input) and only d[] and
// the bitmap occupy shared memory, which roughly triples the resident
// sectors per SM at the price of L2 latency on the window's coordinates.
template <typename CT, bool GC = false>
__host__ __device__ __forceinline__ size_t npdu_warp_bytes(int nmax, int rmax) {
  const size_t np = static_cast<size_t>(npdu_padded(nmax, rmax));
  return (np * (8 + (GC ? 0 : 3 * sizeof(CT))) + np / 8 + 15) & ~size_t(15);
}

// Row key with the index deferred: (max d, ballot of the lanes holding it).
// Rows order their indices (row r < row r' => every index smaller), so the
// sector argmax only needs the lowest row among equal maxima, and the lane
// within it (ffs of the ballot) is resolved once, for the winning row.
__device__ __forceinline__ void row_key_mask(double dj, uint32_t& hi, uint32_t& lo,
                                             uint32_t& mask) {
  const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(dj));
  const uint32_t h = static_cast<uint32_t>(bits >> 32), l = static_cast<uint32_t>(bits);
  const uint32_t mh = __reduce_max_sync(kFull, h);
  const uint32_t ml = __reduce_max_sync(kFull, h == mh ? l : 0u);
  mask = __ballot_sync(kFull, h == mh && l == ml);
  hi = mh;
  lo = ml;
}

template <bool F2F>
__device__ __forceinline__ double to_f64(float v) { return F2F ? static_cast<double>(v) : widen_f32(v); }
template <bool F2F>
__device__ __forceinline__ double to_f64(double v) { return v; }

template <int RPL>
__device__ __forceinline__ void store_row(int r, int lane, uint32_t hi, uint32_t lo, uint32_t j,
                                          uint32_t (&rh)[RPL], uint32_t (&rl)[RPL],
                                          uint32_t (&rj)[RPL]) {
#pragma unroll
  for (int i = 0; i < RPL; ++i)
    if (r == lane + 32 * i) {
      rh[i] = hi;
      rl[i] = lo;
      rj[i] = j;
    }
}

// RMAX > 0: a window spans at most RMAX rows (ceil((k+31)/32)); all RMAX are
// processed unconditionally and unrolled in phases (all loads, then the fp64
// chains, then the stores, then the reductions) so the rows overlap. Rows
// past the window get no writes and re-reduce to their cached value.
// RMAX == 0: runtime row loop (wide windows).
template <typename CT, int RPL, int RMAX, bool GC>
__global__ void __launch_bounds__(768) npdu_warp_kernel(const SampleParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int gid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long flat = static_cast<long long>(blockIdx.x) * p.G + gid;
  if (flat >= p.B * p.M) return;
  const long long b = flat / p.M, s = flat % p.M;
  const SectorGeom g = sector_geom(p.N, p.C, p.M, s);
  const int n = g.n, np = npdu_padded(p.nmax, RMAX);
  unsigned char* base = smem + static_cast<size_t>(gid) * npdu_warp_bytes<CT, GC>(p.nmax, RMAX);
  double* d = reinterpret_cast<double*>(base);
  CT* xs = reinterpret_cast<CT*>(d + np);
  CT* ys = xs + np;
  CT* zs = ys + np;
  unsigned* sampled = reinterpret_cast<unsigned*>(GC ? reinterpret_cast<CT*>(d + np) : zs + np);
  // coordinate fetch: shared SoA, or the global AoS input (clamped into the
  // sector so pad lanes never read past it)
  const CT* gsrc = static_cast<const CT*>(p.xyz) + (b * p.N + g.begin) * 3;
  auto X = [&](int j) -> CT { if constexpr (GC) return __ldg(gsrc + 3 * min(j, n - 1)); else return xs[j]; };
  auto Y = [&](int j) -> CT { if constexpr (GC) return __ldg(gsrc + 3 * min(j, n - 1) + 1); else return ys[j]; };
  auto Z = [&](int j) -> CT { if constexpr (GC) return __ldg(gsrc + 3 * min(j, n - 1) + 2); else return zs[j]; };
  if (sizeof(CT) < sizeof(double) && p.f64) __trap();  // fp32 staging is fp32-input only
  if constexpr (!GC) {
    if (p.f64)
      stage_sector_of<double>(p, b, g.begin, n, xs, ys, zs, lane, 32);
    else
      stage_sector_of<float>(p, b, g.begin, n, xs, ys, zs, lane, 32);
  }
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  for (int j = lane; j < np; j += 32) {
    d[j] = j < n ? kInf : 0.0;
    if constexpr (!GC)
      if (j >= n) xs[j] = ys[j] = zs[j] = CT(0);
  }
  const int rows = (n + 31) >> 5;
  for (int w = lane; w < (np >> 5); w += 32) sampled[w] = 0u;

  if (p.out_sector)
    for (int i = lane; i < g.quota; i += 32)
      p.out_sector[b * p.C + g.out_off + i] = static_cast<int>(s + p.sector_base);
  // row maxima: lane l caches row r = l + 32*i in slot i; initially every
  // point is +inf, so a row's winner is its first point
  // (key = max d and the ballot of the lanes holding it, row_key_mask)
  uint32_t rm_hi[RPL], rm_lo[RPL], rm_m[RPL];
#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    const int r = lane + 32 * i;
    rm_hi[i] = r < rows ? kInfHi : 0u;
    rm_lo[i] = 0u;
    rm_m[i] = r < rows ? 1u : 0u;
  }
  GroupSetup gs;
  gs.b = b;
  gs.s = s;
  gs.g = g;
  int cur = first_point(p, gs);
  // output row of this sector; index written = begin + index_base + local
  const long long out_base = b * p.C + g.out_off;
  const long long index_off = g.begin + p.index_base;
  int* out32 = static_cast<int*>(p.out_idx) + out_base;
  long long* out64 = static_cast<long long*>(p.out_idx) + out_base;
  if (lane == 0) {
    if (p.idx64) out64[0] = index_off + cur;
    else out32[0] = static_cast<int>(index_off + cur);
    sampled[cur >> 5] |= 1u << (cur & 31);
  }
  __syncwarp();
  const long long K = p.K;
  const int half_down = static_cast<int>(K / 2), half_up = static_cast<int>((K + 1) / 2);
  unsigned writes = 0;
  unsigned long long evals = 0;
  double* const trace = p.trace;

  auto iterate = [&](auto f2f_tag) {
  constexpr bool F2F = decltype(f2f_tag)::value;
  for (int it = 1; it < g.quota; ++it) {
    const double px = to_f64<F2F>(X(cur)), py = to_f64<F2F>(Y(cur)), pz = to_f64<F2F>(Z(cur));
    const int wb = cur >= half_down ? cur - half_down : 0;
    const int we = min(n, cur + half_up);
    evals += static_cast<unsigned long long>(we - wb);
    const int r_lo = wb >> 5;
    if constexpr (RMAX > 0) {
      const int j0 = (r_lo << 5) + lane;
      double dj[RMAX], dist[RMAX];
      bool lower[RMAX];
#pragma unroll
      for (int q = 0; q < RMAX; ++q) {
        const int j = j0 + 32 * q;
        dj[q] = d[j];
        dist[q] = dist2(to_f64<F2F>(X(j)), to_f64<F2F>(Y(j)), to_f64<F2F>(Z(j)), px, py, pz);
      }
#pragma unroll
      for (int q = 0; q < RMAX; ++q) {
        const int j = j0 + 32 * q;
        lower[q] = j >= wb && j < we && dist[q] <= dj[q];
        writes += lower[q] ? 1u : 0u;
        dj[q] = lower[q] ? dist[q] : dj[q];
      }
#pragma unroll
      for (int q = 0; q < RMAX; ++q)
        if (lower[q]) d[j0 + 32 * q] = dist[q];
#pragma unroll
      for (int q = 0; q < RMAX; ++q) {
        uint32_t hi, lo, mk;
        row_key_mask(dj[q], hi, lo, mk);
        store_row<RPL>(r_lo + q, lane, hi, lo, mk, rm_hi, rm_lo, rm_m);
      }
    } else {
      const int r_hi = (we - 1) >> 5;
      for (int r = r_lo; r <= r_hi; r += 2) {
        const int ja = (r << 5) + lane, jb = ja + 32;
        double da = d[ja], db = d[jb];
        const double ea = dist2(to_f64<F2F>(X(ja)), to_f64<F2F>(Y(ja)), to_f64<F2F>(Z(ja)), px, py, pz);
        const double eb = dist2(to_f64<F2F>(X(jb)), to_f64<F2F>(Y(jb)), to_f64<F2F>(Z(jb)), px, py, pz);
        const bool la = ja >= wb && ja < we && ea <= da;
        const bool lb = jb >= wb && jb < we && eb <= db;
        writes += (la ? 1u : 0u) + (lb ? 1u : 0u);
        if (la) d[ja] = ea;
        if (lb) d[jb] = eb;
        da = la ? ea : da;
        db = lb ? eb : db;
        uint32_t hi, lo, mk;
        row_key_mask(da, hi, lo, mk);
        store_row<RPL>(r, lane, hi, lo, mk, rm_hi, rm_lo, rm_m);
        row_key_mask(db, hi, lo, mk);
        store_row<RPL>(r + 1, lane, hi, lo, mk, rm_hi, rm_lo, rm_m);
      }
    }
    if (trace) {
      __syncwarp();
      for (int j = lane; j < n; j += 32) trace[static_cast<long long>(it - 1) * n + j] = d[j];
    }
    // whole-sector argmax from the cached row maxima; rows l + 32*i grow with
    // i, so a strict > keeps the lowest index among equal distances
    uint32_t hi = rm_hi[0], lo = rm_lo[0], mk = rm_m[0], rsel = static_cast<uint32_t>(lane);
#pragma unroll
    for (int i = 1; i < RPL; ++i) {
      const bool gt = rm_hi[i] > hi || (rm_hi[i] == hi && rm_lo[i] > lo);
      hi = gt ? rm_hi[i] : hi;
      lo = gt ? rm_lo[i] : lo;
      mk = gt ? rm_m[i] : mk;
      rsel = gt ? static_cast<uint32_t>(lane + 32 * i) : rsel;
    }
    // max d, lowest row among equals, its lowest lane (rows order indices)
    uint32_t j;
    {
      const uint32_t mh = __reduce_max_sync(kFull, hi);
      const uint32_t ml = __reduce_max_sync(kFull, hi == mh ? lo : 0u);
      const uint32_t mr = __reduce_min_sync(kFull, (hi == mh && lo == ml) ? rsel : kNoIndex);
      const uint32_t wm = __shfl_sync(kFull, mk, static_cast<int>(mr & 31u));
      hi = mh;
      lo = ml;
      j = (mr << 5) + static_cast<uint32_t>(__ffs(wm)) - 1u;
    }
    if ((hi | lo) == 0u) {
      // every distance is 0: lowest unsampled index (sampler.cpp:148-154)
      uint32_t jm = kNoIndex;
      for (int w = lane; w < rows && jm == kNoIndex; w += 32) {
        const unsigned free_bits = ~sampled[w];
        if (free_bits) {
          const uint32_t cand = static_cast<uint32_t>(w * 32 + __ffs(free_bits) - 1);
          if (cand < static_cast<uint32_t>(n)) jm = cand;
        }
      }
      j = __reduce_min_sync(kFull, jm);
    }
    cur = static_cast<int>(j);
    if (lane == 0) {
      if (p.idx64) out64[it] = index_off + cur;
      else out32[it] = static_cast<int>(index_off + cur);
      sampled[cur >> 5] |= 1u << (cur & 31);
    }
    __syncwarp();
  }
  };
  // F2F widening here: this kernel is latency-bound and F2F's latency is
  // shorter than the integer widening chain (measured; the XU is not
  // saturated at NPDU's evaluation rate)
  iterate(std::true_type{});
  const unsigned ws = __reduce_add_sync(kFull, writes);
  if (p.stats && lane == 0) {
    unsigned long long* st = p.stats + b * 4;
    const unsigned long long iters = static_cast<unsigned long long>(g.quota - 1);
    if (ws) atomicAdd(st + 1, static_cast<unsigned long long>(ws));
    atomicAdd(st + 0, evals);
    atomicAdd(st + 2, iters * static_cast<unsigned long long>(n));
    atomicAdd(st + 3, iters);
  }
}

template <typename CT, int RPL, int RMAX, bool GC>
cudaError_t run_npdu(SampleParams p, cudaStream_t st) {
  const size_t warp_bytes = npdu_warp_bytes<CT, GC>(p.nmax, RMAX);
  // warps per CTA: as many as shared memory lets one SM hold (one CTA per SM
  // when the batch is large), but never so many that CTAs < SMs
  const long long per_sm = static_cast<long long>(kMaxSmem / warp_bytes);
  const long long sectors = p.B * p.M;
  const int G = static_cast<int>(std::max(1LL, std::min({24LL, per_sm, sectors / 148})));
  const size_t smem = warp_bytes * G;
  if (smem > kMaxSmem) return cudaErrorNotSupported;
  if (plan("npdu_warp_kernel", {sizeof(CT), RPL, RMAX, GC})) return cudaSuccess;
  auto kern = npdu_warp_kernel<CT, RPL, RMAX, GC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  p.G = G;
  const long long blocks = (sectors + G - 1) / G;
  kern<<<static_cast<unsigned>(blocks), 32 * G, smem, st>>>(p);
  return cudaGetLastError();
}

template <typename CT, int RPL, bool GC>
cudaError_t run_npdu_rows(SampleParams p, cudaStream_t st) {
  // rows a window of K consecutive points can touch: ceil((K + 31) / 32)
  const long long rows_needed = (p.K + 62) / 32;
  if (rows_needed <= 2) return run_npdu<CT, RPL, 2, GC>(p, st);
  if (rows_needed <= 3) return run_npdu<CT, RPL, 3, GC>(p, st);
  if (rows_needed <= 5) return run_npdu<CT, RPL, 5, GC>(p, st);
  return run_npdu<CT, RPL, 0, GC>(p, st);
}

template <int RPL>
cudaError_t run_npdu_rpl(SampleParams p, cudaStream_t st) {
  if (p.f64) return run_npdu_rows<double, RPL, false>(p, st);
  // fp32 input: stage fp32 (widened exactly on use) unless fp64 staging
  // still fits 16 warps per SM
  if (npdu_warp_bytes<double>(p.nmax, 5) * 16 <= kMaxSmem) return run_npdu_rows<double, RPL, false>(p, st);
  return run_npdu_rows<float, RPL, false>(p, st);
}


// ---------------------------------------------------------------- TMEM variant
// Same algorithm, with the fp64 min-distances in tensor memory instead of
// shared memory: shared memory then holds only xyz (fp32) and the sampled
// bitmap, so twice as many sectors (= independent dependency chains) fit per
// SM, and the kernel is latency-bound, so resident sectors are throughput.
// Layout: warp w of the CTA uses TMEM lanes 32*(w%4).. (its lane quarter)
// and a column block per warp; row r of its sector (32 points) is the column
// pair (2r, 2r+1) = (lo, hi) words of each lane's double. A window's RMAX rows
// are one or two tcgen05.ld/st per iteration.



// RMAX rows = 2*RMAX columns, as power-of-two tcgen05 shapes
template <int RMAX>
__device__ __forceinline__ void tm_load_rows(uint32_t a, double (&v)[RMAX]) {
  static_assert(RMAX == 2 || RMAX == 3 || RMAX == 5, "row count");
  uint32_t w[2 * RMAX];
  if constexpr (RMAX == 2) {
    uint32_t t[4];
    tm_ld(a, t);
    tm_wait_ld();
    for (int i = 0; i < 4; ++i) w[i] = t[i];
  } else if constexpr (RMAX == 3) {
    uint32_t t[4], u[2];
    tm_ld(a, t);
    tm_ld(a + 4, u);
    tm_wait_ld();
    for (int i = 0; i < 4; ++i) w[i] = t[i];
    w[4] = u[0]; w[5] = u[1];
  } else {
    uint32_t t[8], u[2];
    tm_ld(a, t);
    tm_ld(a + 8, u);
    tm_wait_ld();
    for (int i = 0; i < 8; ++i) w[i] = t[i];
    w[8] = u[0]; w[9] = u[1];
  }
#pragma unroll
  for (int q = 0; q < RMAX; ++q) v[q] = __hiloint2double(static_cast<int>(w[2 * q + 1]), static_cast<int>(w[2 * q]));
}

template <int RMAX>
__device__ __forceinline__ void tm_store_rows(uint32_t a, const double (&v)[RMAX]) {
  uint32_t w[2 * RMAX];
#pragma unroll
  for (int q = 0; q < RMAX; ++q) {
    w[2 * q] = static_cast<uint32_t>(__double2loint(v[q]));
    w[2 * q + 1] = static_cast<uint32_t>(__double2hiint(v[q]));
  }
  if constexpr (RMAX == 2) {
    uint32_t t[4] = {w[0], w[1], w[2], w[3]};
    tm_st(a, t);
  } else if constexpr (RMAX == 3) {
    uint32_t t[4] = {w[0], w[1], w[2], w[3]}, u[2] = {w[4], w[5]};
    tm_st(a, t);
    tm_st(a + 4, u);
  } else {
    uint32_t t[8] = {w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7]}, u[2] = {w[8], w[9]};
    tm_st(a, t);
    tm_st(a + 8, u);
  }
}

// Per-warp capacity NCAP points (a compile-time stride: xs/ys/zs at fixed
// offsets, so one address serves all three loads). The window's RMAX rows
// are clamped into [0, max(NCAP/32, RMAX)) rows, so no padding rows are read
// or written beyond that.
__host__ __device__ constexpr int tm_rows_alloc(int ncap, int rmax) {
  return (ncap >> 5) > rmax ? (ncap >> 5) : rmax;
}
__host__ __device__ constexpr int tm_cols_per_warp(int ncap, int rmax) {
  return 2 * tm_rows_alloc(ncap, rmax);
}
__host__ __device__ constexpr size_t tm_warp_smem(int ncap) {
  return (size_t(12) * ncap + 4 * ((ncap >> 5) + 8) + 15) & ~size_t(15);
}

// Row-key forms of the TMEM kernel (see the cached-key comment inside):
// exact (max d, index) keys, exact (max d, lane ballot) keys, or high-word
// keys with an exact slow path. The high-word form issues the fewest
// instructions (multi-wave launches, which are issue-bound); the exact index
// form has the shortest argmax chain (one-wave launches, latency-bound).
// kKeyMin: the high-word keys of kKeyHigh plus, per row, the index of the
// lowest lane holding the row's high word (a redux.sync.min beside the row's
// ballot), so the sector argmax is max(hi) then min(index) -- two dependent
// redux.sync, no ballot -> find-first-set -> shuffle -> find-first-set chain.
enum NpduKey { kKeyIndex = 0, kKeyBallot = 1, kKeyHigh = 2, kKeyMin = 3 };

// fp32 input, sectors <= NCAP <= 4096 points (1-4 cached rows per lane)
// MAXT: the CTA width the launch uses at most. The register budget follows
// it: the 4-warp CTAs of multi-wave launches (16 warps per SM) and CTAs of up
// to 16 warps get up to 128 registers per thread instead of the 64 a
// 1024-thread bound allows -- the 64-register build rematerialised addresses
// and window terms every iteration (r02 s4, eager launches: cfg4 0.361 ->
// 0.306 ms, 256x32K M=16 0.96 -> 0.86, 256x16K 0.312 -> 0.288;
// profiles/r02_npdu_launch_bounds_ab.log)
template <int RMAX, int NCAP, int KEY, int MAXT = 1024>
__global__ void __launch_bounds__(MAXT, MAXT == 128 ? 4 : 1) npdu_tmem_kernel(const SampleParams p, int tm_cols) {
  static_assert(NCAP >= 32 * RMAX && NCAP <= 4096, "capacity");
  constexpr int RPL = NCAP > 1024 ? NCAP / 1024 : 1;  // rows per lane (row r: lane r % 32)
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t tm_base_sh;
  const int gid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (gid == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&tm_base_sh))), "r"(tm_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm_base = tm_base_sh;
  const long long flat = static_cast<long long>(blockIdx.x) * p.G + gid;
  if (flat < p.B * p.M) {
    const long long b = flat / p.M, s = flat % p.M;
    const SectorGeom g = sector_geom(p.N, p.C, p.M, s);
    const int n = g.n;
    constexpr int cpw = tm_cols_per_warp(NCAP, RMAX);
    // this warp's TMEM: lane quarter (gid % 4), column block (gid / 4)
    const uint32_t tm = tm_base + ((static_cast<uint32_t>(gid & 3) * 32u) << 16) +
                        static_cast<uint32_t>((gid >> 2) * cpw);
    unsigned char* base = smem + static_cast<size_t>(gid) * tm_warp_smem(NCAP);
    float* xs = reinterpret_cast<float*>(base);
    float* ys = xs + NCAP;
    float* zs = ys + NCAP;
    unsigned* sampled = reinterpret_cast<unsigned*>(zs + NCAP);
    stage_sector_of<float>(p, b, g.begin, n, xs, ys, zs, lane, 32);
    const int rows = (n + 31) >> 5;
    for (int w = lane; w < rows + 8; w += 32) sampled[w] = 0u;
    // d = +inf on the sector, 0 on the pad rows
    {
      const double kInf = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll 1
      for (int r = 0; r < tm_rows_alloc(NCAP, RMAX); ++r) {
        const int j = (r << 5) + lane;
        const double v = j < n ? kInf : 0.0;
        uint32_t t[2] = {static_cast<uint32_t>(__double2loint(v)), static_cast<uint32_t>(__double2hiint(v))};
        tm_st(tm + 2 * r, t);
      }
      tm_wait_st();
    }
    if (p.out_sector)
      for (int i = lane; i < g.quota; i += 32)
        p.out_sector[b * p.C + g.out_off + i] = static_cast<int>(s + p.sector_base);
    // cached row keys (row r = lane + 32 i), by KEY:
    //  * kKeyIndex: (max d, lowest index holding it), exact;
    //  * kKeyBallot: (max d, ballot of the lanes holding it), exact, the index
    //    deferred to the winning row (rows order indices);
    //  * kKeyHigh: the HIGH WORD of the row's max d and the ballot of the
    //    lanes whose d carries it -- one redux.sync + one vote per touched
    //    row. The high word orders distances except within a tie of high
    //    words; the argmax is decided from these keys when that cannot
    //    matter (a single candidate lane, or a tie at +inf: 0x7ff00000 is
    //    +inf exactly, all such values are equal, lowest index wins) and
    //    otherwise by an exact slow path that re-reads the candidate rows'
    //    fp64 values from TMEM (measured: 3e-4 of cfg4's iterations).
    uint32_t rm_hi[RPL], rm_lo[RPL], rm_m[RPL], rm_j[RPL];
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = lane + 32 * i;
      rm_hi[i] = r < rows ? kInfHi : 0u;
      rm_lo[i] = 0u;
      rm_j[i] = r < rows ? static_cast<uint32_t>(r * 32) : kNoIndex;
      rm_m[i] = KEY == kKeyIndex ? (r < rows ? static_cast<uint32_t>(r * 32) : kNoIndex)
                                 : (r < rows ? 1u : 0u);
    }
    GroupSetup gs;
    gs.b = b;
    gs.s = s;
    gs.g = g;
    int cur = first_point(p, gs);
    const long long out_base = b * p.C + g.out_off;
    const long long index_off = g.begin + p.index_base;
    int* out32 = static_cast<int*>(p.out_idx) + out_base;
    long long* out64 = static_cast<long long*>(p.out_idx) + out_base;
    const bool idx64 = p.idx64 != 0;
    // output indices are buffered one per lane (sample t in lane t % 32) and
    // stored 32 at a time; the sampled bitmap is only needed by the
    // all-zero slow path, which folds the outputs into it on demand
    int ob = cur;
    const long long K = p.K;
    const int half_down = static_cast<int>(K / 2), half_up = static_cast<int>((K + 1) / 2);
    // dist_evals = the window sizes along the path: output t (t <= quota-2)
    // is the pivot of iteration t+1, so each lane adds its buffered
    // output's window when the block of 32 is stored (off the chain)
    unsigned long long evals = 0;
    auto flush = [&](int t0, int cnt) {
      if (lane < cnt) {
        if (idx64) out64[t0 + lane] = index_off + ob;
        else out32[t0 + lane] = static_cast<int>(index_off + ob);
        if (t0 + lane <= g.quota - 2)
          evals += static_cast<unsigned long long>(min(n, ob + half_up) - max(0, ob - half_down));
      }
    };
    int marked = 0;  // outputs [0, marked) are in the bitmap
    unsigned writes = 0;
    // blocks of 32 outputs: the inner loop has no flush test; windows of
    // <= 3 rows run it unrolled by two (r02 s4: cfg3 0.076 -> 0.074 ms,
    // 256x16K M=16 0.281 -> 0.276; 5-row windows 0.7% slower, not unrolled;
    // profiles/r02_npdu_upd_asm_ab.log)
    constexpr int kIterUnroll = RMAX <= 3 ? 2 : 1;
    for (int blk = 0; blk < g.quota; blk += 32) {
      const int it_end = min(blk + 32, g.quota);
#pragma unroll kIterUnroll
      for (int it = blk > 0 ? blk : 1; it < it_end; ++it) {
        const double px = static_cast<double>(xs[cur]), py = static_cast<double>(ys[cur]),
                     pz = static_cast<double>(zs[cur]);
        const int wb = cur >= half_down ? cur - half_down : 0;
        const int we = min(n, cur + half_up);
        // the RMAX rows from r_lo cover the window; near the sector's end
        // they are shifted down so they stay inside the allocated rows (the
        // extra rows are masked out and stored back unchanged)
        const int r_lo = min(wb >> 5, max(rows - RMAX, 0));
        const int j0 = (r_lo << 5) + lane;
        // j in [wb, we) <=> (unsigned)(j - wb) < we - wb
        const uint32_t t0 = static_cast<uint32_t>(j0 - wb), wlen = static_cast<uint32_t>(we - wb);
        double dj[RMAX], dist[RMAX];
        tm_wait_st();
        tm_load_rows<RMAX>(tm + 2 * r_lo, dj);
#pragma unroll
        for (int q = 0; q < RMAX; ++q) {
          // slots past n hold stale shared memory: evaluated, never used
          const int jc = j0 + 32 * q;
          dist[q] = dist2(static_cast<double>(xs[jc]), static_cast<double>(ys[jc]),
                          static_cast<double>(zs[jc]), px, py, pz);
        }
        if constexpr (RMAX <= 3) {
          // window test, min-update and write count on one predicate, spelled
          // out (r02 s4: windows of <= 3 rows 1-3% faster -- cfg3 0.078 ->
          // 0.076 ms, 256x16K M=16 0.289 -> 0.282; 5-row windows 1% slower
          // and kept on the compiler's form; profiles/r02_npdu_upd_asm_ab.log)
#pragma unroll
          for (int q = 0; q < RMAX; ++q)
            asm("{\n .reg .pred p, w;\n setp.lt.u32 w, %3, %4;\n setp.le.and.f64 p, %2, %1, w;\n"
                " selp.f64 %1, %2, %1, p;\n @p add.u32 %0, %0, 1;\n}"
                : "+r"(writes), "+d"(dj[q]) : "d"(dist[q]), "r"(t0 + 32u * q), "r"(wlen));
        } else {
          unsigned lmask = 0u;
#pragma unroll
          for (int q = 0; q < RMAX; ++q) {
            const bool lower = t0 + 32u * q < wlen && dist[q] <= dj[q];
            lmask |= lower ? 1u << q : 0u;
            dj[q] = lower ? dist[q] : dj[q];
          }
          writes += __popc(lmask);
        }
        tm_store_rows<RMAX>(tm + 2 * r_lo, dj);
        uint32_t mh, ml = 0u, j;
        bool exact;
        if constexpr (KEY == kKeyIndex || KEY == kKeyBallot) {
#pragma unroll
          for (int q = 0; q < RMAX; ++q) {
            uint32_t hi, lo, mk;
            row_key_mask(dj[q], hi, lo, mk);
            if constexpr (KEY == kKeyIndex) mk = static_cast<uint32_t>(((r_lo + q) << 5) + __ffs(mk) - 1);
            store_row<RPL>(r_lo + q, lane, hi, lo, mk, rm_hi, rm_lo, rm_m);
          }
          // this lane's best row (rows grow with i: strict > keeps the lowest),
          // then the warp's: max d, lowest row among equals, its lowest lane
          uint32_t hi = rm_hi[0], lo = rm_lo[0], mk = rm_m[0], rsel = static_cast<uint32_t>(lane);
#pragma unroll
          for (int i = 1; i < RPL; ++i)
            if (rm_hi[i] > hi || (rm_hi[i] == hi && rm_lo[i] > lo)) {
              hi = rm_hi[i]; lo = rm_lo[i]; mk = rm_m[i]; rsel = static_cast<uint32_t>(lane + 32 * i);
            }
          j = mk;
          if constexpr (KEY == kKeyIndex) {
            warp_argmax(hi, lo, j);
          } else {
            const uint32_t wh = __reduce_max_sync(kFull, hi);
            const uint32_t wl = __reduce_max_sync(kFull, hi == wh ? lo : 0u);
            const uint32_t mr = __reduce_min_sync(kFull, (hi == wh && lo == wl) ? rsel : kNoIndex);
            const uint32_t wm = __shfl_sync(kFull, mk, static_cast<int>(mr & 31u));
            hi = wh;
            lo = wl;
            j = (mr << 5) + static_cast<uint32_t>(__ffs(wm)) - 1u;
          }
          mh = hi;
          ml = lo;
          exact = (hi | lo) != 0u;
        } else if constexpr (KEY == kKeyMin) {
#pragma unroll
          for (int q = 0; q < RMAX; ++q) {
            const uint32_t h = static_cast<uint32_t>(__double2hiint(dj[q]));
            const uint32_t wk = __reduce_max_sync(kFull, h);
            const bool eq = h == wk;
            const uint32_t ll = __reduce_min_sync(kFull, eq ? static_cast<uint32_t>(lane) : 32u);
            const uint32_t mk = __ballot_sync(kFull, eq);
            const int r = r_lo + q;
#pragma unroll
            for (int i = 0; i < RPL; ++i)
              if (r == lane + 32 * i) {
                rm_hi[i] = wk;
                rm_j[i] = (static_cast<uint32_t>(r) << 5) + ll;
                rm_m[i] = mk;
              }
          }
          // this lane's best row (max high word, lowest row), then the
          // sector's: max high word, lowest index among the rows holding it.
          // Exact unless a high-word tie is possible: two candidate rows, or a
          // candidate row whose high word two lanes share (+inf ties are exact)
          uint32_t lh = rm_hi[0], lj = rm_j[0], lm = rm_m[0];
#pragma unroll
          for (int i = 1; i < RPL; ++i)
            if (rm_hi[i] > lh) { lh = rm_hi[i]; lj = rm_j[i]; lm = rm_m[i]; }
          int dup = 0;
#pragma unroll
          for (int i = 0; i < RPL; ++i) dup += rm_hi[i] == lh ? 1 : 0;
          mh = __reduce_max_sync(kFull, lh);
          const bool cand = lh == mh;
          j = __reduce_min_sync(kFull, cand ? lj : kNoIndex);
          const uint32_t rb = __ballot_sync(kFull, cand);
          const uint32_t bad = __ballot_sync(kFull, cand && (dup > 1 || (lm & (lm - 1u)) != 0u));
          // (bitwise: one predicate and one branch on the fast path)
          exact = (mh == kInfHi) | ((mh != 0u) & ((rb & (rb - 1u)) == 0u) & (bad == 0u));
        } else {
#pragma unroll
          for (int q = 0; q < RMAX; ++q) {
            const uint32_t h = static_cast<uint32_t>(__double2hiint(dj[q]));
            const uint32_t wk = __reduce_max_sync(kFull, h);
            const uint32_t mk = __ballot_sync(kFull, h == wk);
            const int r = r_lo + q;
#pragma unroll
            for (int i = 0; i < RPL; ++i)
              if (r == lane + 32 * i) {
                rm_hi[i] = wk;
                rm_m[i] = mk;
              }
          }
          // sector argmax on the high words: max, its lowest row, that row's
          // lowest lane (rows order indices)
          uint32_t wm, wr;
          bool unique;
          if constexpr (RPL == 1) {
            mh = __reduce_max_sync(kFull, rm_hi[0]);
            const uint32_t rb = __ballot_sync(kFull, rm_hi[0] == mh);
            wr = static_cast<uint32_t>(__ffs(rb)) - 1u;
            wm = __shfl_sync(kFull, rm_m[0], static_cast<int>(wr));
            unique = (rb & (rb - 1u)) == 0u;
          } else {
            uint32_t lh = rm_hi[0], lm = rm_m[0], ls = static_cast<uint32_t>(lane);
#pragma unroll
            for (int i = 1; i < RPL; ++i)
              if (rm_hi[i] > lh) { lh = rm_hi[i]; lm = rm_m[i]; ls = static_cast<uint32_t>(lane + 32 * i); }
            int dup = 0;
#pragma unroll
            for (int i = 0; i < RPL; ++i) dup += rm_hi[i] == lh ? 1 : 0;
            mh = __reduce_max_sync(kFull, lh);
            const uint32_t rb = __ballot_sync(kFull, lh == mh);
            const uint32_t rd = __ballot_sync(kFull, lh == mh && dup > 1);
            wr = __reduce_min_sync(kFull, lh == mh ? ls : kNoIndex);
            wm = __shfl_sync(kFull, lm, static_cast<int>(wr & 31u));
            unique = (rb & (rb - 1u)) == 0u && rd == 0u;
          }
          j = (wr << 5) + static_cast<uint32_t>(__ffs(wm)) - 1u;
          exact = mh == kInfHi || (mh != 0u && unique && (wm & (wm - 1u)) == 0u);
        }
        if (!exact) {
          uint32_t bh = mh, bl = ml;
          if constexpr (KEY == kKeyHigh || KEY == kKeyMin) {
            // exact resolution over the candidate rows (a high-word tie, or
            // every cached key 0): (max d, lowest index) from the fp64 values
            tm_wait_st();
            bh = bl = 0u;
            j = kNoIndex;
#pragma unroll
            for (int i = 0; i < RPL; ++i) {
              uint32_t cand = __ballot_sync(kFull, rm_hi[i] == mh && lane + 32 * i < rows);
              while (cand) {
                const int r = __ffs(cand) - 1 + 32 * i;
                cand &= cand - 1u;
                uint32_t t[2];
                tm_ld(tm + 2 * r, t);
                tm_wait_ld();
                uint32_t h, l, mk;
                // pad lanes past n hold d = 0 and are never written
                row_key_mask(__hiloint2double(static_cast<int>(t[1]), static_cast<int>(t[0])), h, l, mk);
                if (h > bh || (h == bh && l > bl) || j == kNoIndex) {
                  bh = h;
                  bl = l;
                  j = static_cast<uint32_t>((r << 5) + __ffs(mk) - 1);
                }
              }
            }
          }
          if ((bh | bl) == 0u) {
            // every distance is 0: lowest unsampled index (sampler.cpp:148-154);
            // fold outputs [marked, it) into the bitmap: whole blocks from
            // global memory, the current block from the lanes' buffers
            const int t_blk = (it - 1) & ~31;
            __syncwarp();
            for (int t = marked + lane; t < t_blk; t += 32) {
              const long long v = idx64 ? out64[t] : static_cast<long long>(out32[t]);
              const int jl = static_cast<int>(v - index_off);
              atomicOr(&sampled[jl >> 5], 1u << (jl & 31));
            }
            if (lane <= ((it - 1) & 31) && t_blk + lane >= marked)
              atomicOr(&sampled[ob >> 5], 1u << (ob & 31));
            marked = it;
            __syncwarp();
            uint32_t jm = kNoIndex;
            for (int w = lane; w < rows && jm == kNoIndex; w += 32) {
              const unsigned free_bits = ~sampled[w];
              if (free_bits) {
                const uint32_t cand = static_cast<uint32_t>(w * 32 + __ffs(free_bits) - 1);
                if (cand < static_cast<uint32_t>(n)) jm = cand;
              }
            }
            j = __reduce_min_sync(kFull, jm);
          }
        }
        cur = static_cast<int>(j);
        ob = lane == (it & 31) ? cur : ob;
      }
      flush(blk, it_end - blk);
    }
    tm_wait_st();
    const unsigned ws = __reduce_add_sync(kFull, writes);
    // per-lane window sums (< 2^32 each: a lane holds <= quota/32 outputs
    // of <= n points) -> the warp's
    const unsigned long long ev = __reduce_add_sync(kFull, static_cast<unsigned>(evals));
    if (p.stats && lane == 0) {
      unsigned long long* st = p.stats + b * 4;
      const unsigned long long iters = static_cast<unsigned long long>(g.quota - 1);
      if (ws) atomicAdd(st + 1, static_cast<unsigned long long>(ws));
      atomicAdd(st + 0, ev);
      atomicAdd(st + 2, iters * static_cast<unsigned long long>(n));
      atomicAdd(st + 3, iters);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (gid == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tm_base), "r"(tm_cols));
}

template <int RMAX, int NCAP, int KEY, int MAXT = 1024>
cudaError_t launch_npdu_tmem(SampleParams p, int G, int cols, size_t smem, cudaStream_t st) {
  if (plan("npdu_tmem_kernel", {RMAX, NCAP, KEY})) return cudaSuccess;
  auto kern = npdu_tmem_kernel<RMAX, NCAP, KEY, MAXT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  p.G = G;
  const long long blocks = (p.B * p.M + G - 1) / G;
  kern<<<static_cast<unsigned>(blocks), static_cast<unsigned>(32 * G), smem, st>>>(p, cols);
  return cudaGetLastError();
}

template <int RMAX, int NCAP>
cudaError_t run_npdu_tmem(SampleParams p, cudaStream_t st) {
  constexpr int cpw = tm_cols_per_warp(NCAP, RMAX);
  constexpr size_t wsm = tm_warp_smem(NCAP);
  const long long sectors = p.B * p.M;
  // warps per CTA (one CTA per SM): TMEM holds 4 lane quarters x (512 / cpw)
  // column blocks; shared memory and 32 warps bound it too
  long long G = std::min<long long>({32, 4LL * (512 / cpw), static_cast<long long>(kMaxSmem / wsm)});
  // One wave: balance it (as many CTAs as SMs, the same warps in each).
  // More than one: CTAs of 4 warps (one TMEM column block) -- several per SM,
  // replaced as they finish, so the SMs stay near full occupancy without a
  // wave tail (cfg4 0.404 -> 0.386 ms, 256x32K M=16 1.01 -> 0.93 ms; one-wave
  // batches keep the balanced single CTA: 256x4K 0.065 vs 0.10 ms). More
  // warps per SM than 4-warp CTAs give measured slower (cfg4: 6-warp CTAs,
  // 18 warps/SM 0.359 ms, one 18-warp CTA 0.403, vs 0.341;
  // profiles/r02_npdu_tmem_ab.log).
  const long long waves = (sectors + 148 * G - 1) / (148 * G);
  if (waves >= 2 && G >= 4)
    G = 4;
  else
    G = std::max(1LL, std::min(G, (sectors + 148 * waves - 1) / (148 * waves)));
  int cols = 32;
  while (cols < ((G + 3) / 4) * cpw) cols *= 2;
  if (cols > 512) return cudaErrorNotSupported;
  const size_t smem = wsm * G;
  // key form: launches that keep every SM's issue slots full (two or more
  // waves, or 16+ sectors per SM) take the high-word keys (few instructions
  // per touched row: cfg4 0.358 -> 0.355 ms, 256x32K M=16 1.07 -> 0.96),
  // with the per-row lowest-lane indices (kKeyMin: the sector argmax is two
  // dependent redux.sync instead of a redux -> ballot -> ffs -> shfl -> ffs
  // chain; r02 s3 A/B vs kKeyHigh: 256x16K M=16 0.333 -> 0.310 ms, 256x32K
  // 0.962 -> 0.920, cfg4 0.355 -> 0.351; profiles/r02_npdu_keymin_ab.log); a
  // launch of a few sectors per SM is bound by each warp's argmax chain,
  // where the exact index form is the shortest (cfg3, 7 sectors per SM,
  // 0.082 vs 0.088 ms with high-word keys). PCS_NPDU_KEY forces a form.
  switch (pcs_internal::knobs().npdu_key) {
    case kKeyIndex: return launch_npdu_tmem<RMAX, NCAP, kKeyIndex>(p, static_cast<int>(G), cols, smem, st);
    case kKeyBallot: return launch_npdu_tmem<RMAX, NCAP, kKeyBallot>(p, static_cast<int>(G), cols, smem, st);
    case kKeyHigh: return launch_npdu_tmem<RMAX, NCAP, kKeyHigh>(p, static_cast<int>(G), cols, smem, st);
    case kKeyMin: return launch_npdu_tmem<RMAX, NCAP, kKeyMin>(p, static_cast<int>(G), cols, smem, st);
    default: break;
  }
  const int g = static_cast<int>(G);
  if (G == 4 && waves >= 2) return launch_npdu_tmem<RMAX, NCAP, kKeyMin, 128>(p, 4, cols, smem, st);
  if (waves >= 2 || sectors >= 16 * 148) {
    if (G <= 16) return launch_npdu_tmem<RMAX, NCAP, kKeyMin, 512>(p, g, cols, smem, st);
    return launch_npdu_tmem<RMAX, NCAP, kKeyMin>(p, g, cols, smem, st);
  }
  constexpr int kOneWave = RMAX >= 5 ? kKeyBallot : kKeyIndex;
  if (G <= 16) return launch_npdu_tmem<RMAX, NCAP, kOneWave, 512>(p, g, cols, smem, st);
  return launch_npdu_tmem<RMAX, NCAP, kOneWave>(p, g, cols, smem, st);
}

cudaError_t run_npdu_any(SampleParams p, long long n, cudaStream_t st) {
  // At most one sector per SM: the serial update -> argmax chain is the
  // limit, and the W-warp register kernel (full_kernels.cu) runs it ~18%
  // shorter than one warp per sector. PCS_NPDU_WIDE = the largest batch (in sectors) that
  // takes it (0 disables).
  const pcs_internal::Knobs& kn = pcs_internal::knobs();
  const long long wide_max = kn.npdu_wide >= 0 ? kn.npdu_wide : kNpduWideMax;
  if (p.B * p.M <= wide_max && n <= 4096) {
    const cudaError_t e = run_npdu_wide_any(p, n, st);
    if (e != cudaErrorNotSupported) return e;
  }
  const bool use_tmem = kn.npdu_tmem;
  const long long rows_needed = (p.K + 62) / 32;
  // (the TMEM kernel serves fp32 batches; distance traces come from the
  // fp64 drop-in and take the shared-memory kernels)
  if (use_tmem && !p.f64 && !p.trace && n <= 4096 && rows_needed <= 5) {
    auto by_cap = [&](auto rmax_tag) {
      constexpr int R = decltype(rmax_tag)::value;
      if (n <= 256) return run_npdu_tmem<R, 256>(p, st);
      if (n <= 512) return run_npdu_tmem<R, 512>(p, st);
      if (n <= 1024) return run_npdu_tmem<R, 1024>(p, st);
      if (n <= 2048) return run_npdu_tmem<R, 2048>(p, st);
      return run_npdu_tmem<R, 4096>(p, st);
    };
    if (rows_needed <= 2) return by_cap(std::integral_constant<int, 2>{});
    if (rows_needed <= 3) return by_cap(std::integral_constant<int, 3>{});
    return by_cap(std::integral_constant<int, 5>{});
  }
  if (n <= 1024) return run_npdu_rpl<1>(p, st);
  if (n <= 2048) return run_npdu_rpl<2>(p, st);
  if (n <= 4096) return run_npdu_rpl<4>(p, st);
  if (n <= 8192) return run_npdu_rpl<8>(p, st);
  return cudaErrorNotSupported;
}

}  // namespace pcsk
