// Full-window FPS / AFPS kernels (see sampler_common.cuh for the layout).
#include <cstdlib>

#include "sampler_common.cuh"

#ifdef PCS_PROF
__device__ unsigned long long g_fprof[8];
#define FPROF_T(v) long long v = clock64()
#else
#define FPROF_T(v)
#endif

namespace pcsk {

// A/B switch of the slot loop's hand-spelled update + argmax step
#ifndef PCS_FULL_ASM
#define PCS_FULL_ASM 1
#endif
constexpr bool kSlotAsm = PCS_FULL_ASM != 0;
#ifndef PCS_FULL_CHAIN
#define PCS_FULL_CHAIN 4
#endif
constexpr int kChainLen = PCS_FULL_CHAIN;
// most slots per thread that take the hand-spelled argmax chains
#ifndef PCS_FULL_ARG_MAXP
#define PCS_FULL_ARG_MAXP 8
#endif

// (best, bs) <- (bits, k) when bits > best: one 64-bit compare, three selects
__device__ __forceinline__ void argmax_step(unsigned long long& best, int& bs,
                                            unsigned long long bits, int k) {
  asm("{\n .reg .pred p;\n setp.gt.u64 p, %2, %0;\n selp.b64 %0, %2, %0, p;\n"
      " selp.b32 %1, %3, %1, p;\n}"
      : "+l"(best), "+r"(bs) : "l"(bits), "r"(k));
}

// ---------------------------------------------------------------- full window
// FPS / AFPS: every iteration updates the whole sector (sampler.cpp:115-129
// with window == sector). REGC: sector xyz also cached in registers.
template <int P, int W, bool REGC>
__global__ void __launch_bounds__(W * 32 * (W >= 8 ? 1 : (8 / W)))
    fps_full_kernel(const SampleParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int T = W * 32;
  const int gid = threadIdx.x / T, t = threadIdx.x % T, lane = t & 31, warp = t >> 5;
  GroupSetup gs;
  if (!setup_group<W>(p, smem, gid, t, gs)) return;
  const int n = gs.g.n;
  group_sync<W>(gid);

  double x[REGC ? P : 1], y[REGC ? P : 1], z[REGC ? P : 1], d[P];
  unsigned vmask = 0;
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const int j = k * T + t;
    const bool valid = j < n;
    vmask |= valid ? (1u << k) : 0u;
    if constexpr (REGC) {
      // padding slots: NaN coordinates make every `dist <= d` false there
      const double kNaN = __longlong_as_double(0x7ff8000000000000LL);
      x[k] = valid ? gs.xs[j] : kNaN;
      y[k] = valid ? gs.ys[j] : kNaN;
      z[k] = valid ? gs.zs[j] : kNaN;
    }
    d[k] = valid ? __longlong_as_double(0x7ff0000000000000LL) : 0.0;
  }

  int cur = first_point(p, gs);
  // output indices buffered in warp 0, sample i in lane i % 32, stored 32 at
  // a time (off the iteration's critical path)
  const long long obase = gs.b * p.C + gs.g.out_off;
  const long long ioff = gs.g.begin + p.index_base;
  const bool idx64 = p.idx64 != 0;
  void* const out = p.out_idx;
  // (measured: a win for 1-4 warps per sector, a loss with 8+ where the
  // extra state changes the compiler's schedule of the slot loop)
  constexpr bool kBufOut = W <= 4;
  int ob = cur;
  if (!kBufOut && t == 0) write_index(p, gs.b, gs.g.out_off, gs.g.begin + cur);
  auto flush = [&](int i0, int cnt) {
    if (warp == 0 && lane < cnt) {
      if (idx64) static_cast<long long*>(out)[obase + i0 + lane] = ioff + ob;
      else static_cast<int*>(out)[obase + i0 + lane] = static_cast<int>(ioff + ob);
    }
  };
  unsigned smask = (cur % T == t) ? (1u << (cur / T)) : 0u;
  double* const trace = p.trace;
  unsigned writes = 0;
  int round = 0;

#ifdef PCS_PROF
  unsigned long long pacc[4] = {0, 0, 0, 0};
#endif
  for (int it = 1; it < gs.g.quota; ++it) {
    FPROF_T(t0);
    const double px = gs.xs[cur], py = gs.ys[cur], pz = gs.zs[cur];
    // The update + running-argmax step of a slot, hand-spelled for 4 and 8
    // slots per thread (r02 s4, profiles/r02_full_slot_asm_ab.log: AFPS M=16
    // at 16K 1.31 -> 1.19 ms, M=64 at 32K 1.28 -> 1.20, M=16 at 8K 0.358 ->
    // 0.337; with 16 slots the compiler's own argmax is 18% faster and only
    // the update part is taken, with 1-2 slots there is nothing to gain)
    constexpr bool kAsm = REGC && kSlotAsm && (P == 4 || P == 8 || P == 16);
    // 16 slots: only the update part (the hand-spelled argmax chains cost
    // 18% there, the update part gains 1-3%)
    constexpr bool kAsmUpd = kAsm;
    constexpr bool kAsmArg = kAsm && P <= PCS_FULL_ARG_MAXP;
    constexpr int kChains = (kAsmArg && P > kChainLen) ? P / kChainLen : 1;
    unsigned long long bestc[kChains];
    int bsc[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) { bestc[c] = 0; bsc[c] = -1; }
    // Branch-free over the slots so independent slots interleave (ILP).
    // Padding slots (j >= n) hold d = 0 and NaN coordinates (REGC): they
    // never win the argmax (best starts at 0 with a strict >) and never
    // write (NaN compares false).
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const int j = k * T + t;
      const double xx = REGC ? x[REGC ? k : 0] : gs.xs[min(j, n - 1)];
      const double yy = REGC ? y[REGC ? k : 0] : gs.ys[min(j, n - 1)];
      const double zz = REGC ? z[REGC ? k : 0] : gs.zs[min(j, n - 1)];
      const double dist = dist2(xx, yy, zz, px, py, pz);
      if constexpr (kAsmUpd) {
        // one predicate per step, spelled out: the compiler's own form of
        // this loop re-derives the comparisons for the slot index (4 ISETP +
        // 3 SEL per slot) and counts writes with an add and a move
        // (profiles/r02_full_slot_asm_ab.log)
        asm("{\n .reg .pred p;\n setp.le.f64 p, %2, %1;\n selp.f64 %1, %2, %1, p;\n"
            " @p add.u32 %0, %0, 1;\n}"
            : "+r"(writes), "+d"(d[k]) : "d"(dist));
      } else {
        const bool lower = dist <= d[k];
        writes += (lower && (REGC || ((vmask >> k) & 1u))) ? 1u : 0u;
        d[k] = lower ? dist : d[k];
      }
      const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(d[k]));
      if constexpr (kAsmArg) {
        argmax_step(bestc[k * kChains / P], bsc[k * kChains / P], bits, k);
      } else {
        unsigned long long& best = bestc[0];
        int& bs = bsc[0];
        if (bits > best) {
          best = bits;
          bs = k;
        }
      }
    }
#pragma unroll
    for (int c = 1; c < kChains; ++c) argmax_step(bestc[0], bsc[0], bestc[c], bsc[c]);
    const unsigned long long best = bestc[0];
    const int bs = bsc[0];
    if (trace) {
#pragma unroll
      for (int k = 0; k < P; ++k)
        if ((vmask >> k) & 1u) trace[static_cast<long long>(it - 1) * n + k * T + t] = d[k];
    }
    FPROF_T(t1);
    uint32_t hi = static_cast<uint32_t>(best >> 32), lo = static_cast<uint32_t>(best);
    uint32_t j = bs >= 0 ? static_cast<uint32_t>(bs * T + t) : kNoIndex;
    group_argmax<W>(hi, lo, j, gs.cand, round, gid, lane, warp);
    FPROF_T(t2);
    if ((hi | lo) == 0u)
      j = lowest_unsampled<P, W>(vmask, smask, t, gs.cand, round, gid, lane, warp);
    cur = static_cast<int>(j);
    if constexpr (kBufOut) {
      if (lane == (it & 31)) ob = cur;
      if ((it & 31) == 31) flush(it - 31, 32);
    } else if (t == 0) {
      write_index(p, gs.b, gs.g.out_off + it, gs.g.begin + cur);
    }
    if (cur % T == t) smask |= 1u << (cur / T);
#ifdef PCS_PROF
    FPROF_T(t3);
    pacc[0] += t1 - t0; pacc[1] += t2 - t1; pacc[2] += t3 - t2; pacc[3] += 1;
#endif
  }
#ifdef PCS_PROF
  if (t == 0)
    for (int q = 0; q < 4; ++q) atomicAdd(&g_fprof[q], pacc[q]);
#endif
  if (kBufOut && ((gs.g.quota - 1) & 31) != 31)
    flush((gs.g.quota - 1) & ~31, ((gs.g.quota - 1) & 31) + 1);
  const unsigned long long evals =
      static_cast<unsigned long long>(gs.g.quota - 1) * static_cast<unsigned long long>(n);
  flush_stats<W>(p, gs, t, writes, evals);
}

// ------------------------------------------------------ window, latency form
// NPDU sectors when the SMs hold few of them (the per-iteration chain, not
// issue, is the limit there). The full kernel's layout -- W warps per sector,
// point j = k*T + t in registers, so row r (32 points) belongs to warp r % W,
// slot r / W -- but each iteration evaluates only the slots whose row meets
// update_window [wb, we) (sectors.cpp:53-61): a window of R rows spreads over
// min(R, W) warps that work in parallel, and the per-thread max over P slots
// plus the group argmax replace the one-warp kernel's per-row key cache.
template <int P, int W>
__global__ void __launch_bounds__(W * 32 * (W >= 8 ? 1 : (8 / W)))
    npdu_wide_kernel(const SampleParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int T = W * 32;
  const int gid = threadIdx.x / T, t = threadIdx.x % T, lane = t & 31, warp = t >> 5;
  GroupSetup gs;
  if (!setup_group<W>(p, smem, gid, t, gs)) return;
  const int n = gs.g.n;
  group_sync<W>(gid);

  double x[P], y[P], z[P], d[P];
  unsigned vmask = 0;
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const int j = k * T + t;
    const bool valid = j < n;
    vmask |= valid ? (1u << k) : 0u;
    const double kNaN = __longlong_as_double(0x7ff8000000000000LL);
    x[k] = valid ? gs.xs[j] : kNaN;
    y[k] = valid ? gs.ys[j] : kNaN;
    z[k] = valid ? gs.zs[j] : kNaN;
    d[k] = valid ? __longlong_as_double(0x7ff0000000000000LL) : 0.0;
  }

  int cur = first_point(p, gs);
  const long long obase = gs.b * p.C + gs.g.out_off;
  const long long ioff = gs.g.begin + p.index_base;
  const bool idx64 = p.idx64 != 0;
  void* const out = p.out_idx;
  int ob = cur;
  auto flush = [&](int i0, int cnt) {
    if (warp == 0 && lane < cnt) {
      if (idx64) static_cast<long long*>(out)[obase + i0 + lane] = ioff + ob;
      else static_cast<int*>(out)[obase + i0 + lane] = static_cast<int>(ioff + ob);
    }
  };
  unsigned smask = (cur % T == t) ? (1u << (cur / T)) : 0u;
  double* const trace = p.trace;
  const int half_down = static_cast<int>(p.K / 2), half_up = static_cast<int>((p.K + 1) / 2);
  unsigned writes = 0;
  unsigned long long evals = 0;
  int round = 0;
#ifdef PCS_PROF
  unsigned long long pacc[5] = {0, 0, 0, 0, 0};
#endif
  for (int it = 1; it < gs.g.quota; ++it) {
    FPROF_T(t0);
    const double px = gs.xs[cur], py = gs.ys[cur], pz = gs.zs[cur];
    const int wb = cur >= half_down ? cur - half_down : 0;
    const int we = min(n, cur + half_up);
    evals += static_cast<unsigned long long>(we - wb);
    const int r_lo = wb >> 5, r_hi = (we - 1) >> 5;
    unsigned long long best = 0;
    int bs = -1;
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const int r = k * W + warp;
      if (r >= r_lo && r <= r_hi) {  // warp-uniform: this slot's row meets the window
        const int j = k * T + t;
        const double dist = dist2(x[k], y[k], z[k], px, py, pz);
        const bool lower = j >= wb && j < we && dist <= d[k];
        writes += lower ? 1u : 0u;
        d[k] = lower ? dist : d[k];
      }
      const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(d[k]));
      if (bits > best) {
        best = bits;
        bs = k;
      }
    }
    if (trace) {
#pragma unroll
      for (int k = 0; k < P; ++k)
        if ((vmask >> k) & 1u) trace[static_cast<long long>(it - 1) * n + k * T + t] = d[k];
    }
    uint32_t hi = static_cast<uint32_t>(best >> 32), lo = static_cast<uint32_t>(best);
    uint32_t j = bs >= 0 ? static_cast<uint32_t>(bs * T + t) : kNoIndex;
#ifdef PCS_PROF
    FPROF_T(t1);
    warp_argmax(hi, lo, j);
    FPROF_T(t2);
    {
      uint4* buf = gs.cand + (round & 1) * W;
      if (lane == 0) buf[warp] = make_uint4(hi, lo, j, 0);
      named_bar_sync(1 + gid, W * 32);
      const uint4 v = lane < W ? buf[lane] : make_uint4(0, 0, kNoIndex, 0);
      hi = v.x; lo = v.y; j = v.z;
    }
    FPROF_T(t3);
    warp_argmax(hi, lo, j);
    ++round;
    FPROF_T(t4);
    pacc[0] += t1 - t0; pacc[1] += t2 - t1; pacc[2] += t3 - t2; pacc[3] += t4 - t3; pacc[4] += 1;
#else
    group_argmax<W>(hi, lo, j, gs.cand, round, gid, lane, warp);
#endif
    if ((hi | lo) == 0u)
      j = lowest_unsampled<P, W>(vmask, smask, t, gs.cand, round, gid, lane, warp);
    cur = static_cast<int>(j);
    if (lane == (it & 31)) ob = cur;
    if ((it & 31) == 31) flush(it - 31, 32);
    if (cur % T == t) smask |= 1u << (cur / T);
  }
#ifdef PCS_PROF
  if (t == 0)
    for (int q = 0; q < 5; ++q) atomicAdd(&g_fprof[q], pacc[q]);
#endif
  if (((gs.g.quota - 1) & 31) != 31) flush((gs.g.quota - 1) & ~31, ((gs.g.quota - 1) & 31) + 1);
  flush_stats<W>(p, gs, t, writes, evals);
}

// ------------------------------------------------------ tiny sectors
// Sectors of <= NP points (AFPS with many sectors: M=256 at 2K-4K points):
// one THREAD per sector runs the whole local FPS -- fp64 d in
// registers (every loop unrolled over NP slots, nothing indexed
// dynamically), coordinates (input precision) in shared memory, slot-major. A warp per sector (fps_full_kernel) spent
// most of its time staging 8-32 points and synchronising 32 lanes for one
// to seven iterations. Windowed calls take update_window as usual. OpStats
// are summed over the warp before the atomics when its sectors share a cloud.
template <int NP, typename CT>
__global__ void __launch_bounds__(128) fps_tiny_kernel(const SampleParams p) {
  const long long flat = static_cast<long long>(blockIdx.x) * 128 + threadIdx.x;
  const long long total = p.B * p.M;
  const bool active = flat < total;
  const long long b = active ? flat / p.M : 0, s = active ? flat % p.M : 0;
  const SectorGeom g = sector_geom(p.N, p.C, p.M, s);
  const int n = active ? g.n : 0;
  const CT* cloud = static_cast<const CT*>(p.xyz) + b * p.N * 3;
  const int* permb = p.perm ? p.perm + b * p.N : nullptr;
  // coordinates in shared memory, slot-major (slot i of thread t at
  // i * 128 + t: conflict-free), d in registers
  __shared__ CT sxyz[3][NP * 128];
  CT* const X = sxyz[0] + threadIdx.x;
  CT* const Y = sxyz[1] + threadIdx.x;
  CT* const Z = sxyz[2] + threadIdx.x;
  double d[NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    d[i] = 0.0;
    X[i * 128] = Y[i * 128] = Z[i * 128] = CT(0);
    if (i < n) {
      const long long jj = g.begin + i;
      const long long src = permb ? static_cast<long long>(__ldg(permb + jj)) : jj;
      X[i * 128] = __ldg(cloud + 3 * src);
      Y[i * 128] = __ldg(cloud + 3 * src + 1);
      Z[i * 128] = __ldg(cloud + 3 * src + 2);
      d[i] = __longlong_as_double(0x7ff0000000000000LL);
    }
  }
  unsigned writes = 0, evals = 0;
  int quota = active ? g.quota : 0;
  if (active) {
    GroupSetup gs;
    gs.b = b;
    gs.s = s;
    gs.g = g;
    int cur = first_point(p, gs);
    const long long obase = b * p.C + g.out_off;
    const long long ioff = g.begin + p.index_base;
    auto put = [&](int slot, int v) {
      if (p.idx64) static_cast<long long*>(p.out_idx)[obase + slot] = ioff + v;
      else static_cast<int*>(p.out_idx)[obase + slot] = static_cast<int>(ioff + v);
      if (p.out_sector) p.out_sector[obase + slot] = static_cast<int>(s + p.sector_base);
    };
    put(0, cur);
    uint32_t sampled = NP > 32 ? 0u : (1u << cur);
    double px = 0.0, py = 0.0, pz = 0.0;
    px = static_cast<double>(X[cur * 128]);
    py = static_cast<double>(Y[cur * 128]);
    pz = static_cast<double>(Z[cur * 128]);
    const int half_down = static_cast<int>(p.K / 2), half_up = static_cast<int>((p.K + 1) / 2);
    for (int it = 1; it < quota; ++it) {
      int wb = 0, we = n;
      if (p.K > 0) {
        wb = cur >= half_down ? cur - half_down : 0;
        we = min(n, cur + half_up);
      }
      evals += static_cast<unsigned>(we - wb);
      unsigned long long best = 0;
      int bi = -1;
#pragma unroll
      for (int i = 0; i < NP; ++i) {
        if (i >= wb && i < we) {
          const double dist = dist2(static_cast<double>(X[i * 128]), static_cast<double>(Y[i * 128]),
                                    static_cast<double>(Z[i * 128]), px, py, pz);
          const bool lower = dist <= d[i];
          writes += lower ? 1u : 0u;
          d[i] = lower ? dist : d[i];
        }
        const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(d[i]));
        if (i < n && bits > best) {
          best = bits;
          bi = i;
        }
      }
      if (best == 0ull) {
        // every distance is 0: lowest unsampled index (sampler.cpp:148-154)
        bi = -1;
#pragma unroll
        for (int i = NP - 1; i >= 0; --i)
          if (i < n && !((sampled >> i) & 1u)) bi = i;
      }
      cur = bi;
      px = static_cast<double>(X[cur * 128]);
      py = static_cast<double>(Y[cur * 128]);
      pz = static_cast<double>(Z[cur * 128]);
      sampled |= 1u << cur;
      put(it, cur);
    }
  }
  if (p.stats) {
    const unsigned iters = quota > 0 ? static_cast<unsigned>(quota - 1) : 0u;
    const unsigned scans = iters * static_cast<unsigned>(n);
    if (p.K == 0) evals = scans;
    // one atomic per counter per warp when all its sectors belong to one cloud
    const long long b0 = __shfl_sync(kFull, b, 0);
    const bool same = __all_sync(kFull, !active || b == b0) && __shfl_sync(kFull, active, 0);
    if (same) {
      const unsigned ev = __reduce_add_sync(kFull, evals), wr = __reduce_add_sync(kFull, writes),
                     sc = __reduce_add_sync(kFull, scans), itr = __reduce_add_sync(kFull, iters);
      if ((threadIdx.x & 31) == 0) {
        unsigned long long* st = p.stats + b0 * 4;
        atomicAdd(st + 0, static_cast<unsigned long long>(ev));
        if (wr) atomicAdd(st + 1, static_cast<unsigned long long>(wr));
        atomicAdd(st + 2, static_cast<unsigned long long>(sc));
        atomicAdd(st + 3, static_cast<unsigned long long>(itr));
      }
    } else if (active) {
      unsigned long long* st = p.stats + b * 4;
      atomicAdd(st + 0, static_cast<unsigned long long>(evals));
      if (writes) atomicAdd(st + 1, static_cast<unsigned long long>(writes));
      atomicAdd(st + 2, static_cast<unsigned long long>(scans));
      atomicAdd(st + 3, static_cast<unsigned long long>(iters));
    }
  }
}

template <int NP, typename CT>
cudaError_t run_tiny(SampleParams p, cudaStream_t st) {
  if (plan("fps_tiny_kernel", {NP, sizeof(CT) * 8})) return cudaSuccess;
  const long long blocks = (p.B * p.M + 127) / 128;
  fps_tiny_kernel<NP, CT><<<static_cast<unsigned>(blocks), 128, 0, st>>>(p);
  return cudaGetLastError();
}

// many sectors of <= 16 points; a thread per sector (r02, 256 clouds:
// AFPS M=256 at 2K (8 points) 0.062 -> 0.021 ms, at 4K (16 points) 0.070 ->
// 0.039; at 32 points a warp per sector wins again: M=256 at 8K 0.085 vs
// 0.092, M=64 at 2K 0.025 vs 0.045)
cudaError_t run_tiny_any(SampleParams p, long long n, cudaStream_t st) {
  if (p.trace || n > 16 || p.B * p.M < kTinyMinSectors || !pcs_internal::knobs().tiny)
    return cudaErrorNotSupported;
  if (p.f64) return n <= 8 ? run_tiny<8, double>(p, st) : run_tiny<16, double>(p, st);
  return n <= 8 ? run_tiny<8, float>(p, st) : run_tiny<16, float>(p, st);
}

template <typename Kern>
cudaError_t launch_groups(Kern kern, const char* name, std::initializer_list<long long> targs,
                          SampleParams p, int W, int G, cudaStream_t st) {
  const size_t group_bytes = size_t(24) * p.nmax + 32 * W;
  const size_t smem = group_bytes * G;
  if (smem > kMaxSmem) return cudaErrorInvalidConfiguration;
  if (plan(name, targs)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  p.G = G;
  const long long sectors = p.B * p.M;
  const long long blocks = (sectors + G - 1) / G;
  kern<<<static_cast<unsigned>(blocks), G * W * 32, smem, st>>>(p);
  return cudaGetLastError();
}

// Groups per CTA: up to `max_threads` threads and ~110 KB of shared memory
// (two CTAs per SM), fewer when there are not enough sectors to fill the SMs.
int pick_groups(long long sectors, int W, int nmax, int max_threads) {
  const size_t group_bytes = size_t(24) * nmax + 32 * W;
  int G = std::max(1, max_threads / (W * 32));
  if (W > 1) G = std::min(G, 15);  // named barriers 1..15
  while (G > 1 && group_bytes * G > 110 * 1024) G /= 2;
  while (G > 1 && (sectors + G - 1) / G < 2 * 148) G /= 2;
  return G;
}

template <int P, int W, bool REGC>
cudaError_t run_full(SampleParams p, cudaStream_t st) {
  const int G = pick_groups(p.B * p.M, W, p.nmax, W >= 8 ? W * 32 : 256);
  return launch_groups(fps_full_kernel<P, W, REGC>, "fps_full_kernel", {P, W, REGC}, p, W, std::min(G, W >= 8 ? 1 : 8 / W), st);
}

cudaError_t run_full_any(SampleParams p, long long n, cudaStream_t st) {
  if (n <= 32) return run_full<1, 1, true>(p, st);
  if (n <= 64) return run_full<2, 1, true>(p, st);
  if (n <= 128) return run_full<4, 1, true>(p, st);
  if (n <= 256) {
    // one sector per SM or fewer: 8 warps x 1 slot shorten the serial chain
    // (cfg2 sampler 0.032 -> 0.027 ms with 4 x 2, r02 -> 0.0235 with 8 x 1);
    // with many sectors one warp each wins (AFPS M=16 at 4K: 0.098 vs 0.157 ms)
    if (p.B * p.M <= 148) return run_full<1, 8, true>(p, st);
    return run_full<8, 1, true>(p, st);
  }
  // 8 slots per thread (twice the warps, ~120 registers) hides more latency
  // when an SM holds one sector or at least four; with ~2 sectors per SM the
  // 16-slot form measured faster (r01 sweep: cfg5 FPS 2K 0.374 vs 0.400 ms;
  // AFPS M=4 at 8K 1.69 vs 1.33 ms, cfg1 0.283 vs 0.262 ms).
  const long long sectors = p.B * p.M;
  // (r02: 512-point sectors at ~7 per SM -- 1024 sectors, cfg3 AFPS and
  // cfg5 AFPS M=4 at 2K -- run faster with 16 slots, 0.108 -> 0.094 ms; from
  // 4096 sectors on the 8-slot form wins again, 0.333 vs 0.384 ms at 8K M=16)
  const bool p8 = (sectors >= 4 * 148 && !(n <= 512 && sectors <= 2048)) || sectors <= 148;
  if (p8) {
    // (at most one sector per SM, 512 points: 8 warps x 2 slots, 16 x 512
    // AFPS M=4 0.051 -> 0.046 ms; 1024 points keep 4 warps x 8 slots)
    if (sectors <= 148 && n <= 512) return run_full<2, 8, true>(p, st);
    if (n <= 512) return run_full<8, 2, true>(p, st);
    if (n <= 1024) return run_full<8, 4, true>(p, st);
    if (n <= 2048) return run_full<8, 8, true>(p, st);
    if (n <= 4096) return run_full<8, 16, true>(p, st);
    return cudaErrorNotSupported;
  }
  if (n <= 512) return run_full<16, 1, true>(p, st);
  if (n <= 1024) return run_full<16, 2, true>(p, st);
  if (n <= 2048) return run_full<16, 4, true>(p, st);
  if (n <= 4096) return run_full<16, 8, true>(p, st);
  return cudaErrorNotSupported;
}

template <int P, int W>
cudaError_t run_wide(SampleParams p, cudaStream_t st) {
  const int G = pick_groups(p.B * p.M, W, p.nmax, W >= 8 ? W * 32 : 256);
  return launch_groups(npdu_wide_kernel<P, W>, "npdu_wide_kernel", {P, W}, p, W, std::min(G, W >= 8 ? 1 : 8 / W), st);
}

// Windowed sectors <= 4096 points, W >= 8 warps (a window of <= 8 rows -- k
// <= 225 -- then meets at most one row per warp).
cudaError_t run_npdu_wide_any(SampleParams p, long long n, cudaStream_t st) {
  // (8 warps measured best: 1024-point sectors at 1 per SM, 16 warps x 2
  // slots 0.148 ms, 32 x 1 0.213 ms, 8 x 4 0.117 ms; one warp 0.142 ms)
  if (n <= 256) return run_wide<1, 8>(p, st);
  if (n <= 512) return run_wide<2, 8>(p, st);
  if (n <= 1024) return run_wide<4, 8>(p, st);
  if (n <= 2048) return run_wide<8, 8>(p, st);
  if (n <= 4096) return run_wide<8, 16>(p, st);
  return cudaErrorNotSupported;
}

}  // namespace pcsk
