// Pruned-row sampler for large sectors (FPS / AFPS / NPDU variants), sm_100a.
//
// A sector (up to the whole cloud) lives on chip in one CTA, or split into
// row-aligned chunks over a thread-block cluster of CS CTAs: xyz (input type)
// and the fp64 min-distances d[] in shared memory. Points are grouped in rows
// of 32 consecutive storage indices. Every row keeps, in the registers of the
// lane that owns it, (a) its exact argmax key (max d bits, min index) and a
// float upper bound of that max, and (b) a float bounding box of its points.
//
// One iteration of local_fps (proj/src/sampler.cpp:114-161):
//   1. every lane tests its rows: a row can only change if some point of it
//      can get closer to the pivot than the row's current max d. The test is
//      a rigorous lower bound -- box-to-pivot squared distance in fp32 with
//      round-down arithmetic, shrunk by 2^-20 to cover the fp64 evaluation's
//      own rounding (< 5 * 2^-53 relative) -- against the row max rounded up.
//      A skipped row provably has dist > d[j] for every j: no write, no
//      change of its maximum. The decision never changes a result or a
//      counter; it only avoids work. (NPDU additionally restricts the rows to
//      the update window, proj/src/sectors.cpp:53-61.)
//   2. the surviving rows are updated exactly (fp64, reference operation
//      order, `dist <= d` rule) and re-reduced (2 redux + ballot);
//   3. warp -> CTA (shared memory, one barrier) -> cluster (DSMEM stores and
//      remote mbarrier arrivals; no cluster-wide barrier in the loop) argmax
//      on (max d, min index); candidates carry their coordinates so the next
//      pivot needs no lookup.
// dist_evals / argmax_scans / iterations are the reference's counts (the
// whole window is "evaluated" in its accounting: sampler.cpp:129, 155);
// dist_writes counts actual writes, which skipped rows provably have none of.
#include <cooperative_groups.h>

#include <cstdlib>
#include <type_traits>

#include "rows_common.cuh"

namespace cg = cooperative_groups;

namespace pcsk {

using namespace rows;

// Row ownership: sector row R (points [32R, 32R+32)) lives in cluster CTA
// R % CS as its local row R / CS, and inside the CTA in warp (R / CS) % W.
// Interleaving matters: on axis-sorted clouds the rows near the pivot are
// contiguous, so contiguous chunks would hand one CTA (one warp) all the work.
template <typename CT, int W, int RPL, int CS, bool WINDOWED>
__global__ void __launch_bounds__(W * 32) rows_kernel(const SampleParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rank = CS > 1 ? static_cast<int>(cg::this_cluster().block_rank()) : 0;
  const long long flat = static_cast<long long>(blockIdx.x) / CS;  // one sector per cluster
  const long long b = flat / p.M, s = flat % p.M;
  const SectorGeom g = sector_geom(p.N, p.C, p.M, s);
  const int n = g.n;
  const int srows = (n + 31) >> 5;                          // sector rows
  const int rows = srows > rank ? (srows - rank + CS - 1) / CS : 0;  // local rows
  const int np = (((p.nmax + 31) >> 5) + kRowsPad) << 5;   // local capacity
  double* d = reinterpret_cast<double*>(smem);
  CT* xs = reinterpret_cast<CT*>(d + np);
  CT* ys = xs + np;
  CT* zs = ys + np;
  unsigned* sampled = reinterpret_cast<unsigned*>(zs + np);
  uint4* cand = reinterpret_cast<uint4*>(sampled + (np >> 5) + 4 - ((np >> 5) & 3));
  Cand* xbuf = reinterpret_cast<Cand*>(cand + 2 * W);  // [2][CS]
  uint64_t* xbar = reinterpret_cast<uint64_t*>(xbuf + 2 * CS);  // [2] mbarriers
  if (sizeof(CT) < sizeof(double) && p.f64) __trap();
  // local point jl <-> sector point ((jl / 32) * CS + rank) * 32 + jl % 32
  auto to_sector = [&](int jl) { return (((jl >> 5) * CS + rank) << 5) + (jl & 31); };
  auto to_local = [&](int gj) { return (((gj >> 5) / CS) << 5) + (gj & 31); };

  {
    const long long cloud = (b * p.N + g.begin) * 3;
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
    for (int jl = threadIdx.x; jl < np; jl += W * 32) {
      const int gj = to_sector(jl);
      const bool valid = (jl >> 5) < rows && gj < n;
      double x = 0, y = 0, z = 0;
      if (valid) {
        if (p.f64) {
          const double* q = static_cast<const double*>(p.xyz) + cloud + 3LL * gj;
          x = q[0]; y = q[1]; z = q[2];
        } else {
          const float* q = static_cast<const float*>(p.xyz) + cloud + 3LL * gj;
          x = q[0]; y = q[1]; z = q[2];
        }
      }
      xs[jl] = static_cast<CT>(x);
      ys[jl] = static_cast<CT>(y);
      zs[jl] = static_cast<CT>(z);
      d[jl] = valid ? kInf : 0.0;
    }
  }
  for (int w = threadIdx.x; w < (np >> 5); w += W * 32) sampled[w] = 0u;
  if (p.out_sector && rank == 0)
    for (int i = threadIdx.x; i < g.quota; i += W * 32)
      p.out_sector[b * p.C + g.out_off + i] = static_cast<int>(s + p.sector_base);
  // fp32 subnormals cannot take the integer widening path (see widen_f32)
  bool sub_local = false;
  if constexpr (sizeof(CT) == 4)
    for (int jl = threadIdx.x; jl < np; jl += W * 32)
      sub_local |= is_subnormal_f32(static_cast<float>(xs[jl])) ||
                   is_subnormal_f32(static_cast<float>(ys[jl])) ||
                   is_subnormal_f32(static_cast<float>(zs[jl]));
  if (CS > 1 && threadIdx.x == 0) {
    mbar_init(&xbar[0], CS);
    mbar_init(&xbar[1], CS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const bool any_sub = __syncthreads_or(sub_local) != 0;
  if constexpr (CS > 1) cg::this_cluster().sync();  // every CTA's barriers exist

  // per-lane row metadata: local rows r = warp + W * (lane + 32 * i)
  float bx0[RPL], bx1[RPL], by0[RPL], by1[RPL], bz0[RPL], bz1[RPL];
  uint32_t rmh[RPL], rml[RPL], rmj[RPL];
#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    const int r = warp + W * (lane + 32 * i);
    float x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY, z0 = INFINITY,
          z1 = -INFINITY;
    const int R = r * CS + rank;
    if (r < rows) {
      const int e = min(32, n - R * 32);
      for (int q = 0; q < e; ++q) {
        const int jl = r * 32 + q;
        x0 = fminf(x0, f_lo(xs[jl]));
        x1 = fmaxf(x1, f_hi(xs[jl]));
        y0 = fminf(y0, f_lo(ys[jl]));
        y1 = fmaxf(y1, f_hi(ys[jl]));
        z0 = fminf(z0, f_lo(zs[jl]));
        z1 = fmaxf(z1, f_hi(zs[jl]));
      }
    }
    bx0[i] = x0; bx1[i] = x1; by0[i] = y0; by1[i] = y1; bz0[i] = z0; bz1[i] = z1;
    rmh[i] = r < rows ? kInfHi : 0u;
    rml[i] = 0u;
    rmj[i] = r < rows ? static_cast<uint32_t>(R * 32) : kNoIndex;
  }

  GroupSetup gs;
  gs.b = b;
  gs.s = s;
  gs.g = g;
  int cur = first_point(p, gs);  // sector-local
  double px, py, pz;
  float pfx = 0.f, pfy = 0.f, pfz = 0.f;  // exact fp32 pivot (fp32 input only)
  {
    const long long at = (b * p.N + g.begin + cur) * 3;
    if (p.f64) {
      const double* q = static_cast<const double*>(p.xyz) + at;
      px = q[0]; py = q[1]; pz = q[2];
    } else {
      const float* q = static_cast<const float*>(p.xyz) + at;
      pfx = q[0]; pfy = q[1]; pfz = q[2];
      px = pfx; py = pfy; pz = pfz;
    }
  }
  const long long out_base = b * p.C + g.out_off;
  const long long index_off = g.begin + p.index_base;
  if (rank == 0 && threadIdx.x == 0) {
    if (p.idx64) static_cast<long long*>(p.out_idx)[out_base] = index_off + cur;
    else static_cast<int*>(p.out_idx)[out_base] = static_cast<int>(index_off + cur);
  }
  if (((cur >> 5) % CS) == rank && threadIdx.x == 0) {
    const int jl = to_local(cur);
    sampled[jl >> 5] |= 1u << (jl & 31);
  }
  const long long K = p.K;
  const int half_down = static_cast<int>(K / 2), half_up = static_cast<int>((K + 1) / 2);
  unsigned writes = 0;
  unsigned long long evals = 0;
  int round = 0;

  auto iterate = [&](auto f2f_tag) {
  constexpr bool F2F = decltype(f2f_tag)::value;
  for (int it = 1; it < g.quota; ++it) {
    // window, sector-local (full window: everything)
    int wb = 0, we = n;
    if constexpr (WINDOWED) {
      wb = cur >= half_down ? cur - half_down : 0;
      we = min(n, cur + half_up);
      evals += static_cast<unsigned long long>(we - wb);
    }
    float pxl, pxh, pyl, pyh, pzl, pzh;
    if constexpr (sizeof(CT) == 4) {
      pxl = pxh = pfx; pyl = pyh = pfy; pzl = pzh = pfz;
    } else {
      pxl = f_lo(px); pxh = f_hi(px); pyl = f_lo(py); pyh = f_hi(py);
      pzl = f_lo(pz); pzh = f_hi(pz);
    }
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = warp + W * (lane + 32 * i);
      bool need = r < rows;
      if constexpr (WINDOWED) {
        const int R = r * CS + rank;
        need = need && (R * 32 < we) && (R * 32 + 32 > wb);
      }
      if (need) {
        const float lb = __fadd_rd(__fadd_rd(gap2(bx0[i], bx1[i], pxl, pxh),
                                             gap2(by0[i], by1[i], pyl, pyh)),
                                   gap2(bz0[i], bz1[i], pzl, pzh));
        // skip iff lb * (1 - 2^-20) > row max; compared on fp64 high words
        need = !(f32_as_f64_hi_lb(__fmul_rd(lb, 0.99999904f)) > rmh[i]);
      }
      int la = static_cast<int>(__reduce_min_sync(kFull, need ? lane : 32u));
      while (la < 32) {
        // two rows at a time: loads of both before any store (ILP)
        const int lb2r = static_cast<int>(__reduce_min_sync(kFull, (need && lane > la) ? lane : 32u));
        const int lb2 = lb2r < 32 ? lb2r : la;
        const int ra = warp + W * (la + 32 * i), rb = warp + W * (lb2 + 32 * i);
        const int ja = (ra << 5) + lane, jb = (rb << 5) + lane;          // local
        const int ga = ((ra * CS + rank) << 5) + lane, gb = ((rb * CS + rank) << 5) + lane;
        double da = d[ja], db = d[jb];
        const double ea = dist2(to_f64<F2F>(xs[ja]), to_f64<F2F>(ys[ja]), to_f64<F2F>(zs[ja]),
                                px, py, pz);
        const double eb = dist2(to_f64<F2F>(xs[jb]), to_f64<F2F>(ys[jb]), to_f64<F2F>(zs[jb]),
                                px, py, pz);
        const bool wa = ga >= wb && ga < we && ea <= da;
        const bool wbb = lb2 != la && gb >= wb && gb < we && eb <= db;
        writes += (wa ? 1u : 0u) + (wbb ? 1u : 0u);
        if (wa) d[ja] = ea;
        if (wbb) d[jb] = eb;
        da = wa ? ea : da;
        db = wbb ? eb : db;
        {
          const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(da));
          const uint32_t h0 = static_cast<uint32_t>(bits >> 32), l0 = static_cast<uint32_t>(bits);
          const uint32_t h = __reduce_max_sync(kFull, h0);
          const uint32_t l = __reduce_max_sync(kFull, h0 == h ? l0 : 0u);
          const uint32_t m = __reduce_min_sync(kFull, (h0 == h && l0 == l) ? lane : 32u);
          if (lane == la) {
            rmh[i] = h; rml[i] = l; rmj[i] = static_cast<uint32_t>(ga - lane) + m;
          }
        }
        if (lb2 != la) {
          const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(db));
          const uint32_t h0 = static_cast<uint32_t>(bits >> 32), l0 = static_cast<uint32_t>(bits);
          const uint32_t h = __reduce_max_sync(kFull, h0);
          const uint32_t l = __reduce_max_sync(kFull, h0 == h ? l0 : 0u);
          const uint32_t m = __reduce_min_sync(kFull, (h0 == h && l0 == l) ? lane : 32u);
          if (lane == lb2) {
            rmh[i] = h; rml[i] = l; rmj[i] = static_cast<uint32_t>(gb - lane) + m;
          }
        }
        if (lane == la || lane == lb2) need = false;
        la = static_cast<int>(__reduce_min_sync(kFull, need ? lane : 32u));
      }
    }
    if (p.trace) {
      __syncthreads();
      for (int jl = threadIdx.x; jl < rows * 32; jl += W * 32) {
        const int gj = to_sector(jl);
        if (gj < n) p.trace[static_cast<long long>(it - 1) * n + gj] = d[jl];
      }
    }
    // warp -> CTA argmax over the cached row keys (sector-local indices)
    uint32_t hi = rmh[0], lo = rml[0], j = rmj[0];
#pragma unroll
    for (int i = 1; i < RPL; ++i)
      if (key_gt(rmh[i], rml[i], rmj[i], hi, lo, j)) {
        hi = rmh[i]; lo = rml[i]; j = rmj[i];
      }
    warp_argmax(hi, lo, j);
    if constexpr (W > 1) {
      uint4* buf = cand + (round & 1) * W;
      if (lane == 0) buf[warp] = make_uint4(hi, lo, j, 0);
      __syncthreads();
      const uint4 v = lane < W ? buf[lane] : make_uint4(0, 0, kNoIndex, 0);
      hi = v.x; lo = v.y; j = v.z;
      warp_argmax(hi, lo, j);
    }
    bool zero = (hi | lo) == 0u;
    auto post = [&](Cand* slot, uint32_t h, uint32_t l, uint32_t jj) {
      // every CTA posts (key, index, coords) to every CTA's slot [rank]
      if (warp == 0 && lane < CS) {
        Cand c;
        c.hi = h; c.lo = l; c.j = jj; c.pad0 = c.pad1 = 0.f;
        const int jl = jj == kNoIndex ? 0 : to_local(static_cast<int>(jj));
        c.x = to_f64<F2F>(xs[jl]); c.y = to_f64<F2F>(ys[jl]); c.z = to_f64<F2F>(zs[jl]);
        c.fx = static_cast<float>(sizeof(CT) == 4 ? xs[jl] : CT(0));
        c.fy = static_cast<float>(sizeof(CT) == 4 ? ys[jl] : CT(0));
        c.fz = static_cast<float>(sizeof(CT) == 4 ? zs[jl] : CT(0));
        cg::this_cluster().map_shared_rank(slot, lane)[rank] = c;
        mbar_arrive_remote(&xbar[round & 1], lane);  // release orders the store
      }
    };
    auto wait_round = [&]() { mbar_wait(&xbar[round & 1], (round >> 1) & 1); };
    auto take = [&](const Cand& w) {
      px = w.x; py = w.y; pz = w.z;
      pfx = w.fx; pfy = w.fy; pfz = w.fz;
    };
    auto take_local = [&](uint32_t jj) {
      px = to_f64<F2F>(xs[jj]); py = to_f64<F2F>(ys[jj]); pz = to_f64<F2F>(zs[jj]);
      if constexpr (sizeof(CT) == 4) {
        pfx = static_cast<float>(xs[jj]); pfy = static_cast<float>(ys[jj]);
        pfz = static_cast<float>(zs[jj]);
      }
    };
    if constexpr (CS > 1) {
      Cand* slot = xbuf + (round & 1) * CS;
      post(slot, hi, lo, j);
      wait_round();
      uint32_t h = lane < CS ? slot[lane].hi : 0u, l = lane < CS ? slot[lane].lo : 0u;
      uint32_t jj = lane < CS ? slot[lane].j : kNoIndex;
      warp_argmax(h, l, jj);
      zero = (h | l) == 0u;
      hi = h; lo = l; j = jj;
      if (!zero) {
        const unsigned who =
            __ballot_sync(kFull, lane < CS && slot[lane].j == jj && slot[lane].hi == h && slot[lane].lo == l);
        take(slot[__ffs(who) - 1]);
      }
    } else {
      if (!zero) take_local(j);
    }
    ++round;
    if (zero) {
      // every distance is 0: lowest unsampled index (sampler.cpp:148-154)
      uint32_t jm = kNoIndex;
      for (int w = lane; w < rows && jm == kNoIndex; w += 32) {
        const unsigned free_bits = ~sampled[w];
        if (free_bits) {
          const int c = to_sector(w * 32 + __ffs(free_bits) - 1);
          if (c < n) jm = static_cast<uint32_t>(c);
        }
      }
      jm = __reduce_min_sync(kFull, jm);
      if constexpr (CS > 1) {
        Cand* slot = xbuf + (round & 1) * CS;
        post(slot, jm != kNoIndex ? 1u : 0u, 0u, jm);
        wait_round();
        uint32_t h = lane < CS ? slot[lane].hi : 0u, l = 0u, jj = lane < CS ? slot[lane].j : kNoIndex;
        warp_argmax(h, l, jj);
        const unsigned who = __ballot_sync(kFull, lane < CS && slot[lane].j == jj && slot[lane].hi == h);
        take(slot[__ffs(who) - 1]);
        j = jj;
        ++round;
      } else {
        j = jm;
        take_local(j);
      }
    }
    cur = static_cast<int>(j);  // sector-local
    if (rank == 0 && threadIdx.x == 0) {
      if (p.idx64) static_cast<long long*>(p.out_idx)[out_base + it] = index_off + cur;
      else static_cast<int*>(p.out_idx)[out_base + it] = static_cast<int>(index_off + cur);
    }
    if (((cur >> 5) % CS) == rank && threadIdx.x == 0) {
      const int jl = to_local(cur);
      sampled[jl >> 5] |= 1u << (jl & 31);
    }
  }
  };
  if (sizeof(CT) == 4 && any_sub)
    iterate(std::true_type{});
  else
    iterate(std::false_type{});
  // stats
  const unsigned ws = __reduce_add_sync(kFull, writes);
  if (p.stats) {
    unsigned long long* st = p.stats + b * 4;
    if (lane == 0 && ws) atomicAdd(st + 1, static_cast<unsigned long long>(ws));
    if (rank == 0 && threadIdx.x == 0) {
      const unsigned long long iters = static_cast<unsigned long long>(g.quota - 1);
      atomicAdd(st + 0, WINDOWED ? evals : iters * static_cast<unsigned long long>(n));
      atomicAdd(st + 2, iters * static_cast<unsigned long long>(n));
      atomicAdd(st + 3, iters);
    }
  }
  if constexpr (CS > 1) cg::this_cluster().sync();  // keep smem alive for remote writers
}

template <typename CT>
size_t rows_smem_bytes(int chunk, int W, int CS) {
  const size_t np = static_cast<size_t>((((chunk + 31) >> 5) + kRowsPad) << 5);
  size_t bytes = np * (8 + 3 * sizeof(CT));
  bytes += ((np >> 5) + 4 - ((np >> 5) & 3)) * 4;  // sampled bits, 16 B aligned
  bytes += 2 * W * sizeof(uint4);
  bytes += 2 * CS * sizeof(Cand);
  bytes += 2 * sizeof(uint64_t);  // exchange mbarriers
  return bytes;
}

template <typename CT, int W, int RPL, int CS, bool WIN>
cudaError_t launch_rows(SampleParams p, int chunk, cudaStream_t st) {
  p.nmax = chunk;
  const size_t smem = rows_smem_bytes<CT>(chunk, W, CS);
  if (smem > kMaxSmem) return cudaErrorNotSupported;
  if (plan("rows_kernel", {sizeof(CT), W, RPL, CS, WIN})) return cudaSuccess;
  auto kern = rows_kernel<CT, W, RPL, CS, WIN>;
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
  e = cudaLaunchKernelEx(&cfg, kern, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// Local rows -> warps: about 8 rows per warp (more warps = more rows updated
// in parallel per iteration), up to 32 warps, then 2 rows per lane.
// Warps per CTA from the CTA's row count: more warps update more candidate
// rows in parallel but each adds fixed per-iteration reduction work; 16 was
// best measured for 128-512 rows (cfg5 FPS 8K/16K, r01 sweep). A CTA never
// holds more than 512 rows (shared memory caps a chunk at ~11K fp32 points),
// so one row per lane suffices.
template <typename CT, int CS, bool WIN>
cudaError_t launch_rows_w(SampleParams p, int chunk, cudaStream_t st) {
  const int rows = (chunk + 31) / 32;
  if (rows <= 32) return launch_rows<CT, 4, 1, CS, WIN>(p, chunk, st);
  if (rows <= 64) return launch_rows<CT, 8, 1, CS, WIN>(p, chunk, st);
  if (rows <= 512) return launch_rows<CT, 16, 1, CS, WIN>(p, chunk, st);
  return cudaErrorNotSupported;
}

template <typename CT, bool WIN>
cudaError_t launch_rows_cs(SampleParams p, long long n, cudaStream_t st) {
  // largest chunk that fits shared memory, rounded down to whole rows
  const int cap = static_cast<int>(((kMaxSmem - 4096) / (8 + 3 * sizeof(CT)) / 32 - kRowsPad) * 32);
  const long long cs_needed = (n + cap - 1) / cap;
  int CS = 1;
  while (CS < cs_needed) CS *= 2;
  if (CS > 16) return cudaErrorNotSupported;
  const long long srows = (n + 31) / 32;
  const int chunk = static_cast<int>((srows + CS - 1) / CS * 32);  // local rows x 32
  switch (CS) {
    case 1: return launch_rows_w<CT, 1, WIN>(p, chunk, st);
    case 2: return launch_rows_w<CT, 2, WIN>(p, chunk, st);
    case 4: return launch_rows_w<CT, 4, WIN>(p, chunk, st);
    case 8: return launch_rows_w<CT, 8, WIN>(p, chunk, st);
    default: return launch_rows_w<CT, 16, WIN>(p, chunk, st);
  }
}

cudaError_t run_rows_any(SampleParams p, long long n, bool windowed, cudaStream_t st) {
  if (p.f64)
    return windowed ? launch_rows_cs<double, true>(p, n, st) : launch_rows_cs<double, false>(p, n, st);
  return windowed ? launch_rows_cs<float, true>(p, n, st) : launch_rows_cs<float, false>(p, n, st);
}

}  // namespace pcsk
