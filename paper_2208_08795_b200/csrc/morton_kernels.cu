// Morton-row sampler for large full-window sectors (FPS / AFPS), sm_100a.
//
// Same exact iteration as the pruned-row engine (rows_kernels.cu) -- fp64
// distances in the reference's operation order, `dist <= d` writes, argmax on
// (max d, min index) -- but the rows are not runs of consecutive STORAGE
// indices. At staging every CTA sorts its points along a Z-order (Morton)
// curve of their quantised coordinates and regroups them into rows of 32
// Morton-consecutive points, so each row's bounding box is a compact cell
// instead of a slab across the cloud. The box-to-pivot test of a row then
// fails (=> the row is skipped, provably unchanged) far more often: on a
// uniform 8K-point cube ~13 of 256 rows need an update per iteration instead
// of ~44 for x-slabs.
//
// The reordering is internal: orig[] maps a slot to its sector-local index,
// row keys carry that index (the reference's tie-break,
// proj/src/sampler.cpp:137-154), outputs/trace/stats are in reference terms.
// The ordering itself only decides which rows are examined together; any
// order gives identical results.
#include <cooperative_groups.h>

#include <cstdlib>
#include <type_traits>

#include "rows_common.cuh"

namespace cg = cooperative_groups;

#ifdef PCS_PROF
__device__ unsigned long long g_mprof[8];
#define MPROF_T(v) long long v = clock64()
#else
#define MPROF_T(v)
#endif

namespace pcsk {

using namespace rows;


// Z-order cells of ~8 points for the slot bucketing (2^5 .. 2^12 cells)
__host__ __device__ __forceinline__ int morton_smem_cell_bits(int np) {
  int b = 5;
  while (b < 12 && (1 << b) * 8 < np) ++b;
  return b;
}

// Local slot layout: the CTA's storage points (sector rows R % CS == rank,
// interleaved as in rows_kernel) sorted by Morton code; slots [0, held) hold
// points, rows of 32 slots. Local row r belongs to warp r % W, lane r / W.
template <typename CT, int W, int CS>
__global__ void __launch_bounds__(W * 32) morton_rows_kernel(const SampleParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int T = W * 32;
  const int rank = CS > 1 ? static_cast<int>(cg::this_cluster().block_rank()) : 0;
  const long long flat = static_cast<long long>(blockIdx.x) / CS;
  const long long b = flat / p.M, s = flat % p.M;
  const SectorGeom g = sector_geom(p.N, p.C, p.M, s);
  const int n = g.n;
  const int srows = (n + 31) >> 5;
  const int srows_local = srows > rank ? (srows - rank + CS - 1) / CS : 0;
  const int np = p.nmax;  // slot capacity, multiple of 32
  double* d = reinterpret_cast<double*>(smem);
  CT* xs = reinterpret_cast<CT*>(d + np);
  CT* ys = xs + np;
  CT* zs = ys + np;
  uint32_t* orig = reinterpret_cast<uint32_t*>(zs + np);
  unsigned* sampled = orig + np;
  uint4* cand = reinterpret_cast<uint4*>(sampled + (np >> 5) + 4 - ((np >> 5) & 3));
  Msg* xbuf = reinterpret_cast<Msg*>(cand + 2 * W);              // [2][CS * W]
  uint64_t* xbar = reinterpret_cast<uint64_t*>(xbuf + (CS > 1 ? 2 * CS * W : 0));  // [2]
  int* scratch = reinterpret_cast<int*>(xbar + 2);                // [8]
  uint32_t* hist = reinterpret_cast<uint32_t*>(scratch + 8);      // bucketing histogram
  if (sizeof(CT) < sizeof(double) && p.f64) __trap();
  auto to_sector = [&](int jl) { return (((jl >> 5) * CS + rank) << 5) + (jl & 31); };

  // ---- 1. stage in storage order, CTA bounding box
  if (threadIdx.x < 6) scratch[threadIdx.x] = (threadIdx.x & 1) ? INT_MIN : INT_MAX;
  __syncthreads();
  {
    const long long cloud = (b * p.N + g.begin) * 3;
    float x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY, z0 = INFINITY,
          z1 = -INFINITY;
    for (int jl = threadIdx.x; jl < np; jl += T) {
      const int gj = to_sector(jl);
      const bool valid = (jl >> 5) < srows_local && gj < n;
      CT x = 0, y = 0, z = 0;
      if (valid) {
        if (p.f64) {
          const double* q = static_cast<const double*>(p.xyz) + cloud + 3LL * gj;
          x = static_cast<CT>(q[0]); y = static_cast<CT>(q[1]); z = static_cast<CT>(q[2]);
        } else {
          const float* q = static_cast<const float*>(p.xyz) + cloud + 3LL * gj;
          x = static_cast<CT>(q[0]); y = static_cast<CT>(q[1]); z = static_cast<CT>(q[2]);
        }
        x0 = fminf(x0, f_lo(x)); x1 = fmaxf(x1, f_hi(x));
        y0 = fminf(y0, f_lo(y)); y1 = fmaxf(y1, f_hi(y));
        z0 = fminf(z0, f_lo(z)); z1 = fmaxf(z1, f_hi(z));
      }
      xs[jl] = x; ys[jl] = y; zs[jl] = z;
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
  // number of points this CTA holds: all local storage rows are full but the
  // sector's last row
  int held = 0;
  if (srows_local > 0) {
    const int last_R = (srows_local - 1) * CS + rank;
    held = (srows_local - 1) * 32 + min(32, n - last_R * 32);
  }
  // ---- 2./3. Z-order bucketing: counting sort of the points by the top
  //         bits of their Morton code (cells of ~8 points; the order inside
  //         a cell is the shared-memory atomics' -- any order is exact).
  //         orig[slot] = storage slot, kNoIndex past the points
  {
    const int cb = morton_smem_cell_bits(np);
    const int cells = 1 << cb;
    uint32_t* rank_of = reinterpret_cast<uint32_t*>(d);
    uint32_t* cell_of = rank_of + np;
    for (int i = threadIdx.x; i < cells; i += T) hist[i] = 0u;
    for (int i = threadIdx.x; i < np; i += T) orig[i] = kNoIndex;
    __syncthreads();
    const float bx0 = ord2f(scratch[0]), by0 = ord2f(scratch[2]), bz0 = ord2f(scratch[4]);
    const float ext = fmaxf(fmaxf(ord2f(scratch[1]) - bx0, ord2f(scratch[3]) - by0),
                            ord2f(scratch[5]) - bz0);
    const float sc = (ext > 0.f && ext < INFINITY) ? 1023.0f / ext : 0.f;
    for (int jl = threadIdx.x; jl < np; jl += T) {
      const int gj = to_sector(jl);
      uint32_t cell = kNoIndex;
      if ((jl >> 5) < srows_local && gj < n) {
        auto q = [&](CT c, float c0) {
          const float t = fminf(fmaxf((static_cast<float>(c) - c0) * sc, 0.f), 1023.f);
          return spread3(static_cast<uint32_t>(t));
        };
        const uint32_t code = q(xs[jl], bx0) | (q(ys[jl], by0) << 1) | (q(zs[jl], bz0) << 2);
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
      if (cell != kNoIndex) orig[hist[cell] + rank_of[jl]] = static_cast<uint32_t>(jl);
    }
  }
  // ---- 4. permute coordinates (d[] is the scratch row)
  __syncthreads();
  {
    CT* tmp = reinterpret_cast<CT*>(d);
    auto permute = [&](CT* ax) {
      for (int i = threadIdx.x; i < np; i += T) {
        const uint32_t o = orig[i];
        tmp[i] = o < static_cast<uint32_t>(np) ? ax[o] : CT(0);
      }
      __syncthreads();
      for (int i = threadIdx.x; i < np; i += T) ax[i] = tmp[i];
      __syncthreads();
    };
    permute(xs);
    permute(ys);
    permute(zs);
  }
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  for (int i = threadIdx.x; i < np; i += T) {
    const bool valid = i < held;
    orig[i] = valid ? static_cast<uint32_t>(to_sector(static_cast<int>(orig[i]))) : kNoIndex;
    d[i] = valid ? kInf : 0.0;
  }
  for (int w = threadIdx.x; w < (np >> 5); w += T) sampled[w] = 0u;
  if (p.out_sector && rank == 0)
    for (int i = threadIdx.x; i < g.quota; i += T)
      p.out_sector[b * p.C + g.out_off + i] = static_cast<int>(s + p.sector_base);
  bool sub_local = false;
  if constexpr (sizeof(CT) == 4)
    for (int i = threadIdx.x; i < held; i += T)
      sub_local |= is_subnormal_f32(static_cast<float>(xs[i])) ||
                   is_subnormal_f32(static_cast<float>(ys[i])) ||
                   is_subnormal_f32(static_cast<float>(zs[i]));
  if (CS > 1 && threadIdx.x == 0) {
    mbar_init(&xbar[0], 1);  // one local arrive.expect_tx per round
    mbar_init(&xbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const bool any_sub = __syncthreads_or(sub_local) != 0;
  if constexpr (CS > 1) cg::this_cluster().sync();

  // ---- 5. per-lane row metadata (one row per lane): box + the exact
  //         maximum of the high words of the row's d[] (the full key --
  //         low word, index -- is resolved only for the winning rows)
  const int rows = (held + 31) >> 5;
  const int r = warp + W * lane;
  float bx0, bx1, by0, by1, bz0, bz1;
  uint32_t rmh;
  {
    float x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY, z0 = INFINITY,
          z1 = -INFINITY;
    if (r < rows) {
      const int e = min(32, held - r * 32);
      for (int q = 0; q < e; ++q) {
        const int i = r * 32 + q;
        x0 = fminf(x0, f_lo(xs[i])); x1 = fmaxf(x1, f_hi(xs[i]));
        y0 = fminf(y0, f_lo(ys[i])); y1 = fmaxf(y1, f_hi(ys[i]));
        z0 = fminf(z0, f_lo(zs[i])); z1 = fmaxf(z1, f_hi(zs[i]));
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
  double px, py, pz;
  float pfx = 0.f, pfy = 0.f, pfz = 0.f;
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
  for (int i = threadIdx.x; i < held; i += T)
    if (orig[i] == static_cast<uint32_t>(cur)) sampled[i >> 5] |= 1u << (i & 31);  // unique slot
  unsigned writes = 0;
  int round = 0;
#ifdef PCS_PROF
  unsigned long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif

  auto iterate = [&](auto f2f_tag) {
  constexpr bool F2F = decltype(f2f_tag)::value;
  for (int it = 1; it < g.quota; ++it) {
    MPROF_T(t0);
    float pxl, pxh, pyl, pyh, pzl, pzh;
    if constexpr (sizeof(CT) == 4) {
      pxl = pxh = pfx; pyl = pyh = pfy; pzl = pzh = pfz;
    } else {
      pxl = f_lo(px); pxh = f_hi(px); pyl = f_lo(py); pyh = f_hi(py);
      pzl = f_lo(pz); pzh = f_hi(pz);
    }
    bool need = r < rows;
    if (need) {
      const float lb = __fadd_rd(__fadd_rd(gap2(bx0, bx1, pxl, pxh), gap2(by0, by1, pyl, pyh)),
                                 gap2(bz0, bz1, pzl, pzh));
      need = !(f32_as_f64_hi_lb(__fmul_rd(lb, 0.99999904f)) > rmh);
    }
    // rows to update, two at a time (independent chains interleave)
    unsigned todo = __ballot_sync(kFull, need);
#ifdef PCS_PROF
    pacc[4] += __popc(todo);
#endif
    while (todo) {
#ifdef PCS_PROF
      pacc[5] += 1;
#endif
      const int la = __ffs(todo) - 1;
      todo &= todo - 1;
      const int lb2 = todo ? __ffs(todo) - 1 : la;
      todo &= todo - 1;
      const int ja = ((warp + W * la) << 5) + lane, jb = ((warp + W * lb2) << 5) + lane;
      double da = d[ja], db = d[jb];
      const uint32_t oa = orig[ja], ob = orig[jb];
      const double ea = dist2(to_f64<F2F>(xs[ja]), to_f64<F2F>(ys[ja]), to_f64<F2F>(zs[ja]),
                              px, py, pz);
      const double eb = dist2(to_f64<F2F>(xs[jb]), to_f64<F2F>(ys[jb]), to_f64<F2F>(zs[jb]),
                              px, py, pz);
      const bool wa = oa != kNoIndex && ea <= da;
      const bool wbb = lb2 != la && ob != kNoIndex && eb <= db;
      writes += (wa ? 1u : 0u) + (wbb ? 1u : 0u);
      if (wa) d[ja] = ea;
      if (wbb) d[jb] = eb;
      da = wa ? ea : da;
      db = wbb ? eb : db;
      const uint32_t ha = __reduce_max_sync(
          kFull, static_cast<uint32_t>(static_cast<unsigned long long>(__double_as_longlong(da)) >> 32));
      const uint32_t hb = __reduce_max_sync(
          kFull, static_cast<uint32_t>(static_cast<unsigned long long>(__double_as_longlong(db)) >> 32));
      if (lane == lb2) rmh = hb;
      if (lane == la) rmh = ha;  // lb2 == la: db is the pre-update row
    }
    if (p.trace) {
      __syncthreads();
      for (int i = threadIdx.x; i < held; i += T)
        p.trace[static_cast<long long>(it - 1) * n + orig[i]] = d[i];
    }
    MPROF_T(t1);
    // warp argmax: the rows holding the largest high word, then their exact
    // (low word, min index) from d[] -- usually a single row
    uint32_t hi = __reduce_max_sync(kFull, rmh), lo = 0u, j = kNoIndex, pos = 0u;
    {
      unsigned tied = __ballot_sync(kFull, r < rows && rmh == hi);
      while (tied) {
        const int L = __ffs(tied) - 1;
        tied &= tied - 1;
        const int row = warp + W * L, i = (row << 5) + lane;
        const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(d[i]));
        const uint32_t h0 = static_cast<uint32_t>(bits >> 32), l0 = static_cast<uint32_t>(bits);
        const uint32_t o = orig[i];
        const uint32_t l = __reduce_max_sync(kFull, h0 == hi ? l0 : 0u);
        const uint32_t m = __reduce_min_sync(
            kFull, (h0 == hi && l0 == l && o != kNoIndex) ? (o << 5) | lane : kNoIndex);
        if (l > lo || (l == lo && m < j)) {
          lo = l; j = m; pos = (static_cast<uint32_t>(row) << 5) | (m & 31u);
        }
      }
      j = j == kNoIndex ? kNoIndex : j >> 5;
    }
    MPROF_T(t2);
    auto take_local = [&](uint32_t i) {
      px = to_f64<F2F>(xs[i]); py = to_f64<F2F>(ys[i]); pz = to_f64<F2F>(zs[i]);
      if constexpr (sizeof(CT) == 4) {
        pfx = static_cast<float>(xs[i]); pfy = static_cast<float>(ys[i]);
        pfz = static_cast<float>(zs[i]);
      }
    };
    // CS > 1: every warp sends its candidate straight to every CTA of the
    // cluster (st.async + complete_tx on the receiver's mbarrier); each CTA
    // reduces the W x CS candidates itself -- no CTA barrier on the way
    constexpr unsigned kMsg = sizeof(CT) == 4 ? 32u : 40u;
    auto exchange = [&](uint32_t h, uint32_t l, uint32_t jj, uint32_t at, bool& mine_out) {
      Msg* mb = xbuf + (round & 1) * (CS * W);
      if (lane < CS) {
        const int i = jj == kNoIndex ? 0 : static_cast<int>(at);
        const uint32_t rs = mapa(mb + rank * W + warp, lane), rb = mapa(&xbar[round & 1], lane);
        st_async_v4(rs, rb, h, l, jj, at);
        if constexpr (sizeof(CT) == 4) {
          st_async_v4(rs + 16, rb, __float_as_uint(static_cast<float>(xs[i])),
                      __float_as_uint(static_cast<float>(ys[i])),
                      __float_as_uint(static_cast<float>(zs[i])), 0u);
        } else {
          const double x = static_cast<double>(xs[i]), y = static_cast<double>(ys[i]),
                       z = static_cast<double>(zs[i]);
          st_async_v4(rs + 16, rb, __double2loint(x), __double2hiint(x), __double2loint(y),
                      __double2hiint(y));
          st_async_v2(rs + 32, rb, __double2loint(z), __double2hiint(z));
        }
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
      if ((h2 | l2) != 0u || j2 != kNoIndex) {
        if constexpr (sizeof(CT) == 4) {
          pfx = __uint_as_float(w.c[0]); pfy = __uint_as_float(w.c[1]); pfz = __uint_as_float(w.c[2]);
          px = to_f64<F2F>(pfx); py = to_f64<F2F>(pfy); pz = to_f64<F2F>(pfz);
        } else {
          px = __hiloint2double(static_cast<int>(w.c[1]), static_cast<int>(w.c[0]));
          py = __hiloint2double(static_cast<int>(w.c[3]), static_cast<int>(w.c[2]));
          pz = __hiloint2double(static_cast<int>(w.c[5]), static_cast<int>(w.c[4]));
        }
      }
      mine_out = e / W == rank;
      pos = w.pos;
      hi = h2; lo = l2; j = j2;
      ++round;
    };
    // mine: this CTA holds the winner at slot `pos`
    bool mine = true;
    if constexpr (CS > 1) {
      exchange(hi, lo, j, pos, mine);
    } else {
      if constexpr (W > 1) {
        uint4* buf = cand + (round & 1) * W;
        if (lane == 0) buf[warp] = make_uint4(hi, lo, j, pos);
        __syncthreads();
        const uint4 v = lane < W ? buf[lane] : make_uint4(0, 0, kNoIndex, 0);
        hi = v.x; lo = v.y; j = v.z;
        warp_argmax(hi, lo, j);
        const unsigned who = __ballot_sync(kFull, lane < W && v.x == hi && v.y == lo && v.z == j);
        pos = buf[who ? __ffs(who) - 1 : 0].w;
        ++round;
      }
      if ((hi | lo) != 0u) take_local(pos);
    }
    MPROF_T(t3);
    if ((hi | lo) == 0u) {
      // every distance is 0: lowest unsampled index (sampler.cpp:148-154)
      uint32_t jm = kNoIndex;
      for (int i = lane; i < held; i += 32)
        if (!((sampled[i >> 5] >> (i & 31)) & 1u)) jm = min(jm, orig[i]);
      jm = __reduce_min_sync(kFull, jm);
      uint32_t at = 0;
      if (jm != kNoIndex)
        for (int i0 = 0; i0 < held; i0 += 32) {
          const int i = i0 + lane;
          const unsigned hit = __ballot_sync(kFull, i < held && orig[i] == jm);
          if (hit) { at = static_cast<uint32_t>(i0 + __ffs(hit) - 1); break; }
        }
      if constexpr (CS > 1) {
        // every warp of the CTA posts the same (1, 0, jm) candidate
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
    MPROF_T(t4);
    pacc[0] += t1 - t0; pacc[1] += t2 - t1; pacc[2] += t3 - t2; pacc[3] += t4 - t3;
#endif
  }
  };
  if (sizeof(CT) == 4 && any_sub)
    iterate(std::true_type{});
  else
    iterate(std::false_type{});
#ifdef PCS_PROF
  if (lane == 0)
    for (int q = 0; q < 6; ++q) atomicAdd(&g_mprof[q], pacc[q]);
#endif
  const unsigned ws = __reduce_add_sync(kFull, writes);
  if (p.stats) {
    unsigned long long* st = p.stats + b * 4;
    if (lane == 0 && ws) atomicAdd(st + 1, static_cast<unsigned long long>(ws));
    if (rank == 0 && threadIdx.x == 0) {
      const unsigned long long iters = static_cast<unsigned long long>(g.quota - 1);
      atomicAdd(st + 0, iters * static_cast<unsigned long long>(n));
      atomicAdd(st + 2, iters * static_cast<unsigned long long>(n));
      atomicAdd(st + 3, iters);
    }
  }
  if constexpr (CS > 1) cg::this_cluster().sync();
}

template <typename CT>
size_t morton_smem_bytes(int np, int W, int CS) {
  size_t bytes = static_cast<size_t>(np) * (8 + 3 * sizeof(CT) + 4);
  bytes += ((np >> 5) + 4 - ((np >> 5) & 3)) * 4;
  bytes += 2 * W * sizeof(uint4);
  bytes += CS > 1 ? 2 * CS * W * sizeof(Msg) : 0;
  bytes += 2 * sizeof(uint64_t) + 8 * sizeof(int);
  bytes += sizeof(uint32_t) << morton_smem_cell_bits(np);
  return bytes;
}

template <typename CT, int W, int CS>
cudaError_t launch_morton(SampleParams p, int np, cudaStream_t st) {
  p.nmax = np;
  const size_t smem = morton_smem_bytes<CT>(np, W, CS);
  if (smem > kMaxSmem) return cudaErrorNotSupported;
  if (plan("morton_rows_kernel", {sizeof(CT), W, CS})) return cudaSuccess;
  auto kern = morton_rows_kernel<CT, W, CS>;
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

// Warps per CTA: one row per lane, so W >= rows / 32. Morton rows leave far
// fewer rows to update per iteration than slab rows, so the fixed per-warp
// reduction cost argues for the smallest W that holds the rows.
int morton_w(int rows) {
  return rows <= 128 ? 4 : rows <= 256 ? 8 : 16;
}

template <typename CT, int CS>
cudaError_t launch_morton_w(SampleParams p, int chunk, cudaStream_t st) {
  const int rows = (chunk + 31) / 32;
  const int np = (rows + kRowsPad) * 32;
  const int w = morton_w(rows);
  if (rows > 32 * w) return cudaErrorNotSupported;
  switch (w) {
    case 4: return launch_morton<CT, 4, CS>(p, np, st);
    case 8: return launch_morton<CT, 8, CS>(p, np, st);
    default: return launch_morton<CT, 16, CS>(p, np, st);
  }
}

// Smallest cluster whose per-CTA share (rows interleaved over the CTAs)
// fits shared memory with its exchange buffers.
template <typename CT>
cudaError_t launch_morton_cs(SampleParams p, long long n, cudaStream_t st) {
  const long long srows = (n + 31) / 32;
  for (int CS = 1; CS <= 16; CS *= 2) {
    const int rows = static_cast<int>((srows + CS - 1) / CS);
    const int w = morton_w(rows);
    if (rows > 32 * w) continue;
    if (morton_smem_bytes<CT>((rows + kRowsPad) * 32, w, CS) > kMaxSmem) continue;
    const int chunk = rows * 32;
    switch (CS) {
      case 1: return launch_morton_w<CT, 1>(p, chunk, st);
      case 2: return launch_morton_w<CT, 2>(p, chunk, st);
      case 4: return launch_morton_w<CT, 4>(p, chunk, st);
      case 8: return launch_morton_w<CT, 8>(p, chunk, st);
      default: return launch_morton_w<CT, 16>(p, chunk, st);
    }
  }
  return cudaErrorNotSupported;
}

cudaError_t run_morton_any(SampleParams p, long long n, cudaStream_t st) {
  return p.f64 ? launch_morton_cs<double>(p, n, st) : launch_morton_cs<float>(p, n, st);
}

}  // namespace pcsk
