// Device helpers shared by the sampler and sort kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pcsk {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kNoIndex = 0xffffffffu;

// SplitMix64, proj/include/pcs/rng.hpp:16-30 (next, below by rejection).
__device__ __forceinline__ uint64_t splitmix_next(uint64_t& state) {
  uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t splitmix_below(uint64_t state, uint64_t bound) {
  const uint64_t threshold = (0 - bound) % bound;
  for (;;) {
    const uint64_t r = splitmix_next(state);
    if (r >= threshold) return r % bound;
  }
}

// One sector of one cloud: storage range, quota and output offset, from the
// reference's remainder rule (proj/src/sectors.cpp:9-36).
struct SectorGeom {
  int begin;    // first point, index within the cloud
  int n;        // points in the sector
  int quota;    // samples owed
  int out_off;  // first output slot of this sector within the cloud's row
};

__device__ __forceinline__ SectorGeom sector_geom(long long N, long long C, long long M,
                                                  long long s) {
  const long long nb = N / M, nr = N % M, cb = C / M, cr = C % M;
  SectorGeom g;
  g.n = static_cast<int>(nb + (s < nr ? 1 : 0));
  g.begin = static_cast<int>(s * nb + (s < nr ? s : nr));
  g.quota = static_cast<int>(cb + (s < cr ? 1 : 0));
  g.out_off = static_cast<int>(s * cb + (s < cr ? s : cr));
  return g;
}

// Squared distance exactly as proj/src/sampler.cpp:121-124 evaluates it in
// its default (no-FMA) build: three subtractions, three products, and the
// left-to-right sum ((dx*dx + dy*dy) + dz*dz), each rounded to nearest.
__device__ __forceinline__ double dist2(double x, double y, double z, double px, double py,
                                        double pz) {
  const double dx = __dsub_rn(x, px);
  const double dy = __dsub_rn(y, py);
  const double dz = __dsub_rn(z, pz);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// Argmax key: distances are >= 0 (or +inf), so their IEEE bits order like
// the values as unsigned integers. Winner = max distance, then min index
// (the reference's "first index holding the max", sampler.cpp:137-154).
// Three redux.sync steps; every lane returns the warp's winner.
__device__ __forceinline__ void warp_argmax(uint32_t& hi, uint32_t& lo, uint32_t& j) {
  const uint32_t mh = __reduce_max_sync(kFull, hi);
  const uint32_t ml = __reduce_max_sync(kFull, hi == mh ? lo : 0u);
  const uint32_t mj = __reduce_min_sync(kFull, (hi == mh && lo == ml) ? j : kNoIndex);
  hi = mh;
  lo = ml;
  j = mj;
}

// Exact fp32 -> fp64 widening on the integer pipe (F2F.F64.F32 issues on the
// XU at ~1/4 of the DADD rate and saturates it in the samplers' inner
// loops). Exact for normal numbers and +-0, which is all the kernels stage
// for fp32 input (stagers route a sector containing a subnormal to the F2F
// path; inf/NaN are outside the reference's precondition).
__device__ __forceinline__ double widen_f32(float f) {
  const uint32_t b = __float_as_uint(f), a = b & 0x7fffffffu;
  const uint32_t hi = (a ? (a >> 3) + 0x38000000u : 0u) | (b & 0x80000000u);
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(b << 29));
}

__device__ __forceinline__ bool is_subnormal_f32(float f) {
  const uint32_t a = __float_as_uint(f) & 0x7fffffffu;
  return a != 0 && a < 0x00800000u;
}

// High word of the fp64 value of a non-negative fp32 (subnormals -> 0, a
// lower bound). Used to compare an fp32 lower bound against an fp64 key.
__device__ __forceinline__ uint32_t f32_as_f64_hi_lb(float f) {
  const uint32_t a = __float_as_uint(f) & 0x7fffffffu;
  return a >= 0x00800000u ? (a >> 3) + 0x38000000u : 0u;
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace pcsk
