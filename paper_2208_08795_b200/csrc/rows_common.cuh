// Helpers shared by the pruned-row samplers (rows_kernels.cu,
// morton_kernels.cu): cluster candidate exchange, fp32 box bounds, keys.
#pragma once

#include <cooperative_groups.h>

#include "sampler_common.cuh"

namespace pcsk {

namespace rows {

constexpr int kRowsPad = 2;  // zero rows after each chunk (pair processing)

struct alignas(16) Cand {  // 64 B: st.async writes 16 B-aligned pieces
  uint32_t hi, lo, j;
  float fx, fy, fz, pad0, pad1;
  double x, y, z, pad2;
};

// Cluster exchange without a cluster-wide barrier: each CTA stores its
// candidate into every CTA's slot and arrives (release, cluster scope) on
// that CTA's mbarrier for the round; each CTA waits (acquire) on its own.
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"
               :: "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* local_bar, int target_rank) {
  unsigned local = static_cast<unsigned>(__cvta_generic_to_shared(local_bar)), remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(target_rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(remote) : "memory");
}
// Asynchronous DSMEM stores that complete-tx on the receiver's mbarrier
// (no release fence on the sender); the receiver arms the round with one
// local arrive.expect_tx for the bytes all senders will deliver.
__device__ __forceinline__ uint32_t mapa(const void* local, int target_rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(remote) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(local))), "r"(target_rank));
  return remote;
}
__device__ __forceinline__ void st_async_v4(uint32_t raddr, uint32_t rbar, uint32_t a, uint32_t b,
                                            uint32_t c, uint32_t d) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
               :: "r"(raddr), "r"(a), "r"(b), "r"(c), "r"(d), "r"(rbar) : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t raddr, uint32_t rbar, uint32_t a, uint32_t b) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];"
               :: "r"(raddr), "r"(a), "r"(b), "r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n .reg .pred done;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 done, [%0], %1;\n"
      " @!done bra WAIT_%=;\n}" :: "r"(a), "r"(parity) : "memory");
}

template <bool F2F>
__device__ __forceinline__ double to_f64(float v) { return F2F ? static_cast<double>(v) : widen_f32(v); }
template <bool F2F>
__device__ __forceinline__ double to_f64(double v) { return v; }

__device__ __forceinline__ float f_lo(float v) { return v; }
__device__ __forceinline__ float f_hi(float v) { return v; }
__device__ __forceinline__ float f_lo(double v) { return __double2float_rd(v); }
__device__ __forceinline__ float f_hi(double v) { return __double2float_ru(v); }

// Lower bound (round-down fp32) of the squared distance from the pivot
// interval [pl, ph] to the box [b0, b1] on one axis.
__device__ __forceinline__ float gap2(float b0, float b1, float pl, float ph) {
  const float g = fmaxf(fmaxf(__fsub_rd(b0, ph), __fsub_rd(pl, b1)), 0.0f);
  return __fmul_rd(g, g);
}

__device__ __forceinline__ bool key_gt(uint32_t h1, uint32_t l1, uint32_t j1, uint32_t h2,
                                       uint32_t l2, uint32_t j2) {
  return h1 > h2 || (h1 == h2 && (l1 > l2 || (l1 == l2 && j1 < j2)));
}

// ---- Morton-row engines
__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // 10 bits -> every 3rd bit
  v &= 1023u;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

// float <-> int with the same order (for redux / atomic min-max of floats)
__device__ __forceinline__ int f2ord(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

// One warp's candidate as seen by every CTA of the cluster: key, sector-local
// index, slot in the sender CTA, pivot coordinates (3 floats or 3 doubles).
struct alignas(16) Msg {
  uint32_t hi, lo, j, pos;
  uint32_t c[6];
  uint32_t pad[2];
};

}  // namespace rows

}  // namespace pcsk
