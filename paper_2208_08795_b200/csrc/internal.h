// Host-side internals shared by the C-ABI translation units.
#pragma once

#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "pcs_gpu.h"

namespace pcs_internal {

// Stream-ordered workspace from the device's default memory pool, which is
// set (once per device) to keep freed memory instead of returning it to the
// driver at every synchronisation -- otherwise each call re-maps its
// workspace (measured: a 1M-point sort 0.27 ms warm vs 0.48 ms re-mapped).
cudaError_t workspace_alloc(void** p, size_t bytes, cudaStream_t st);

// Argument validation in the reference's order with its exact messages
// (proj/src/sampler.cpp:20-23 check_sample_count, proj/src/sectors.cpp:9-51
// SectorPlan::make, proj/src/sampler.cpp:89-94 local_fps). Returns PCS_OK
// or PCS_ERR_INVALID_ARGUMENT with *msg set.
int validate_sample(int method, int64_t n, int64_t c, int64_t m, int64_t k, std::string* msg);

// Enqueues the batched sampler (args already validated). Zeroes out_stats.
cudaError_t launch_sample(const pcs_gpu_args& a, cudaStream_t stream, std::string* msg);

// The kernel launch_sample would make for `a` (no device work): 0 and its
// name (e.g. "npdu_tmem_kernel<5,1024>"), or -1 with *msg when none fits.
int plan_sample(const pcs_gpu_args& a, std::string* name, std::string* msg);

// Enqueues the batched stable axis sort.
cudaError_t launch_sort(int coord_dtype, const void* xyz, int64_t batch, int64_t n, int axis,
                        void* out_xyz, int32_t* out_perm, cudaStream_t stream);

// Debug path for pcs_local_fps_host: one sector [sb, se) of a single cloud,
// optional DistanceTrace buffer on the device.
cudaError_t launch_local_fps(const double* xyz, int64_t n, int64_t sb, int64_t se,
                             int64_t quota, int64_t k, int random_first, uint64_t seed,
                             int64_t* out_idx, uint64_t* out_stats, double* trace,
                             cudaStream_t stream, std::string* msg);

// Batched coverage_radius (which = 0) / separation (which = 1): out[b] is
// the metric of cloud b (NaN when a sample index is out of range).
cudaError_t launch_metric(int which, int coord_dtype, const void* xyz, int64_t batch, int64_t n,
                          int index_dtype, const void* idx, int64_t c, double* out,
                          cudaStream_t stream);

// Engine-selection overrides for tests and A/B measurements, read from the
// environment ONCE per process (never per launch); pcs_debug_reload_knobs()
// re-reads them (test hook).
struct Knobs {
  int sampler = 0;            // PCS_SAMPLER: 0 auto, 1 "rows" (pruned rows), 2 "stream"
  bool morton = true;         // PCS_MORTON=0: storage-order rows instead of Morton rows
  bool morton_tmem = true;    // PCS_MORTON_TMEM=0: Morton rows keep d in shared memory
  long long morton_min = -1;  // PCS_MORTON_MIN: full-window Morton crossover (points)
  long long npdu_wide = -1;   // PCS_NPDU_WIDE: most sectors the W-warp NPDU form takes
  bool npdu_tmem = true;      // PCS_NPDU_TMEM=0: one-warp NPDU keeps d in shared memory
  bool tiny = true;           // PCS_TINY=0: tiny sectors keep a warp each (fps_full_kernel)
  bool npdu_big = true;       // PCS_NPDU_BIG=0: no TMEM row engine for big windowed sectors
  bool sort_radix = true;     // PCS_SORT_RADIX=0: bitonic networks instead of on-chip radix
  bool sort_bucket = true;    // PCS_SORT_BUCKET=0: 38+ clouds <= 32K take the radix CTA sort
  bool cluster = true;        // PCS_CLUSTER=0: no cluster-spread full-window kernel
  int cluster_cs = 8;         // PCS_CLUSTER_CS: largest cluster it may use (2, 4 or 8)
  int npdu_key = -1;          // PCS_NPDU_KEY: force the TMEM NPDU row-key form (0-3)
  int morton_w = 0;           // PCS_MORTON_W: force the TMEM Morton engine's warps per CTA (4, 8, 16)
};
const Knobs& knobs();
void reload_knobs();

void set_error(const std::string& msg);
void clear_error();

}  // namespace pcs_internal
