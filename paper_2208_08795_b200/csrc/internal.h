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

void set_error(const std::string& msg);
void clear_error();

}  // namespace pcs_internal
