/*
 * pcs_gpu.h -- C-ABI of the B200-native sampling hot path (FPS / AFPS /
 * NPDU-FPS / NPDU-AFPS and the per-cloud axis sort of arXiv 2208.08795).
 *
 * Plain C types only: pointers, sizes, status codes. No exceptions, no torch
 * types. Everything above this boundary (the C++ drop-in `pcs::` API in
 * include/pcs/, the Python `_core` module, the torch batched op) calls these
 * entry points; everything below is sm_100a CUDA in
 * paper_2208_08795_b200/csrc/.
 *
 * Which reference interface each entry replaces (paths relative to
 * /root/reference/proj):
 *
 *   pcs_sample_host      <- the pybind sampler lambdas
 *                           bindings/pcsample_module.cpp:150-190
 *                           (fps / afps / npdu_fps / npdu_afps), i.e.
 *                           pcs::fps/afps/npdu_fps/npdu_afps,
 *                           include/pcs/sampler.hpp:41-66, src/sampler.cpp:171-204
 *   pcs_local_fps_host   <- pcs::detail::local_fps (+ DistanceTrace),
 *                           include/pcs/sampler.hpp:34-37, src/sampler.cpp:85-167
 *   pcs_exact_sort_host  <- pcs::exact_sort, include/pcs/order.hpp:10,
 *                           src/order.cpp:11-24; pybind exact_sort
 *                           bindings/pcsample_module.cpp:122-127
 *   pcs_gpu_sample       <- batched, device-resident, stream-ordered form of
 *                           the four samplers (no reference equivalent: the
 *                           reference is per-cloud only)
 *   pcs_gpu_sort_axis    <- batched device form of exact_sort
 *   pcs_sample_host_batch <- the per-cloud samplers called over a batch of
 *                           host clouds (+ exact_sort), in one pipelined call
 *   pcs_sample_host_multi <- the same batch spread over several devices: the
 *                           cross-GPU form of the reference's sector work
 *                           split + ordered merge, src/sampler.cpp:25-79
 *
 * Semantics are the reference's, bit for bit: indices, sector_of and the
 * OpStats counters (include/pcs/op_stats.hpp:10-25) equal the reference CPU
 * implementation's on the same coordinates. Distances are evaluated in fp64
 * as ((dx*dx + dy*dy) + dz*dz) with no FMA contraction (src/sampler.cpp:
 * 121-124); fp32 inputs are widened exactly, as the reference's f32_bin
 * reader does (src/io.cpp:84-86).
 *
 * Errors: argument errors return PCS_ERR_INVALID_ARGUMENT and leave the
 * reference's exact std::invalid_argument message in pcs_last_error()
 * (validated on the host, in the reference's order, before any launch).
 * CUDA failures return PCS_ERR_CUDA. The message buffer is thread-local.
 */
#ifndef PCS_GPU_H_
#define PCS_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCS_GPU_ABI_VERSION 2

typedef enum {
  PCS_OK = 0,
  PCS_ERR_INVALID_ARGUMENT = 1, /* reference std::invalid_argument */
  PCS_ERR_CUDA = 2,             /* CUDA runtime / launch failure   */
  PCS_ERR_UNSUPPORTED = 3       /* e.g. no sm_100 device           */
} pcs_status;

/* Matches pcs::Method minus the out-of-scope baselines (rps, grid). */
typedef enum {
  PCS_METHOD_FPS = 1,
  PCS_METHOD_AFPS = 2,
  PCS_METHOD_NPDU_FPS = 3,
  PCS_METHOD_NPDU_AFPS = 4
} pcs_method;

typedef enum { PCS_DTYPE_F32 = 0, PCS_DTYPE_F64 = 1 } pcs_coord_dtype;
typedef enum { PCS_INDEX_I32 = 0, PCS_INDEX_I64 = 1 } pcs_index_dtype;

/* pcs::SeedPolicy (include/pcs/sampler_spec.hpp:13-17). */
typedef enum { PCS_RANDOM_FIRST_POINT = 0, PCS_FIXED_FIRST_POINT = 1 } pcs_seed_policy;

/* Batched, device-resident sampling request. B clouds of N points each,
 * AoS xyz (the f32_bin layout when coord_dtype is F32). */
typedef struct pcs_gpu_args {
  int32_t method;            /* pcs_method                                   */
  int32_t coord_dtype;       /* pcs_coord_dtype                              */
  const void* xyz;           /* device, (B, N, 3)                            */
  int64_t batch;             /* B >= 1                                       */
  int64_t n;                 /* N points per cloud                           */
  int64_t c;                 /* samples per cloud                            */
  int64_t m;                 /* sectors (AFPS variants; ignored otherwise)   */
  int64_t k;                 /* update window (NPDU variants; else ignored)  */
  int32_t seed_policy;       /* pcs_seed_policy                              */
  uint64_t seed;             /* per-sector stream is seed ^ sector_id        */
  const uint64_t* seeds;     /* device (B), optional per-cloud seed override */
  int32_t index_dtype;       /* pcs_index_dtype                              */
  void* out_indices;         /* device (B, c): absolute indices, sector order*/
  int32_t* out_sector;       /* device (B, c), optional: sector_of           */
  uint64_t* out_stats;       /* device (B, 4), optional: evals, writes,
                                argmax_scans, iterations                     */
  /* Sharding (one cloud's sectors split across GPUs): this call's clouds are
   * the storage slice that starts at point `index_base` and sector
   * `sector_base` of a larger cloud. Output indices are offset by
   * index_base; sector ids (sector_of, and the seed ^ sector stream) by
   * sector_base. Zero for an ordinary call. */
  int64_t index_base;
  int64_t sector_base;
  /* Optional device (B, N) int32 sort permutation (sorted position ->
   * storage index, as pcs_gpu_sort_axis returns it): sample the clouds in
   * that order, i.e. exactly as if xyz had been replaced by the sorted copy
   * (indices refer to sorted positions) -- without the copy. NULL: storage
   * order. Added in ABI version 2. */
  const int32_t* perm;
} pcs_gpu_args;

/* Stream-ordered batched sampling. `stream` is a cudaStream_t (NULL = legacy
 * default stream). Returns after the launches are enqueued. */
int pcs_gpu_sample(const pcs_gpu_args* args, void* stream);
/* The same entry under the name SURVEY.md §8(b) gives it. */
int pcs_gpu_sample_batched(const pcs_gpu_args* args, void* stream);

/* Stable ascending sort of every cloud along `axis` (0 x, 1 y, 2 z) with the
 * reference's operator< on the coordinate (-0.0 == +0.0, ties keep storage
 * order). Writes, each optionally (NULL skips it), the gathered cloud (same
 * dtype as the input; may not alias xyz) and the permutation (int32, sorted
 * position -> original index). The permutation alone plus
 * pcs_gpu_args.perm is the cheap way to sample sorted clouds.
 * Stream-ordered. */
int pcs_gpu_sort_axis(int32_t coord_dtype, const void* xyz, int64_t batch, int64_t n,
                      int32_t axis, void* out_xyz, int32_t* out_perm, void* stream);

/* Host-buffer drop-ins for the reference's per-cloud API. xyz is host
 * float64 (N, 3) as the pybind layer passes it; results are host int64 /
 * uint64 like pcsample._core returns. Synchronous. `threads` is accepted
 * for signature parity and ignored (the GPU schedule is deterministic). */
int pcs_sample_host(int32_t method, const double* xyz, int64_t n, int64_t c, int64_t m,
                    int64_t k, int32_t seed_policy, uint64_t seed, uint32_t threads,
                    int64_t* out_indices, int64_t* out_sector, uint64_t* out_stats);

/* Host-buffer batch: the reference's per-cloud samplers over B clouds in one
 * call (what a caller of pcs::npdu_afps & co. does in a loop over its
 * clouds). Same fields as pcs_gpu_args, but xyz, out_indices, out_sector and
 * out_stats are HOST pointers (seeds, when given, too). The batch streams
 * through the device in `chunks` pieces (<= 0: a default): the copy of
 * piece i+1 overlaps the axis sort + sampling of piece i, results return
 * as pieces complete. sort_axis -1: no sort; 0/1/2: the clouds are first
 * stably sorted along x/y/z (exact_sort) and indices refer to the sorted
 * clouds; out_perm (host int32 (B, N), optional) receives the sort
 * permutation. Pinned host memory gives the overlap; pageable memory works.
 * Synchronous. */
int pcs_sample_host_batch(const pcs_gpu_args* host_args, int32_t sort_axis, int32_t* out_perm,
                          int32_t chunks);

/* Multi-device host batch (one process, several GPUs): as
 * pcs_sample_host_batch, with the work split over `devices[0..ndevices)`
 * (CUDA ordinals; repeats allowed -- shards on one device run in turn).
 * Clouds split by cloud, device r taking the r-th of ndevices contiguous
 * runs (the first B % ndevices one cloud larger, partition_sectors' rule,
 * src/sectors.cpp:9-24). A single cloud under AFPS / NPDU-AFPS with
 * m >= ndevices splits by sector run instead: every device copies and sorts
 * the whole cloud, samples its sectors with the global index / sector bases
 * (so indices, sector_of and the seed ^ sector starts are the one-device
 * ones), and its indices fill its slots of the row; stats are summed.
 * Results are written straight into the host outputs -- the only "gather".
 * No collective and no peer traffic. Synchronous; bit-identical to
 * pcs_sample_host_batch on one device. */
int pcs_sample_host_multi(const pcs_gpu_args* host_args, int32_t sort_axis, int32_t* out_perm,
                          const int32_t* devices, int32_t ndevices);

/* detail::local_fps over one storage range [sector_begin, sector_end) of a
 * cloud. k < 0 means no window (std::nullopt); k == 0 is rejected exactly as
 * the reference rejects window_k == 0. trace, when non-NULL, must
 * hold (quota-1) * (sector_end-sector_begin) doubles and receives the
 * DistanceTrace snapshots. */
int pcs_local_fps_host(const double* xyz, int64_t n, int64_t sector_begin,
                       int64_t sector_end, int64_t quota, int64_t k, int32_t seed_policy,
                       uint64_t seed, int64_t* out_indices, uint64_t* out_stats,
                       double* trace);

/* exact_sort on a host float64 cloud. out_xyz (N,3) and out_perm (N) may be
 * NULL independently. */
int pcs_exact_sort_host(const double* xyz, int64_t n, int32_t axis, double* out_xyz,
                        int64_t* out_perm);

/* Sample-quality metrics (proj/src/metrics.cpp:16-52),
 * bit-identical to the reference's: coverage_radius = max over points of the
 * distance to the nearest sample; separation = min pairwise distance among
 * the samples. Batched device form: samples (B, c) int32/int64, out (B)
 * doubles; an out-of-range sample index yields NaN for that cloud. Host form:
 * one float64 (N, 3) cloud, int64 samples, reference argument checks and
 * messages ("coverage_radius: sample set is empty", "... index out of
 * range", "separation: need at least 2 samples"). */
int pcs_gpu_coverage_radius(int32_t coord_dtype, const void* xyz, int64_t batch, int64_t n,
                            int32_t index_dtype, const void* samples, int64_t c, double* out,
                            void* stream);
int pcs_gpu_separation(int32_t coord_dtype, const void* xyz, int64_t batch, int64_t n,
                       int32_t index_dtype, const void* samples, int64_t c, double* out,
                       void* stream);
int pcs_coverage_radius_host(const double* xyz, int64_t n, const int64_t* samples, int64_t c,
                             double* out);
int pcs_separation_host(const double* xyz, int64_t n, const int64_t* samples, int64_t c,
                        double* out);

/* Cloud files (proj/src/io.cpp:32-122). format 0 = xyz_text,
 * 1 = f32_bin. pcs_read_cloud_host returns N and copies min(N, capacity)
 * points (call with out_xyz NULL to size), or -1 with the reference's
 * std::runtime_error message in pcs_last_error(). */
long long pcs_read_cloud_host(const char* path, int32_t format, double* out_xyz, int64_t capacity);
int pcs_write_cloud_host(const char* path, int32_t format, const double* xyz, int64_t n);

/* The kernel pcs_gpu_sample would launch for `args` (batch, n, c, m, k,
 * method, coord_dtype and trace-free; pointers are ignored), e.g.
 * "npdu_tmem_kernel<5,1024>", written NUL-terminated into name[capacity].
 * Touches no device. Validation errors as pcs_gpu_sample. */
int pcs_kernel_family(const pcs_gpu_args* args, char* name, size_t capacity);

/* Test hook: re-read the PCS_* engine-override environment variables, which
 * are otherwise read once per process. */
void pcs_debug_reload_knobs(void);

/* Last error message of the calling thread ("" after success). */
const char* pcs_last_error(void);
const char* pcs_status_string(int status);
const char* pcs_gpu_status_string(int status); /* alias of pcs_status_string */
int pcs_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PCS_GPU_H_ */
