// C-ABI entry points (include/pcs_gpu.h): host-side validation in the
// reference's order, error plumbing, and the host-buffer drop-ins that the
// reference-facing bindings call.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"
#include "pcs_gpu.h"

namespace pcs_internal {

cudaError_t workspace_alloc(void** p, size_t bytes, cudaStream_t st) {
  // one private stream-ordered pool per device (< 64), created on first use:
  // it keeps freed workspace mapped for the next call (release threshold =
  // max) without changing the behaviour of the device's default pool, which
  // the caller's allocator (e.g. torch) may use
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, st);
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      e = cudaMemPoolCreate(&pools[dev], &props);
      if (e != cudaSuccess) {
        pools[dev] = nullptr;
        return e;
      }
      unsigned long long keep = ~0ull;
      cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool = pools[dev];
  }
  return cudaMallocFromPoolAsync(p, bytes, pool, st);
}

namespace {
thread_local std::string g_error;

Knobs read_knobs() {
  Knobs k;
  auto env = [](const char* name) -> const char* { return std::getenv(name); };
  if (const char* v = env("PCS_SAMPLER")) k.sampler = std::string(v) == "rows" ? 1 : std::string(v) == "stream" ? 2 : 0;
  if (const char* v = env("PCS_MORTON")) k.morton = v[0] != '0';
  if (const char* v = env("PCS_MORTON_TMEM")) k.morton_tmem = v[0] != '0';
  if (const char* v = env("PCS_MORTON_MIN")) k.morton_min = std::atoll(v);
  if (const char* v = env("PCS_NPDU_WIDE")) k.npdu_wide = std::atoll(v);
  if (const char* v = env("PCS_NPDU_TMEM")) k.npdu_tmem = v[0] != '0';
  if (const char* v = env("PCS_NPDU_KEY")) k.npdu_key = std::atoi(v);
  if (const char* v = env("PCS_MORTON_W")) k.morton_w = std::atoi(v);
  if (const char* v = env("PCS_TINY")) k.tiny = v[0] != '0';
  if (const char* v = env("PCS_NPDU_BIG")) k.npdu_big = v[0] != '0';
  if (const char* v = env("PCS_SORT_RADIX")) k.sort_radix = v[0] != '0';
  if (const char* v = env("PCS_SORT_BUCKET")) k.sort_bucket = v[0] != '0';
  if (const char* v = env("PCS_CLUSTER")) k.cluster = v[0] != '0';
  if (const char* v = env("PCS_CLUSTER_CS")) k.cluster_cs = std::atoi(v) >= 8 ? 8 : std::atoi(v) >= 4 ? 4 : 2;
  return k;
}

// Snapshots are immutable and never freed (a reload is a test-only event),
// so a launch racing a reload reads either snapshot, never a torn one.
std::atomic<const Knobs*> g_knobs{nullptr};

const char* who(int method) {
  switch (method) {
    case PCS_METHOD_FPS: return "fps";
    case PCS_METHOD_AFPS: return "afps";
    case PCS_METHOD_NPDU_FPS: return "npdu_fps";
    case PCS_METHOD_NPDU_AFPS: return "npdu_afps";
  }
  return "run_sampler";
}

int cuda_fail(cudaError_t e, const std::string& extra = "") {
  if (e == cudaErrorNotSupported && !extra.empty()) {
    set_error(extra);
    return PCS_ERR_UNSUPPORTED;
  }
  set_error(std::string("CUDA error: ") + cudaGetErrorString(e) + (extra.empty() ? "" : " (" + extra + ")"));
  return PCS_ERR_CUDA;
}

// RAII device buffer on a stream (stream-ordered allocator).
struct DevBuf {
  void* p = nullptr;
  cudaStream_t s;
  explicit DevBuf(cudaStream_t st) : s(st) {}
  cudaError_t alloc(size_t bytes) {
    return pcs_internal::workspace_alloc(&p, bytes ? bytes : 16, s);
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

}  // namespace

const Knobs& knobs() {
  const Knobs* k = g_knobs.load(std::memory_order_acquire);
  if (!k) {
    const Knobs* fresh = new Knobs(read_knobs());
    if (!g_knobs.compare_exchange_strong(k, fresh, std::memory_order_acq_rel)) delete fresh;
    else k = fresh;
  }
  return *k;
}

void reload_knobs() { g_knobs.store(new Knobs(read_knobs()), std::memory_order_release); }

void set_error(const std::string& msg) { g_error = msg; }
void clear_error() { g_error.clear(); }

int validate_sample(int method, int64_t n, int64_t c, int64_t m, int64_t k, std::string* msg) {
  if (method < PCS_METHOD_FPS || method > PCS_METHOD_NPDU_AFPS) {
    *msg = "run_sampler: unknown method";
    return PCS_ERR_INVALID_ARGUMENT;
  }
  const std::string w = who(method);
  // check_sample_count, proj/src/sampler.cpp:20-23
  if (c < 1) { *msg = w + ": c must be >= 1"; return PCS_ERR_INVALID_ARGUMENT; }
  if (c > n) { *msg = w + ": c exceeds point count"; return PCS_ERR_INVALID_ARGUMENT; }
  const bool sectored = method == PCS_METHOD_AFPS || method == PCS_METHOD_NPDU_AFPS;
  if (sectored) {
    // SectorPlan::make -> partition_sectors -> allocate_samples -> feasibility,
    // proj/src/sectors.cpp:9-51
    if (m < 1) { *msg = "partition_sectors: m must be >= 1"; return PCS_ERR_INVALID_ARGUMENT; }
    if (m > n) { *msg = "partition_sectors: m exceeds point count"; return PCS_ERR_INVALID_ARGUMENT; }
    if (m > c) { *msg = "allocate_samples: m exceeds sample count"; return PCS_ERR_INVALID_ARGUMENT; }
    // First infeasible sector, if any: sizes nb+[s<nr], quotas cb+[s<cr].
    const int64_t nb = n / m, nr = n % m, cb = c / m, cr = c % m;
    int64_t bad = -1;
    if (cb > nb) bad = 0;
    else if (cb == nb && cr > nr) bad = nr;
    if (bad >= 0) {
      *msg = "sector " + std::to_string(bad) + " holds " + std::to_string(nb + (bad < nr)) +
             " points but owes " + std::to_string(cb + (bad < cr)) + " samples";
      return PCS_ERR_INVALID_ARGUMENT;
    }
  }
  // local_fps, proj/src/sampler.cpp:89-94 (range and quota hold by now)
  const bool windowed = method == PCS_METHOD_NPDU_FPS || method == PCS_METHOD_NPDU_AFPS;
  if (windowed && k < 1) { *msg = "local_fps: window size must be >= 1"; return PCS_ERR_INVALID_ARGUMENT; }
  if (n > 0x7fffffffLL) { *msg = "clouds above 2^31-1 points are not supported"; return PCS_ERR_UNSUPPORTED; }
  return PCS_OK;
}

}  // namespace pcs_internal

using namespace pcs_internal;

extern "C" {

int pcs_abi_version(void) { return PCS_GPU_ABI_VERSION; }

const char* pcs_last_error(void) { return g_error.c_str(); }

const char* pcs_status_string(int status) {
  switch (status) {
    case PCS_OK: return "ok";
    case PCS_ERR_INVALID_ARGUMENT: return "invalid argument";
    case PCS_ERR_CUDA: return "CUDA error";
    case PCS_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

int pcs_gpu_sample(const pcs_gpu_args* a, void* stream) {
  clear_error();
  if (!a) { set_error("pcs_gpu_sample: null args"); return PCS_ERR_INVALID_ARGUMENT; }
  std::string msg;
  const int rc = validate_sample(a->method, a->n, a->c, a->m, a->k, &msg);
  if (rc) { set_error(msg); return rc; }
  if (a->batch < 0) { set_error("pcs_gpu_sample: batch must be >= 0"); return PCS_ERR_INVALID_ARGUMENT; }
  if (a->batch == 0) return PCS_OK;
  if (!a->xyz || !a->out_indices) { set_error("pcs_gpu_sample: null buffer"); return PCS_ERR_INVALID_ARGUMENT; }
  const cudaError_t e = launch_sample(*a, static_cast<cudaStream_t>(stream), &msg);
  return e == cudaSuccess ? PCS_OK : cuda_fail(e, msg);
}

int pcs_gpu_sample_batched(const pcs_gpu_args* a, void* stream) { return pcs_gpu_sample(a, stream); }

const char* pcs_gpu_status_string(int status) { return pcs_status_string(status); }

int pcs_kernel_family(const pcs_gpu_args* a, char* name, size_t capacity) {
  clear_error();
  if (!a) { set_error("pcs_kernel_family: null args"); return PCS_ERR_INVALID_ARGUMENT; }
  std::string msg;
  const int rc = validate_sample(a->method, a->n, a->c, a->m, a->k, &msg);
  if (rc) { set_error(msg); return rc; }
  std::string plan;
  if (plan_sample(*a, &plan, &msg) != 0) { set_error(msg); return PCS_ERR_UNSUPPORTED; }
  if (name && capacity) {
    const size_t len = std::min(capacity - 1, plan.size());
    std::memcpy(name, plan.data(), len);
    name[len] = '\0';
  }
  return PCS_OK;
}

void pcs_debug_reload_knobs(void) { reload_knobs(); }

int pcs_gpu_sort_axis(int32_t coord_dtype, const void* xyz, int64_t batch, int64_t n,
                      int32_t axis, void* out_xyz, int32_t* out_perm, void* stream) {
  clear_error();
  if (axis < 0 || axis > 2) { set_error("axis must be x, y, or z"); return PCS_ERR_INVALID_ARGUMENT; }
  if (n > 0x7fffffffLL) { set_error("clouds above 2^31-1 points are not supported"); return PCS_ERR_UNSUPPORTED; }
  const cudaError_t e = launch_sort(coord_dtype, xyz, batch, n, axis, out_xyz, out_perm,
                                    static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? PCS_OK : cuda_fail(e);
}

namespace {

// One copy stream + kWorkers compute streams + events per device, created
// once and kept (creating streams per call costs more than sampling a small
// batch); host-buffer calls on one device serialise on its mutex.
constexpr int kWorkers = 4, kEvents = 64;
struct DevStreams {
  std::mutex mu;
  cudaStream_t copy = nullptr, work[kWorkers] = {};
  cudaEvent_t ev[kEvents] = {};
  bool ok = false;
  // pinned host staging for the per-cloud drop-in entries (grown on demand,
  // used under `mu`): copies from pinned memory are true async DMA, while a
  // pageable source goes through the driver's bounce buffers
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
};

// The caller holds ds.mu; previous users of the buffer have synchronised.
cudaError_t pinned_scratch(DevStreams& ds, size_t bytes, void** out) {
  if (bytes > ds.pinned_bytes) {
    if (ds.pinned) cudaFreeHost(ds.pinned);
    ds.pinned = nullptr;
    ds.pinned_bytes = 0;
    const size_t want = std::max(bytes, size_t(1) << 20);
    const cudaError_t e = cudaHostAlloc(&ds.pinned, want, cudaHostAllocDefault);
    if (e != cudaSuccess) return e;
    ds.pinned_bytes = want;
  }
  *out = ds.pinned;
  return cudaSuccess;
}

cudaError_t device_streams(DevStreams** out) {
  static std::mutex init_mu;
  static DevStreams per_dev[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  DevStreams& ds = per_dev[dev];
  std::lock_guard<std::mutex> lock(init_mu);
  if (!ds.ok) {
    e = cudaStreamCreateWithFlags(&ds.copy, cudaStreamNonBlocking);
    for (int w = 0; w < kWorkers && e == cudaSuccess; ++w)
      e = cudaStreamCreateWithFlags(&ds.work[w], cudaStreamNonBlocking);
    for (int i = 0; i < kEvents && e == cudaSuccess; ++i)
      e = cudaEventCreateWithFlags(&ds.ev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    ds.ok = true;
  }
  *out = &ds;
  return cudaSuccess;
}

}  // namespace

namespace {

int fail_to(cudaError_t e, const std::string& extra, std::string* err) {
  const int rc = cuda_fail(e, extra);
  *err = pcs_last_error();
  return rc;
}

// The host-batch pipeline on the calling thread's current device (arguments
// already validated). Thread-safe: callers on one device serialise on its
// stream set. Errors go to *err (the caller may be a worker thread).
int host_batch_device(const pcs_gpu_args* ha, int32_t sort_axis, int32_t* out_perm,
                      int32_t chunks, std::string* err) {
  std::string msg;
  const int64_t B = ha->batch, N = ha->n, C = ha->c;
  if (B == 0) return PCS_OK;
  const size_t csize = ha->coord_dtype == PCS_DTYPE_F64 ? 8 : 4;
  const size_t isize = ha->index_dtype == PCS_INDEX_I64 ? 8 : 4;
  const size_t cloud_bytes = csize * 3 * static_cast<size_t>(N);
  // Chunk boundaries: `chunks` equal chunks (<= 0: by input size). (Splitting the last
  // chunk s/2, s/4, s/4 so its sectors take the lower-latency W-warp NPDU
  // kernel measured slower: cfg4 e2e 1.14 -> 1.22 ms, the small chunks'
  // kernels overlap on the worker streams.)
  std::vector<int64_t> bounds{0};
  {
    // default: one chunk per ~1.5 MiB of input, at most 8 (small batches
    // are dominated by per-chunk API and launch overhead, not by the copy;
    // r02 sweep, tools/e2e_parts.py: cfg3 (6.3 MB) 0.288 ms in one chunk vs
    // 0.255 in four, cfg4 (50 MB) best at 8)
    const int64_t by_size = static_cast<int64_t>((cloud_bytes * B) / (size_t(3) << 19));
    int64_t def = std::max<int64_t>(1, std::min<int64_t>(8, by_size));
    // inputs beyond ~50 MB keep chunks of ~6 MiB, up to 16 (r02 s4,
    // tools/e2e_parts.py: 256 x 32K (100 MB) NPDU 2.43 ms in 8 chunks vs 2.34
    // in 12-16, AFPS M=256 2.29 vs 2.17; cfg4 (50 MB) stays best at 8)
    if (def == 8)
      def = std::max<int64_t>(8, std::min<int64_t>(16, static_cast<int64_t>((cloud_bytes * B) / (size_t(6) << 20))));
    // Compute-heavy calls with few sectors (many reference distance
    // evaluations per input point, about one wave of sectors: full-window
    // FPS / AFPS M=1) are bound by their kernels' serial iteration chains,
    // not by the copy: chunks then only split the batch into launches that
    // wait on one another (r02,
    // tools/e2e_parts.py: 256 x 4K FPS 1.86 ms in 4 chunks vs 1.35 in 2,
    // 256 x 8K 3.64 vs 2.67, 256 x 2K 0.77 vs 0.56 in 1).
    {
      const bool windowed = ha->method == PCS_METHOD_NPDU_FPS || ha->method == PCS_METHOD_NPDU_AFPS;
      const bool sectored = ha->method == PCS_METHOD_AFPS || ha->method == PCS_METHOD_NPDU_AFPS;
      const int64_t sector = (N + (sectored ? ha->m : 1) - 1) / (sectored ? ha->m : 1);
      const int64_t per_iter = windowed ? std::min<int64_t>(ha->k, sector) : sector;
      const double evals_per_point = static_cast<double>(per_iter) * static_cast<double>(C) /
                                     static_cast<double>(N > 0 ? N : 1);
      const int64_t sectors = B * (sectored ? ha->m : 1);
      if (evals_per_point > 256 && sectors <= 2 * 148)
        def = std::min<int64_t>(def, sector > 2048 ? 2 : 1);
    }
    const int64_t nu = std::min<int64_t>(std::min<int64_t>(B, chunks > 0 ? chunks : def), kEvents - 4);
    for (int64_t i = 1; i <= nu; ++i) bounds.push_back(B * i / nu);
  }
  int nch = static_cast<int>(bounds.size()) - 1;
  DevStreams* dsp = nullptr;
  cudaError_t e = device_streams(&dsp);
  if (e != cudaSuccess) return fail_to(e, "", err);
  std::lock_guard<std::mutex> lock(dsp->mu);
  DevStreams& ds = *dsp;
  cudaStream_t copy = ds.copy;
  cudaStream_t* work = ds.work;
  void* ws = nullptr;
  size_t off_xyz = 0, off_perm = 0, off_idx = 0, off_sec = 0, off_st = 0, off_seed = 0;
  if (e == cudaSuccess) {
    size_t bytes = 0;
    auto take = [&](size_t& off, size_t len) { off = bytes; bytes += (len + 255) & ~size_t(255); };
    take(off_xyz, cloud_bytes * B);
    take(off_perm, sort_axis >= 0 ? 4 * static_cast<size_t>(N) * B : 0);
    take(off_idx, isize * static_cast<size_t>(C) * B);
    take(off_sec, ha->out_sector ? 4 * static_cast<size_t>(C) * B : 0);
    take(off_st, ha->out_stats ? 32 * static_cast<size_t>(B) : 0);
    take(off_seed, ha->seeds ? 8 * static_cast<size_t>(B) : 0);
    e = workspace_alloc(&ws, bytes, copy);
  }
  char* base = static_cast<char*>(ws);
  if (e == cudaSuccess && ha->seeds)
    e = cudaMemcpyAsync(base + off_seed, ha->seeds, 8 * B, cudaMemcpyHostToDevice, copy);
  const bool single = nch == 1;
  cudaEvent_t seeds_ready = ds.ev[kEvents - 1];  // the workspace (and seeds) exist
  if (e == cudaSuccess && !single) e = cudaEventRecord(seeds_ready, copy);
  for (int i = 0; i < nch && e == cudaSuccess; ++i) {
    const int64_t b0 = bounds[i], b1 = bounds[i + 1], nb = b1 - b0;
    if (nb == 0) continue;
    // one chunk: everything in order on the copy stream (no events, one
    // synchronize); several: the chunk's work stream waits for its copy
    cudaStream_t w = single ? copy : work[i % kWorkers];
    char* dx = base + off_xyz + cloud_bytes * b0;
    e = cudaMemcpyAsync(dx, static_cast<const char*>(ha->xyz) + cloud_bytes * b0,
                        cloud_bytes * nb, cudaMemcpyHostToDevice, copy);
    if (!single) {
      cudaEvent_t ready = ds.ev[i];
      if (e == cudaSuccess) e = cudaEventRecord(ready, copy);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(w, ready, 0);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(w, seeds_ready, 0);
    }
    int32_t* dperm = reinterpret_cast<int32_t*>(base + off_perm) + N * b0;
    // the sort writes only the permutation; the sampler gathers through it
    if (e == cudaSuccess && sort_axis >= 0)
      e = launch_sort(ha->coord_dtype, dx, nb, N, sort_axis, nullptr, dperm, w);
    pcs_gpu_args a = *ha;
    a.xyz = dx;
    a.perm = sort_axis >= 0 ? dperm : nullptr;
    a.batch = nb;
    a.seeds = ha->seeds ? reinterpret_cast<const uint64_t*>(base + off_seed) + b0 : nullptr;
    a.out_indices = base + off_idx + isize * C * b0;
    a.out_sector = ha->out_sector ? reinterpret_cast<int32_t*>(base + off_sec) + C * b0 : nullptr;
    a.out_stats = ha->out_stats ? reinterpret_cast<uint64_t*>(base + off_st) + 4 * b0 : nullptr;
    if (e == cudaSuccess) {
      e = launch_sample(a, w, &msg);
      if (e != cudaSuccess) break;
    }
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(static_cast<char*>(ha->out_indices) + isize * C * b0, a.out_indices,
                          isize * C * nb, cudaMemcpyDeviceToHost, w);
    if (e == cudaSuccess && ha->out_sector)
      e = cudaMemcpyAsync(ha->out_sector + C * b0, a.out_sector, 4 * C * nb, cudaMemcpyDeviceToHost, w);
    if (e == cudaSuccess && ha->out_stats)
      e = cudaMemcpyAsync(ha->out_stats + 4 * b0, a.out_stats, 32 * nb, cudaMemcpyDeviceToHost, w);
    if (e == cudaSuccess && sort_axis >= 0 && out_perm)
      e = cudaMemcpyAsync(out_perm + N * b0, dperm, 4 * N * nb, cudaMemcpyDeviceToHost, w);
  }
  for (int w = 0; w < kWorkers && !single; ++w) {
    const cudaError_t e2 = cudaStreamSynchronize(work[w]);
    if (e == cudaSuccess) e = e2;
  }
  if (ws) cudaFreeAsync(ws, copy);  // every use above has completed (or precedes it on `copy`)
  {
    const cudaError_t e2 = cudaStreamSynchronize(copy);
    if (e == cudaSuccess) e = e2;
  }
  if (e != cudaSuccess) return fail_to(e, msg, err);
  return PCS_OK;
}


// One storage slice (a run of sectors) of a single cloud on the current
// device: the whole cloud goes over and is sorted there (every device sorts
// it itself -- the sort is cheap next to a cross-device broadcast), then the
// slice [point_lo, point_hi) is sampled with the global index / sector
// bases; its indices land in out slots [out_lo, out_lo + c) of the row.
int host_sector_slice(const pcs_gpu_args* ha, int32_t sort_axis, int32_t* out_perm,
                      int64_t point_lo, int64_t point_hi, int64_t sector_lo, int64_t m,
                      int64_t out_lo, int64_t c, uint64_t* stats, std::string* err) {
  std::string msg;
  const int64_t N = ha->n;
  const size_t csize = ha->coord_dtype == PCS_DTYPE_F64 ? 8 : 4;
  const size_t isize = ha->index_dtype == PCS_INDEX_I64 ? 8 : 4;
  const size_t cloud_bytes = csize * 3 * static_cast<size_t>(N);
  DevStreams* dsp = nullptr;
  cudaError_t e = device_streams(&dsp);
  if (e != cudaSuccess) return fail_to(e, "", err);
  std::lock_guard<std::mutex> lock(dsp->mu);
  cudaStream_t st = dsp->work[0];
  size_t bytes = 0, off_perm = 0, off_idx = 0, off_sec = 0, off_st = 0, off_seed = 0;
  auto take = [&](size_t& off, size_t len) { off = bytes; bytes += (len + 255) & ~size_t(255); };
  size_t off_xyz = 0;
  take(off_xyz, cloud_bytes);
  take(off_perm, sort_axis >= 0 ? 4 * static_cast<size_t>(N) : 0);
  take(off_idx, isize * static_cast<size_t>(c));
  take(off_sec, 4 * static_cast<size_t>(c));
  take(off_st, 32);
  take(off_seed, 8);
  void* ws = nullptr;
  e = workspace_alloc(&ws, bytes, st);
  if (e != cudaSuccess) return fail_to(e, "", err);
  char* base = static_cast<char*>(ws);
  e = cudaMemcpyAsync(base + off_xyz, ha->xyz, cloud_bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && ha->seeds)
    e = cudaMemcpyAsync(base + off_seed, ha->seeds, 8, cudaMemcpyHostToDevice, st);
  int32_t* dperm = reinterpret_cast<int32_t*>(base + off_perm);
  if (e == cudaSuccess && sort_axis >= 0)
    e = launch_sort(ha->coord_dtype, base + off_xyz, 1, N, sort_axis, nullptr, dperm, st);
  pcs_gpu_args a = *ha;
  // the slice of the sorted order: through the permutation (storage
  // indices of the whole cloud), or the storage slice when not sorting
  a.xyz = base + off_xyz + (sort_axis >= 0 ? 0 : csize * 3 * static_cast<size_t>(point_lo));
  a.perm = sort_axis >= 0 ? dperm + point_lo : nullptr;
  a.batch = 1;
  a.n = point_hi - point_lo;
  a.m = m;
  a.c = c;
  a.index_base = ha->index_base + point_lo;
  a.sector_base = ha->sector_base + sector_lo;
  a.seeds = ha->seeds ? reinterpret_cast<const uint64_t*>(base + off_seed) : nullptr;
  a.out_indices = base + off_idx;
  a.out_sector = reinterpret_cast<int32_t*>(base + off_sec);
  a.out_stats = reinterpret_cast<uint64_t*>(base + off_st);
  if (e == cudaSuccess) e = launch_sample(a, st, &msg);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(static_cast<char*>(ha->out_indices) + isize * out_lo, a.out_indices,
                        isize * c, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && ha->out_sector)
    e = cudaMemcpyAsync(ha->out_sector + out_lo, a.out_sector, 4 * c, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(stats, a.out_stats, 32, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && sort_axis >= 0 && out_perm)
    e = cudaMemcpyAsync(out_perm, dperm, 4 * N, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(ws, st);
  const cudaError_t e2 = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = e2;
  return e == cudaSuccess ? PCS_OK : fail_to(e, msg, err);
}

int check_host_args(const pcs_gpu_args* ha, int32_t sort_axis, const char* who) {
  if (!ha) { set_error(std::string(who) + ": null args"); return PCS_ERR_INVALID_ARGUMENT; }
  std::string msg;
  const int rc = validate_sample(ha->method, ha->n, ha->c, ha->m, ha->k, &msg);
  if (rc) { set_error(msg); return rc; }
  if (ha->batch < 0) { set_error(std::string(who) + ": batch must be >= 0"); return PCS_ERR_INVALID_ARGUMENT; }
  if (sort_axis < -1 || sort_axis > 2) { set_error("axis must be x, y, or z"); return PCS_ERR_INVALID_ARGUMENT; }
  if (ha->batch > 0 && (!ha->xyz || !ha->out_indices)) { set_error(std::string(who) + ": null buffer"); return PCS_ERR_INVALID_ARGUMENT; }
  if (ha->perm) { set_error(std::string(who) + ": perm is a device-call field; use sort_axis"); return PCS_ERR_INVALID_ARGUMENT; }
  return PCS_OK;
}

// [lo, hi) of part r of `total` split `parts` ways, the first total % parts
// parts one larger (partition_sectors' rule, proj/src/sectors.cpp:9-24)
void split_range(int64_t total, int64_t parts, int64_t r, int64_t* lo, int64_t* hi) {
  const int64_t base = total / parts, rem = total % parts;
  *lo = r * base + std::min(r, rem);
  *hi = *lo + base + (r < rem ? 1 : 0);
}

}  // namespace

int pcs_sample_host_batch(const pcs_gpu_args* ha, int32_t sort_axis, int32_t* out_perm,
                          int32_t chunks) {
  clear_error();
  int rc = check_host_args(ha, sort_axis, "pcs_sample_host_batch");
  if (rc) return rc;
  std::string err;
  rc = host_batch_device(ha, sort_axis, out_perm, chunks, &err);
  if (rc) set_error(err);
  return rc;
}

int pcs_sample_host_multi(const pcs_gpu_args* ha, int32_t sort_axis, int32_t* out_perm,
                          const int32_t* devices, int32_t ndevices) {
  clear_error();
  int rc = check_host_args(ha, sort_axis, "pcs_sample_host_multi");
  if (rc) return rc;
  if (!devices || ndevices < 1) { set_error("pcs_sample_host_multi: need at least one device"); return PCS_ERR_INVALID_ARGUMENT; }
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess) return cuda_fail(e);
  for (int i = 0; i < ndevices; ++i)
    if (devices[i] < 0 || devices[i] >= count) { set_error("pcs_sample_host_multi: no such device " + std::to_string(devices[i])); return PCS_ERR_INVALID_ARGUMENT; }
  const int64_t B = ha->batch;
  if (B == 0) return PCS_OK;
  const bool sectored = ha->method == PCS_METHOD_AFPS || ha->method == PCS_METHOD_NPDU_AFPS;
  const bool by_sector = B == 1 && sectored && ndevices > 1 && ha->m >= ndevices;
  const int64_t parts = by_sector ? ndevices : std::min<int64_t>(ndevices, B);
  std::vector<int> rcs(parts, PCS_OK);
  std::vector<std::string> errs(parts);
  std::vector<uint64_t> stats(4 * parts, 0);
  const size_t csize = ha->coord_dtype == PCS_DTYPE_F64 ? 8 : 4;
  const size_t isize = ha->index_dtype == PCS_INDEX_I64 ? 8 : 4;
  auto work = [&](int64_t r) {
    cudaError_t ce = cudaSetDevice(devices[r]);
    if (ce != cudaSuccess) { rcs[r] = fail_to(ce, "", &errs[r]); return; }
    if (by_sector) {
      // one cloud: a contiguous run of sectors per device; with the
      // reference's remainder rule a run re-partitions to the same
      // boundaries and quotas (sectors.cpp:9-36)
      int64_t s0, s1, p0, p1, o0, o1, t;
      split_range(ha->m, parts, r, &s0, &s1);
      split_range(ha->n, ha->m, s0, &p0, &t);
      split_range(ha->n, ha->m, s1, &p1, &t);
      split_range(ha->c, ha->m, s0, &o0, &t);
      split_range(ha->c, ha->m, s1, &o1, &t);
      if (s1 == ha->m) { p1 = ha->n; o1 = ha->c; }
      rcs[r] = host_sector_slice(ha, sort_axis, r == 0 ? out_perm : nullptr, p0, p1, s0,
                                 s1 - s0, o0, o1 - o0, &stats[4 * r], &errs[r]);
      return;
    }
    int64_t b0, b1;
    split_range(B, parts, r, &b0, &b1);
    pcs_gpu_args a = *ha;
    a.batch = b1 - b0;
    a.xyz = static_cast<const char*>(ha->xyz) + csize * 3 * static_cast<size_t>(ha->n) * b0;
    a.seeds = ha->seeds ? ha->seeds + b0 : nullptr;
    a.out_indices = static_cast<char*>(ha->out_indices) + isize * static_cast<size_t>(ha->c) * b0;
    a.out_sector = ha->out_sector ? ha->out_sector + ha->c * b0 : nullptr;
    a.out_stats = ha->out_stats ? ha->out_stats + 4 * b0 : nullptr;
    rcs[r] = host_batch_device(&a, sort_axis, out_perm ? out_perm + ha->n * b0 : nullptr, 0,
                               &errs[r]);
  };
  int prev = 0;
  e = cudaGetDevice(&prev);
  if (e != cudaSuccess) return cuda_fail(e);
  {
    std::vector<std::thread> pool;
    for (int64_t r = 1; r < parts; ++r) pool.emplace_back(work, r);
    work(0);
    for (auto& th : pool) th.join();
  }
  cudaSetDevice(prev);
  for (int64_t r = 0; r < parts; ++r)
    if (rcs[r] != PCS_OK) {
      set_error(errs[r]);
      return rcs[r];
    }
  if (by_sector && ha->out_stats)
    for (int j = 0; j < 4; ++j) {
      uint64_t sum = 0;
      for (int64_t r = 0; r < parts; ++r) sum += stats[4 * r + j];
      ha->out_stats[j] = sum;
    }
  return PCS_OK;
}

int pcs_sample_host(int32_t method, const double* xyz, int64_t n, int64_t c, int64_t m,
                    int64_t k, int32_t seed_policy, uint64_t seed, uint32_t threads,
                    int64_t* out_indices, int64_t* out_sector, uint64_t* out_stats) {
  (void)threads;  // accepted for pcs::afps(..., threads) parity; GPU schedule is fixed
  clear_error();
  std::string msg;
  int rc = validate_sample(method, n, c, m, k, &msg);
  if (rc) { set_error(msg); return rc; }
  DevStreams* dsp = nullptr;
  cudaError_t e = device_streams(&dsp);
  if (e != cudaSuccess) return cuda_fail(e);
  std::lock_guard<std::mutex> lock(dsp->mu);
  cudaStream_t st = dsp->copy;
  // Full-window samplers on coordinates that are all exactly representable
  // in fp32 (the usual case: clouds read from f32_bin files or float32
  // arrays, forcecast to float64 by the binding) run from an fp32 copy: the
  // kernels widen fp32 exactly, so every distance and every result is the
  // same, the copy is halved and large sectors get the tensor-memory Morton
  // engine. (Windowed samplers keep fp64 staging: one cloud's NPDU sectors
  // are latency-bound and fp64 coordinates need no per-iteration widening.)
  const bool windowed = method == PCS_METHOD_NPDU_FPS || method == PCS_METHOD_NPDU_AFPS;
  bool use32 = !windowed;
  for (int64_t i = 0; i < 3 * n && use32; ++i) {
    const float f = static_cast<float>(xyz[i]);
    use32 = static_cast<double>(f) == xyz[i];  // NaN: not exact
  }
  use32 = use32 || n == 0;
  const size_t coord_bytes = (use32 ? sizeof(float) : sizeof(double)) * 3 * n;
  // the cloud (fp32 copy or the doubles) staged in pinned memory
  void* stage = nullptr;
  e = pinned_scratch(*dsp, coord_bytes, &stage);
  if (e != cudaSuccess) return cuda_fail(e);
  if (use32) {
    float* f32 = static_cast<float*>(stage);
    for (int64_t i = 0; i < 3 * n; ++i) f32[i] = static_cast<float>(xyz[i]);
  } else {
    std::memcpy(stage, xyz, coord_bytes);
  }
  // one workspace: cloud, indices, sector ids (int32 on the device), stats
  const size_t b_xyz = (coord_bytes + 255) & ~size_t(255);
  const size_t b_idx = (sizeof(int64_t) * c + 255) & ~size_t(255);
  const size_t b_sec = (sizeof(int32_t) * c + 255) & ~size_t(255);
  void* ws = nullptr;
  e = workspace_alloc(&ws, b_xyz + b_idx + b_sec + 32, st);
  if (e != cudaSuccess) return cuda_fail(e);
  char* base = static_cast<char*>(ws);
  int32_t* dsec = reinterpret_cast<int32_t*>(base + b_xyz + b_idx);
  uint64_t* dstat = reinterpret_cast<uint64_t*>(base + b_xyz + b_idx + b_sec);
  std::vector<int32_t> sec32(out_sector ? static_cast<size_t>(c) : 0);
  e = cudaMemcpyAsync(base, stage, coord_bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    pcs_gpu_args a{};
    a.method = method;
    a.coord_dtype = use32 ? PCS_DTYPE_F32 : PCS_DTYPE_F64;
    a.xyz = base;
    a.batch = 1;
    a.n = n;
    a.c = c;
    a.m = m;
    a.k = k;
    a.seed_policy = seed_policy;
    a.seed = seed;
    a.index_dtype = PCS_INDEX_I64;
    a.out_indices = base + b_xyz;
    a.out_sector = out_sector ? dsec : nullptr;
    a.out_stats = dstat;
    e = launch_sample(a, st, &msg);
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out_indices, base + b_xyz, sizeof(int64_t) * c, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && out_sector)
    e = cudaMemcpyAsync(sec32.data(), dsec, sizeof(int32_t) * c, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && out_stats)
    e = cudaMemcpyAsync(out_stats, dstat, sizeof(uint64_t) * 4, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(ws, st);
  const cudaError_t e2 = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return cuda_fail(e, msg);
  for (int64_t i = 0; out_sector && i < c; ++i) out_sector[i] = sec32[i];
  return PCS_OK;
}

int pcs_local_fps_host(const double* xyz, int64_t n, int64_t sb, int64_t se, int64_t quota,
                       int64_t k, int32_t seed_policy, uint64_t seed, int64_t* out_indices,
                       uint64_t* out_stats, double* trace) {
  clear_error();
  // proj/src/sampler.cpp:89-94, same order and messages.
  if (se > n || sb < 0 || sb >= se) { set_error("local_fps: sector out of range"); return PCS_ERR_INVALID_ARGUMENT; }
  if (quota < 1 || quota > se - sb) { set_error("local_fps: quota infeasible for sector"); return PCS_ERR_INVALID_ARGUMENT; }
  if (k == 0) { set_error("local_fps: window size must be >= 1"); return PCS_ERR_INVALID_ARGUMENT; }
  if (n > 0x7fffffffLL) { set_error("clouds above 2^31-1 points are not supported"); return PCS_ERR_UNSUPPORTED; }
  // k < 0 encodes std::nullopt (full window).
  DevStreams* dsp = nullptr;
  cudaError_t e = device_streams(&dsp);
  if (e != cudaSuccess) return cuda_fail(e);
  std::lock_guard<std::mutex> lock(dsp->mu);
  cudaStream_t st = dsp->copy;
  int rc = PCS_OK;
  const int64_t len = se - sb;
  {
    DevBuf dx(st), didx(st), dstat(st), dtr(st);
    const size_t trace_n = trace ? static_cast<size_t>(quota > 1 ? quota - 1 : 0) * len : 0;
    std::string msg;
    if ((e = dx.alloc(sizeof(double) * 3 * n)) != cudaSuccess ||
        (e = didx.alloc(sizeof(int64_t) * quota)) != cudaSuccess ||
        (e = dstat.alloc(sizeof(uint64_t) * 4)) != cudaSuccess ||
        (trace && (e = dtr.alloc(sizeof(double) * trace_n)) != cudaSuccess) ||
        (e = cudaMemcpyAsync(dx.p, xyz, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = launch_local_fps(static_cast<double*>(dx.p), n, sb, se, quota, k < 0 ? 0 : k,
                              seed_policy == PCS_RANDOM_FIRST_POINT, seed,
                              static_cast<int64_t*>(didx.p), static_cast<uint64_t*>(dstat.p),
                              trace ? static_cast<double*>(dtr.p) : nullptr, st, &msg)) != cudaSuccess ||
        (e = cudaMemcpyAsync(out_indices, didx.p, sizeof(int64_t) * quota, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(out_stats, dstat.p, sizeof(uint64_t) * 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (trace && trace_n && (e = cudaMemcpyAsync(trace, dtr.p, sizeof(double) * trace_n, cudaMemcpyDeviceToHost, st)) != cudaSuccess) ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
      rc = cuda_fail(e, msg);
  }
  cudaStreamSynchronize(st);
  return rc;
}

int pcs_exact_sort_host(const double* xyz, int64_t n, int32_t axis, double* out_xyz,
                        int64_t* out_perm) {
  clear_error();
  if (axis < 0 || axis > 2) { set_error("axis must be x, y, or z"); return PCS_ERR_INVALID_ARGUMENT; }
  if (n <= 0) return PCS_OK;
  // int32 permutation and 32-bit sort indices on every path
  if (n > 0x7fffffffLL) { set_error("clouds above 2^31-1 points are not supported"); return PCS_ERR_UNSUPPORTED; }
  DevStreams* dsp = nullptr;
  cudaError_t e = device_streams(&dsp);
  if (e != cudaSuccess) return cuda_fail(e);
  std::lock_guard<std::mutex> lock(dsp->mu);
  cudaStream_t st = dsp->copy;
  int rc = PCS_OK;
  // The order depends on the axis column alone. When every axis value is
  // exactly representable in fp32 (clouds read from f32_bin files or float32
  // arrays, forcecast to float64 by the binding), sort fp32 keys: the same
  // operator< order (fp32 widens exactly; -0.0 folds onto +0.0 either way),
  // a third of the copy, the on-chip fp32 sort kernels; only the permutation
  // comes back and the host gathers the float64 points through it.
  bool f32_keys = true;
  for (int64_t i = 0; i < n && f32_keys; ++i) {
    const double v = xyz[3 * i + axis];
    f32_keys = static_cast<double>(static_cast<float>(v)) == v;  // NaN: not exact
  }
  if (f32_keys) {
    DevBuf dk(st), dperm(st);
    // pinned staging: the keys in column 0 of an (n, 3) fp32 array (the
    // sort kernels' layout, sorted on axis 0), then the permutation
    void* stage = nullptr;
    if ((e = pinned_scratch(*dsp, sizeof(float) * 4 * n, &stage)) != cudaSuccess) return cuda_fail(e);
    float* keys = static_cast<float*>(stage);
    int32_t* perm32 = reinterpret_cast<int32_t*>(keys + 3 * n);
    for (int64_t i = 0; i < n; ++i) keys[3 * i] = static_cast<float>(xyz[3 * i + axis]);
    if ((e = dk.alloc(sizeof(float) * 3 * n)) != cudaSuccess ||
        (e = dperm.alloc(sizeof(int32_t) * n)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dk.p, keys, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = launch_sort(PCS_DTYPE_F32, dk.p, 1, n, 0, nullptr, static_cast<int32_t*>(dperm.p), st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(perm32, dperm.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess) {
      rc = cuda_fail(e);
    } else {
      for (int64_t i = 0; i < n; ++i) {
        const int64_t from = perm32[i];
        if (out_perm) out_perm[i] = from;
        if (out_xyz) {
          out_xyz[3 * i] = xyz[3 * from];
          out_xyz[3 * i + 1] = xyz[3 * from + 1];
          out_xyz[3 * i + 2] = xyz[3 * from + 2];
        }
      }
    }
    cudaStreamSynchronize(st);
    return rc;
  }
  {
    DevBuf dx(st), dout(st), dperm(st);
    int32_t* perm32 = new int32_t[n];
    if ((e = dx.alloc(sizeof(double) * 3 * n)) != cudaSuccess ||
        (e = dout.alloc(sizeof(double) * 3 * n)) != cudaSuccess ||
        (e = dperm.alloc(sizeof(int32_t) * n)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dx.p, xyz, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = launch_sort(PCS_DTYPE_F64, dx.p, 1, n, axis, dout.p, static_cast<int32_t*>(dperm.p), st)) != cudaSuccess ||
        (out_xyz && (e = cudaMemcpyAsync(out_xyz, dout.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, st)) != cudaSuccess) ||
        (e = cudaMemcpyAsync(perm32, dperm.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess) {
      rc = cuda_fail(e);
    } else if (out_perm) {
      for (int64_t i = 0; i < n; ++i) out_perm[i] = perm32[i];
    }
    delete[] perm32;
  }
  cudaStreamSynchronize(st);
  return rc;
}

int pcs_gpu_coverage_radius(int32_t coord_dtype, const void* xyz, int64_t batch, int64_t n,
                            int32_t index_dtype, const void* samples, int64_t c, double* out,
                            void* stream) {
  clear_error();
  if (c < 1) { set_error("coverage_radius: sample set is empty"); return PCS_ERR_INVALID_ARGUMENT; }
  const cudaError_t e = launch_metric(0, coord_dtype, xyz, batch, n, index_dtype, samples, c, out,
                                      static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? PCS_OK : cuda_fail(e);
}

int pcs_gpu_separation(int32_t coord_dtype, const void* xyz, int64_t batch, int64_t n,
                       int32_t index_dtype, const void* samples, int64_t c, double* out,
                       void* stream) {
  clear_error();
  if (c < 2) { set_error("separation: need at least 2 samples"); return PCS_ERR_INVALID_ARGUMENT; }
  const cudaError_t e = launch_metric(1, coord_dtype, xyz, batch, n, index_dtype, samples, c, out,
                                      static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? PCS_OK : cuda_fail(e);
}

static int metric_host(int which, const double* xyz, int64_t n, const int64_t* samples, int64_t c,
                       double* out) {
  clear_error();
  const char* who = which == 0 ? "coverage_radius" : "separation";
  // proj/src/metrics.cpp:18-21, 37-40: same checks, same order
  if (which == 0 && c < 1) { set_error("coverage_radius: sample set is empty"); return PCS_ERR_INVALID_ARGUMENT; }
  if (which == 1 && c < 2) { set_error("separation: need at least 2 samples"); return PCS_ERR_INVALID_ARGUMENT; }
  for (int64_t i = 0; i < c; ++i)
    if (samples[i] < 0 || samples[i] >= n) {
      set_error(std::string(who) + ": index out of range");
      return PCS_ERR_INVALID_ARGUMENT;
    }
  DevStreams* dsp = nullptr;
  cudaError_t e = device_streams(&dsp);
  if (e != cudaSuccess) return cuda_fail(e);
  std::lock_guard<std::mutex> lock(dsp->mu);
  cudaStream_t st = dsp->copy;
  int rc = PCS_OK;
  {
    DevBuf dx(st), di(st), dout(st);
    if ((e = dx.alloc(sizeof(double) * 3 * n)) != cudaSuccess ||
        (e = di.alloc(sizeof(int64_t) * c)) != cudaSuccess ||
        (e = dout.alloc(sizeof(double))) != cudaSuccess ||
        (e = cudaMemcpyAsync(dx.p, xyz, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(di.p, samples, sizeof(int64_t) * c, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = launch_metric(which, PCS_DTYPE_F64, dx.p, 1, n, PCS_INDEX_I64, di.p, c,
                           static_cast<double*>(dout.p), st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(out, dout.p, sizeof(double), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
      rc = cuda_fail(e);
  }
  cudaStreamSynchronize(st);
  return rc;
}

int pcs_coverage_radius_host(const double* xyz, int64_t n, const int64_t* samples, int64_t c,
                             double* out) {
  return metric_host(0, xyz, n, samples, c, out);
}

int pcs_separation_host(const double* xyz, int64_t n, const int64_t* samples, int64_t c,
                        double* out) {
  return metric_host(1, xyz, n, samples, c, out);
}

}  // extern "C"
