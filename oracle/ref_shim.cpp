// REFERENCE SHIM -- TEST INFRASTRUCTURE ONLY.
//
// A C-callable face over the UNMODIFIED reference library, compiled from the
// sources where they lie under /root/reference/proj/src by oracle/Makefile
// into oracle/_ref/libpcsref.so (git-ignored, shipped to the GPU box with the
// snapshot). Used to (1) validate the C restatement in pcs_oracle.c, (2)
// generate tests/golden/ fixtures, and (3) serve as the bench's
// `--impl reference` arm and cpu_baseline (kind "reference"). Never linked
// into the product.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "pcs/bench.hpp"
#include "pcs/io.hpp"
#include "pcs/metrics.hpp"
#include "pcs/order.hpp"
#include "pcs/sampler.hpp"

namespace {

void put_err(char* err, std::size_t errlen, const char* msg) {
  if (err && errlen) {
    std::strncpy(err, msg, errlen - 1);
    err[errlen - 1] = 0;
  }
}

pcs::PointCloud cloud_f64(const double* xyz, std::uint64_t n) {
  pcs::PointCloud cloud;
  cloud.points.resize(n);
  for (std::uint64_t i = 0; i < n; ++i)
    cloud.points[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  return cloud;
}

pcs::SampleResult dispatch(int method, const pcs::PointCloud& cloud, std::uint64_t c,
                           std::uint64_t m, std::uint64_t k, int random_first,
                           std::uint64_t seed, unsigned threads) {
  const auto policy = random_first ? pcs::SeedPolicy::RandomFirstPoint
                                   : pcs::SeedPolicy::FixedFirstPoint;
  switch (method) {
    case 1: return pcs::fps(cloud, c, policy, seed);
    case 2: return pcs::afps(cloud, c, m, policy, seed, threads);
    case 3: return pcs::npdu_fps(cloud, c, k, policy, seed);
    case 4: return pcs::npdu_afps(cloud, c, m, k, policy, seed, threads);
  }
  throw std::invalid_argument("run_sampler: unknown method");
}

}  // namespace

extern "C" {

// method: 1 fps, 2 afps, 3 npdu_fps, 4 npdu_afps. Returns 0, or 1 with the
// reference's std::invalid_argument message in err.
int ref_sample(int method, const double* xyz, std::uint64_t n, std::uint64_t c,
               std::uint64_t m, std::uint64_t k, int random_first, std::uint64_t seed,
               unsigned threads, std::int64_t* out_idx, std::int64_t* out_sector,
               std::uint64_t* stats, char* err, std::size_t errlen) {
  try {
    const auto r = dispatch(method, cloud_f64(xyz, n), c, m, k, random_first, seed, threads);
    for (std::size_t i = 0; i < r.indices.size(); ++i) {
      out_idx[i] = static_cast<std::int64_t>(r.indices[i]);
      out_sector[i] = static_cast<std::int64_t>(r.sector_of[i]);
    }
    stats[0] = r.stats.dist_evals;
    stats[1] = r.stats.dist_writes;
    stats[2] = r.stats.argmax_scans;
    stats[3] = r.stats.iterations;
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

// detail::local_fps with a DistanceTrace (proj/include/pcs/sampler.hpp:16-37).
int ref_local_fps_trace(const double* xyz, std::uint64_t n, std::uint64_t sb,
                        std::uint64_t se, std::uint64_t quota, int windowed,
                        std::uint64_t k, int random_first, std::uint64_t seed,
                        std::int64_t* out_idx, std::uint64_t* stats, double* trace,
                        char* err, std::size_t errlen) {
  try {
    pcs::DistanceTrace tr;
    const auto policy = random_first ? pcs::SeedPolicy::RandomFirstPoint
                                     : pcs::SeedPolicy::FixedFirstPoint;
    std::optional<std::size_t> wk;
    if (windowed) wk = k;
    const auto r = pcs::detail::local_fps(cloud_f64(xyz, n), {sb, se}, quota, wk,
                                          policy, seed, trace ? &tr : nullptr);
    for (std::size_t i = 0; i < r.indices.size(); ++i)
      out_idx[i] = static_cast<std::int64_t>(r.indices[i]);
    stats[0] = r.stats.dist_evals;
    stats[1] = r.stats.dist_writes;
    stats[2] = r.stats.argmax_scans;
    stats[3] = r.stats.iterations;
    if (trace)
      for (std::size_t p = 0; p < tr.snapshots.size(); ++p)
        std::memcpy(trace + p * (se - sb), tr.snapshots[p].data(),
                    (se - sb) * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

// exact_sort (proj/src/order.cpp:11-24); perm recovered by matching is not
// needed: the gathered cloud is returned and the tests compare coordinates.
int ref_exact_sort(const double* xyz, std::uint64_t n, int axis, double* out) {
  const auto sorted = pcs::exact_sort(cloud_f64(xyz, n), static_cast<pcs::Axis>(axis));
  for (std::uint64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) out[3 * i + a] = sorted.points[i][a];
  return 0;
}

// Batched fp32 clouds (the f32_bin layout, widened exactly to double as
// proj/src/io.cpp:84-86 does), one cloud per worker thread with the sampler
// at threads=1, mirroring the reference bench harness (proj/src/bench.cpp:
// 90-92,104-120). Returns the number of clouds processed; *seconds is the
// wall time of the worker phase.
int ref_sample_batch_f32(int method, const float* xyz, std::uint64_t batch,
                         std::uint64_t n, std::uint64_t c, std::uint64_t m,
                         std::uint64_t k, int random_first, std::uint64_t seed,
                         unsigned workers, std::int64_t* out_idx, std::uint64_t* stats,
                         double* seconds, char* err, std::size_t errlen) {
  std::vector<pcs::PointCloud> clouds(batch);
  for (std::uint64_t b = 0; b < batch; ++b) {
    clouds[b].points.resize(n);
    const float* src = xyz + b * 3 * n;
    for (std::uint64_t i = 0; i < n; ++i)
      clouds[b].points[i] = {static_cast<double>(src[3 * i]),
                             static_cast<double>(src[3 * i + 1]),
                             static_cast<double>(src[3 * i + 2])};
  }
  std::atomic<std::uint64_t> next{0};
  std::atomic<int> failed{0};
  std::string first_err;
  std::mutex mu;
  auto work = [&] {
    for (;;) {
      const std::uint64_t b = next.fetch_add(1);
      if (b >= batch) return;
      try {
        const auto r = dispatch(method, clouds[b], c, m, k, random_first, seed, 1);
        for (std::uint64_t i = 0; i < c; ++i)
          out_idx[b * c + i] = static_cast<std::int64_t>(r.indices[i]);
        stats[4 * b + 0] = r.stats.dist_evals;
        stats[4 * b + 1] = r.stats.dist_writes;
        stats[4 * b + 2] = r.stats.argmax_scans;
        stats[4 * b + 3] = r.stats.iterations;
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> g(mu);
        if (!failed.exchange(1)) first_err = e.what();
      }
    }
  };
  if (workers < 1) workers = 1;
  // timed region: the sampler calls only (proj/src/bench.cpp:89-94), not the
  // fp32 -> PointCloud widening above.
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < workers; ++t) pool.emplace_back(work);
  for (auto& t : pool) t.join();
  if (seconds)
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (failed) {
    put_err(err, errlen, first_err.c_str());
    return -1;
  }
  return static_cast<int>(batch);
}

// coverage_radius / separation (proj/src/metrics.cpp:16-52)
int ref_metric(int which, const double* xyz, std::uint64_t n, const std::int64_t* samples,
               std::uint64_t c, double* out, char* err, std::size_t errlen) {
  try {
    std::vector<std::size_t> idx(samples, samples + c);
    const auto cloud = cloud_f64(xyz, n);
    *out = which == 0 ? pcs::coverage_radius(cloud, idx) : pcs::separation(cloud, idx);
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

// read_cloud (proj/src/io.cpp:93-98): returns N (>= 1) and fills xyz (up
// to cap points), or -1 with the error message.
long long ref_read_cloud(const char* path, int format, double* xyz, std::uint64_t cap, char* err,
                         std::size_t errlen) {
  try {
    const auto cloud = pcs::read_cloud(path, format == 0 ? pcs::CloudFormat::XyzText
                                                         : pcs::CloudFormat::F32Bin);
    for (std::size_t i = 0; i < cloud.size() && i < cap; ++i)
      for (int a = 0; a < 3; ++a) xyz[3 * i + a] = cloud.points[i][a];
    return static_cast<long long>(cloud.size());
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return -1;
  }
}

int ref_write_cloud(const char* path, int format, const double* xyz, std::uint64_t n) {
  pcs::write_cloud(cloud_f64(xyz, n), path,
                   format == 0 ? pcs::CloudFormat::XyzText : pcs::CloudFormat::F32Bin);
  return 0;
}

// run_bench + bench_csv (proj/src/bench.cpp:34-136) over caller-provided
// clouds: cloud i (n_values[i] points) starts at xyz + 3 * offsets[i].
// Methods as pcs::Method ints. Writes the CSV into out (truncated to cap).
long long ref_run_bench_csv(const int* methods, std::uint64_t n_methods, const double* xyz,
                            const std::uint64_t* offsets, const std::uint64_t* n_values,
                            std::uint64_t n_sizes, const std::uint64_t* m_values,
                            std::uint64_t n_m, const std::uint64_t* k_values, std::uint64_t n_k,
                            std::uint64_t c, std::uint64_t g, std::uint64_t trials,
                            std::uint64_t seed, int random_first, unsigned threads, char* out,
                            std::size_t cap) {
  pcs::BenchOptions o;
  for (std::uint64_t i = 0; i < n_methods; ++i) o.methods.push_back(static_cast<pcs::Method>(methods[i]));
  o.n_values.assign(n_values, n_values + n_sizes);
  o.m_values.assign(m_values, m_values + n_m);
  o.k_values.assign(k_values, k_values + n_k);
  o.c = c;
  o.g = g;
  o.trials = trials;
  o.seed = seed;
  o.seed_policy = random_first ? pcs::SeedPolicy::RandomFirstPoint : pcs::SeedPolicy::FixedFirstPoint;
  o.threads = threads;
  auto provider = [&](std::size_t n) {
    for (std::uint64_t i = 0; i < n_sizes; ++i)
      if (n_values[i] == n) return cloud_f64(xyz + 3 * offsets[i], n);
    throw std::invalid_argument("no cloud of that size");
  };
  const auto rows = pcs::run_bench(o, provider);
  const std::string csv = pcs::bench_csv(rows);
  std::strncpy(out, csv.c_str(), cap - 1);
  out[cap - 1] = 0;
  return static_cast<long long>(csv.size());
}

}  // extern "C"
