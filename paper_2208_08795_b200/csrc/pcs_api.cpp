// The reference's C++ operator API (namespace pcs, proj/include/pcs/
// sampler.hpp, sectors.hpp, order.hpp, sampler_spec.hpp, point_cloud.hpp)
// re-implemented on top of the C-ABI (include/pcs_gpu.h). Host integer
// helpers (sector plans, windows, names) are native C++; every distance
// evaluation runs in the sm_100a kernels.
#include <stdexcept>
#include <string>
#include <vector>

#include "pcs/metrics.hpp"
#include "pcs/order.hpp"
#include "pcs/point_cloud.hpp"
#include "pcs/sampler.hpp"
#include "pcs/sampler_spec.hpp"
#include "pcs/sectors.hpp"
#include "pcs_gpu.h"

namespace pcs {
namespace {

[[noreturn]] void raise(int status) {
  const std::string msg = pcs_last_error();
  if (status == PCS_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg.empty() ? pcs_status_string(status) : msg);
}

const double* flat(const PointCloud& cloud) {
  static_assert(sizeof(Point) == 3 * sizeof(double), "Point must be packed xyz");
  return cloud.points.empty() ? nullptr : cloud.points.front().data();
}

SampleResult run(int method, const PointCloud& cloud, std::size_t c, std::size_t m,
                 std::size_t k, SeedPolicy policy, std::uint64_t seed) {
  const auto n = static_cast<int64_t>(cloud.size());
  std::vector<int64_t> idx(c ? c : 1), sec(c ? c : 1);
  uint64_t st[4] = {0, 0, 0, 0};
  const int rc = pcs_sample_host(
      method, flat(cloud), n, static_cast<int64_t>(c), static_cast<int64_t>(m),
      static_cast<int64_t>(k),
      policy == SeedPolicy::RandomFirstPoint ? PCS_RANDOM_FIRST_POINT : PCS_FIXED_FIRST_POINT,
      seed, 1, idx.data(), sec.data(), st);
  if (rc != PCS_OK) raise(rc);
  SampleResult out;
  out.indices.assign(idx.begin(), idx.begin() + static_cast<std::ptrdiff_t>(c));
  out.sector_of.reserve(c);
  for (std::size_t i = 0; i < c; ++i) out.sector_of.push_back(static_cast<std::uint32_t>(sec[i]));
  out.stats = OpStats{st[0], st[1], st[2], st[3]};
  return out;
}

}  // namespace

// ------------------------------------------------------------ point_cloud
const char* axis_name(Axis axis) {
  static const char* names[] = {"x", "y", "z"};
  const int a = static_cast<int>(axis);
  return a >= 0 && a < 3 ? names[a] : "?";
}

std::optional<Axis> parse_axis(std::string_view name) {
  if (name.size() == 1 && name[0] >= 'x' && name[0] <= 'z') return static_cast<Axis>(name[0] - 'x');
  return std::nullopt;
}

std::string to_string(const OrderTag& tag) {
  if (tag.kind == OrderKind::ExactlySorted) return std::string("exactly_sorted(") + axis_name(tag.axis) + ")";
  if (tag.kind == OrderKind::ApproxSorted)
    return std::string("approx_sorted(") + axis_name(tag.axis) + ",b=" + std::to_string(tag.bin_size) + ")";
  return "unsorted";
}

// ------------------------------------------------------------ sampler_spec
const char* method_name(Method method) {
  switch (method) {
    case Method::Rps: return "rps";
    case Method::Fps: return "fps";
    case Method::Afps: return "afps";
    case Method::NpduFps: return "npdu-fps";
    case Method::NpduAfps: return "npdu-afps";
    case Method::GridVoxel: return "grid";
  }
  return "?";
}

std::optional<Method> parse_method(std::string_view name) {
  for (Method m : {Method::Rps, Method::Fps, Method::Afps, Method::NpduFps, Method::NpduAfps,
                   Method::GridVoxel})
    if (name == method_name(m)) return m;
  return std::nullopt;
}

std::string spec_params(const SamplerSpec& spec) {
  switch (spec.method) {
    case Method::Afps: return "m=" + std::to_string(spec.m);
    case Method::NpduFps: return "k=" + std::to_string(spec.k);
    case Method::NpduAfps: return "m=" + std::to_string(spec.m) + ",k=" + std::to_string(spec.k);
    case Method::GridVoxel: return "g=" + std::to_string(spec.g);
    default: return "";
  }
}

// ------------------------------------------------------------ sectors
// proj/src/sectors.cpp:9-61, same messages.
std::vector<IndexRange> partition_sectors(std::size_t n, std::size_t m) {
  if (m < 1) throw std::invalid_argument("partition_sectors: m must be >= 1");
  if (m > n) throw std::invalid_argument("partition_sectors: m exceeds point count");
  std::vector<IndexRange> out(m);
  const std::size_t q = n / m, r = n % m;
  std::size_t at = 0;
  for (std::size_t s = 0; s < m; ++s) {
    const std::size_t len = q + (s < r);
    out[s] = {at, at + len};
    at += len;
  }
  return out;
}

std::vector<std::size_t> allocate_samples(std::size_t c, std::size_t m) {
  if (m < 1) throw std::invalid_argument("allocate_samples: m must be >= 1");
  if (m > c) throw std::invalid_argument("allocate_samples: m exceeds sample count");
  std::vector<std::size_t> out(m);
  for (std::size_t s = 0; s < m; ++s) out[s] = c / m + (s < c % m);
  return out;
}

SectorPlan SectorPlan::make(std::size_t n, std::size_t c, std::size_t m) {
  SectorPlan plan{partition_sectors(n, m), allocate_samples(c, m)};
  for (std::size_t s = 0; s < m; ++s)
    if (plan.quotas[s] > plan.ranges[s].size())
      throw std::invalid_argument("sector " + std::to_string(s) + " holds " +
                                  std::to_string(plan.ranges[s].size()) + " points but owes " +
                                  std::to_string(plan.quotas[s]) + " samples");
  return plan;
}

IndexRange update_window(IndexRange sector, std::size_t sample_idx, std::size_t k) {
  const std::size_t lo = sample_idx >= k / 2 ? sample_idx - k / 2 : 0;
  const std::size_t hi = sample_idx + (k + 1) / 2;
  return {lo > sector.begin ? lo : sector.begin, hi < sector.end ? hi : sector.end};
}

// ------------------------------------------------------------ sampler
namespace detail {

SampleResult local_fps(const PointCloud& cloud, IndexRange sector, std::size_t quota,
                       std::optional<std::size_t> window_k, SeedPolicy seed_policy,
                       std::uint64_t seed, DistanceTrace* trace) {
  const auto n = static_cast<int64_t>(cloud.size());
  // validated again below the boundary; checked here so out-of-range ranges
  // never size the trace buffer
  if (sector.end > cloud.size() || sector.begin >= sector.end)
    throw std::invalid_argument("local_fps: sector out of range");
  if (quota < 1 || quota > sector.size())
    throw std::invalid_argument("local_fps: quota infeasible for sector");
  const std::size_t len = sector.size();
  std::vector<int64_t> idx(quota);
  std::vector<double> tr(trace ? (quota - 1) * len : 0);
  uint64_t st[4] = {0, 0, 0, 0};
  const int rc = pcs_local_fps_host(
      flat(cloud), n, static_cast<int64_t>(sector.begin), static_cast<int64_t>(sector.end),
      static_cast<int64_t>(quota), window_k ? static_cast<int64_t>(*window_k) : -1,
      seed_policy == SeedPolicy::RandomFirstPoint ? PCS_RANDOM_FIRST_POINT : PCS_FIXED_FIRST_POINT,
      seed, idx.data(), st, trace ? tr.data() : nullptr);
  if (rc != PCS_OK) raise(rc);
  SampleResult out;
  out.indices.assign(idx.begin(), idx.end());
  out.sector_of.assign(quota, 0);
  out.stats = OpStats{st[0], st[1], st[2], st[3]};
  if (trace)
    for (std::size_t p = 0; p + 1 < quota; ++p)
      trace->snapshots.emplace_back(tr.begin() + static_cast<std::ptrdiff_t>(p * len),
                                    tr.begin() + static_cast<std::ptrdiff_t>((p + 1) * len));
  return out;
}

}  // namespace detail

SampleResult fps(const PointCloud& cloud, std::size_t c, SeedPolicy seed_policy,
                 std::uint64_t seed) {
  return run(PCS_METHOD_FPS, cloud, c, 1, 0, seed_policy, seed);
}

SampleResult afps(const PointCloud& cloud, std::size_t c, std::size_t m, SeedPolicy seed_policy,
                  std::uint64_t seed, unsigned /*threads*/) {
  return run(PCS_METHOD_AFPS, cloud, c, m, 0, seed_policy, seed);
}

SampleResult npdu_fps(const PointCloud& cloud, std::size_t c, std::size_t k,
                      SeedPolicy seed_policy, std::uint64_t seed) {
  return run(PCS_METHOD_NPDU_FPS, cloud, c, 1, k, seed_policy, seed);
}

SampleResult npdu_afps(const PointCloud& cloud, std::size_t c, std::size_t m, std::size_t k,
                       SeedPolicy seed_policy, std::uint64_t seed, unsigned /*threads*/) {
  return run(PCS_METHOD_NPDU_AFPS, cloud, c, m, k, seed_policy, seed);
}

SampleResult run_sampler(const PointCloud& cloud, const SamplerSpec& spec, unsigned threads) {
  switch (spec.method) {
    case Method::Fps: return fps(cloud, spec.c, spec.seed_policy, spec.seed);
    case Method::Afps: return afps(cloud, spec.c, spec.m, spec.seed_policy, spec.seed, threads);
    case Method::NpduFps: return npdu_fps(cloud, spec.c, spec.k, spec.seed_policy, spec.seed);
    case Method::NpduAfps:
      return npdu_afps(cloud, spec.c, spec.m, spec.k, spec.seed_policy, spec.seed, threads);
    case Method::Rps:
    case Method::GridVoxel:
      throw std::invalid_argument(std::string("run_sampler: ") + method_name(spec.method) +
                                  " is not on the GPU sampling path");
  }
  throw std::invalid_argument("run_sampler: unknown method");
}

// ------------------------------------------------------------ metrics
namespace {
double metric(int which, const PointCloud& cloud, std::span<const std::size_t> samples) {
  std::vector<int64_t> idx(samples.begin(), samples.end());
  double out = 0;
  const auto n = static_cast<int64_t>(cloud.size());
  const int rc = which == 0
      ? pcs_coverage_radius_host(flat(cloud), n, idx.data(), static_cast<int64_t>(idx.size()), &out)
      : pcs_separation_host(flat(cloud), n, idx.data(), static_cast<int64_t>(idx.size()), &out);
  if (rc != PCS_OK) raise(rc);
  return out;
}
}  // namespace

double coverage_radius(const PointCloud& cloud, std::span<const std::size_t> samples) {
  return metric(0, cloud, samples);
}

double separation(const PointCloud& cloud, std::span<const std::size_t> samples) {
  return metric(1, cloud, samples);
}

// ------------------------------------------------------------ order
PointCloud exact_sort(const PointCloud& cloud, Axis axis) {
  PointCloud out;
  out.points.resize(cloud.size());
  if (!cloud.points.empty()) {
    const int rc = pcs_exact_sort_host(flat(cloud), static_cast<int64_t>(cloud.size()),
                                       static_cast<int>(axis), out.points.front().data(), nullptr);
    if (rc != PCS_OK) raise(rc);
  }
  out.order_tag = OrderTag::exactly_sorted(axis);
  return out;
}

}  // namespace pcs
