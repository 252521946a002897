// C++ drop-in API test (namespace pcs, include/pcs/*.hpp) against the
// reference's own unit-test known answers -- the cases of
// proj/tests/test_sampler.cpp and test_order.cpp re-stated here because the
// reference's doctest suites cannot build (vendor/doctest.h is absent,
// SURVEY.md 8(c)). Links paper_2208_08795_b200/lib/libpcs_gpu.so; needs a GPU.
// Built by paper_2208_08795_b200/_build.py, run by tests/test_gpu_parity.py.
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "pcs/order.hpp"
#include "pcs/point_cloud.hpp"
#include "pcs/rng.hpp"
#include "pcs/sampler.hpp"
#include "pcs/sampler_spec.hpp"
#include "pcs/sectors.hpp"

namespace {

int g_failures = 0;

void expect(bool ok, const char* what, int line) {
  if (!ok) {
    std::fprintf(stderr, "FAIL line %d: %s\n", line, what);
    ++g_failures;
  }
}
#define EXPECT(cond) expect((cond), #cond, __LINE__)

template <typename Fn>
void expect_invalid(Fn&& fn, const std::string& msg, int line) {
  try {
    fn();
    std::fprintf(stderr, "FAIL line %d: no exception (want \"%s\")\n", line, msg.c_str());
    ++g_failures;
  } catch (const std::invalid_argument& e) {
    if (msg != e.what()) {
      std::fprintf(stderr, "FAIL line %d: \"%s\" != \"%s\"\n", line, e.what(), msg.c_str());
      ++g_failures;
    }
  }
}
#define EXPECT_INVALID(expr, msg) expect_invalid([&] { (void)(expr); }, (msg), __LINE__)

pcs::PointCloud line(std::size_t n) {
  pcs::PointCloud c;
  for (std::size_t i = 0; i < n; ++i) c.points.push_back({static_cast<double>(i), 0.0, 0.0});
  return c;
}

pcs::PointCloud random_cloud(std::size_t n, std::uint64_t seed) {
  pcs::SplitMix64 rng(seed);
  pcs::PointCloud c;
  for (std::size_t i = 0; i < n; ++i)
    c.points.push_back({rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-1, 1)});
  return c;
}

std::vector<std::size_t> idx(std::initializer_list<std::size_t> v) { return v; }

constexpr auto Fixed = pcs::SeedPolicy::FixedFirstPoint;
constexpr auto Random = pcs::SeedPolicy::RandomFirstPoint;

}  // namespace

int main() {
  // FPS line-cloud traces, proj/tests/test_sampler.cpp:88-100
  EXPECT(pcs::fps(line(4), 2, Fixed, 0).indices == idx({0, 3}));
  EXPECT(pcs::fps(line(4), 3, Fixed, 0).indices == idx({0, 3, 1}));
  EXPECT(pcs::fps(line(4), 4, Fixed, 0).indices == idx({0, 3, 1, 2}));
  // op counts, :102-113
  {
    const auto r = pcs::fps(random_cloud(100, 17), 25, Random, 5);
    EXPECT(r.stats.dist_evals == 2400 && r.stats.argmax_scans == 2400 && r.stats.iterations == 24);
    EXPECT(r.sector_of == std::vector<std::uint32_t>(25, 0));
    const auto one = pcs::fps(random_cloud(100, 17), 1, Fixed, 0);
    EXPECT(one.indices == idx({0}) && one.stats == pcs::OpStats{});
  }
  // AFPS: m = 1 equals fps; 2048/512/32 -> 30720 evals; uneven 10/4/3 -> 4;
  // m = c; confinement and quotas; thread-count independence (:184-252)
  {
    const auto cloud = random_cloud(500, 3);
    const auto f = pcs::fps(cloud, 60, Random, 9);
    const auto a = pcs::afps(cloud, 60, 1, Random, 9);
    EXPECT(f.indices == a.indices && f.stats == a.stats);
    const auto big = pcs::afps(random_cloud(2048, 2), 512, 32, Random, 1);
    EXPECT(big.stats.dist_evals == 30720);
    EXPECT(pcs::afps(random_cloud(10, 3), 4, 3, Fixed, 0).stats.dist_evals == 4);
    const auto mc = pcs::afps(random_cloud(100, 5), 20, 20, Random, 77);
    EXPECT(mc.stats.dist_evals == 0);
    for (std::size_t i = 0; i < 20; ++i) EXPECT(mc.sector_of[i] == i);
    const auto plan = pcs::SectorPlan::make(2048, 512, 32);
    std::vector<std::size_t> per(32, 0);
    for (std::size_t i = 0; i < big.indices.size(); ++i) {
      const auto s = big.sector_of[i];
      EXPECT(plan.ranges[s].contains(big.indices[i]));
      ++per[s];
    }
    for (std::size_t s = 0; s < 32; ++s) EXPECT(per[s] == plan.quotas[s]);
    const auto t4 = pcs::afps(random_cloud(2048, 2), 512, 32, Random, 1, 4);
    EXPECT(t4.indices == big.indices && t4.stats == big.stats);
  }
  // NPDU: line traces k=2 -> [0,1,2] (evals 3, writes 2, iterations 2), k=4 ->
  // [0,2,4]; full window equals fps; k=1 gives c-1 evals (:267-316)
  {
    const auto k2 = pcs::npdu_fps(line(8), 3, 2, Fixed, 0);
    EXPECT(k2.indices == idx({0, 1, 2}));
    EXPECT(k2.stats.dist_evals == 3 && k2.stats.dist_writes == 2 && k2.stats.iterations == 2);
    EXPECT(pcs::npdu_fps(line(8), 3, 4, Fixed, 0).indices == idx({0, 2, 4}));
    const auto cloud = random_cloud(300, 11);
    const auto f = pcs::fps(cloud, 40, Random, 4);
    const auto w = pcs::npdu_fps(cloud, 40, 600, Random, 4);
    EXPECT(f.indices == w.indices && f.stats == w.stats);
    EXPECT(pcs::npdu_fps(random_cloud(64, 4), 10, 1, Random, 8).stats.dist_evals == 9);
    const auto na = pcs::npdu_afps(random_cloud(2048, 6), 512, 32, 16, Random, 2);
    EXPECT(na.stats.dist_evals <= 7680);
    const auto na4 = pcs::npdu_afps(random_cloud(2048, 6), 512, 32, 16, Random, 2, 4);
    EXPECT(na4.indices == na.indices && na4.stats == na.stats);
  }
  // degenerate clouds: no duplicates (:410-433)
  {
    pcs::PointCloud same;
    same.points.assign(50, pcs::Point{0.25, -0.5, 1.0});
    const auto r = pcs::fps(same, 50, Fixed, 0);
    std::vector<int> seen(50, 0);
    for (auto i : r.indices) seen[i]++;
    for (int s : seen) EXPECT(s == 1);
    const auto na = pcs::npdu_afps(same, 50, 5, 3, Fixed, 0);
    std::vector<int> seen2(50, 0);
    for (auto i : na.indices) seen2[i]++;
    for (int s : seen2) EXPECT(s == 1);
  }
  // run_sampler dispatch (:435-446); RPS / grid voxel have no GPU path
  {
    const auto cloud = random_cloud(400, 21);
    pcs::SamplerSpec spec;
    spec.method = pcs::Method::NpduAfps;
    spec.c = 64;
    spec.m = 8;
    spec.k = 9;
    spec.seed = 13;
    const auto r = pcs::run_sampler(cloud, spec);
    const auto d = pcs::npdu_afps(cloud, 64, 8, 9, Random, 13);
    EXPECT(r.indices == d.indices && r.stats == d.stats);
    spec.method = pcs::Method::Rps;
    bool threw = false;
    try {
      pcs::run_sampler(cloud, spec);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    EXPECT(threw);
  }
  // errors, same messages and order as the reference (sampler.cpp:20-23,
  // sectors.cpp:10-11,28,44-47, sampler.cpp:89-94)
  {
    const auto cloud = random_cloud(10, 1);
    EXPECT_INVALID(pcs::fps(cloud, 0, Fixed, 0), "fps: c must be >= 1");
    EXPECT_INVALID(pcs::fps(cloud, 11, Fixed, 0), "fps: c exceeds point count");
    EXPECT_INVALID(pcs::afps(cloud, 4, 0, Fixed, 0), "partition_sectors: m must be >= 1");
    EXPECT_INVALID(pcs::afps(cloud, 4, 5, Fixed, 0), "allocate_samples: m exceeds sample count");
    EXPECT_INVALID(pcs::npdu_fps(cloud, 4, 0, Fixed, 0), "local_fps: window size must be >= 1");
  }
  // exact_sort: stable on ties, -0.0 == +0.0 keeps storage order
  // (proj/tests/test_order.cpp:26-48)
  {
    pcs::PointCloud c;
    c.points = {{1.0, 0, 0}, {-0.0, 1, 0}, {0.0, 2, 0}, {1.0, 3, 0}, {-2.5, 4, 0}, {0.0, 5, 0}};
    const auto s = pcs::exact_sort(c, pcs::Axis::X);
    const double want_y[] = {4, 1, 2, 5, 0, 3};
    for (int i = 0; i < 6; ++i) EXPECT(s.points[i][1] == want_y[i]);
    EXPECT(s.order_tag == pcs::OrderTag::exactly_sorted(pcs::Axis::X));
    const auto big = random_cloud(40000, 8);
    const auto sb = pcs::exact_sort(big, pcs::Axis::Z);
    for (std::size_t i = 1; i < sb.size(); ++i) EXPECT(sb.points[i - 1][2] <= sb.points[i][2]);
  }
  if (g_failures) {
    std::fprintf(stderr, "%d failure(s)\n", g_failures);
    return 1;
  }
  std::printf("test_pcs_api: all checks passed\n");
  return 0;
}
