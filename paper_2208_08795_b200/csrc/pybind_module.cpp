// Python module `paper_2208_08795_b200._core`: the reference's pcsample._core
// sampler surface (proj/bindings/pcsample_module.cpp:122-190) -- same names,
// keyword arguments, defaults, return types and exception classes -- plus raw
// device-pointer entry points used by the torch batched op. The samplers and
// exact_sort call the C-ABI host entries (include/pcs_gpu.h) on the numpy
// buffer directly; the rest goes through the C++ drop-in (include/pcs/*.hpp).
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "pcs/io.hpp"
#include "pcs/metrics.hpp"
#include "pcs/order.hpp"
#include "pcs/sampler.hpp"
#include "pcs_gpu.h"

namespace py = pybind11;

namespace {

using F64Array = py::array_t<double, py::array::c_style | py::array::forcecast>;

pcs::PointCloud to_cloud(const F64Array& a) {
  const auto info = a.request();
  if (info.ndim != 2 || info.shape[1] != 3) throw std::invalid_argument("expected an (N, 3) array");
  pcs::PointCloud cloud;
  const auto n = static_cast<std::size_t>(info.shape[0]);
  cloud.points.resize(n);
  const double* src = static_cast<const double*>(info.ptr);
  for (std::size_t i = 0; i < n; ++i) cloud.points[i] = {src[3 * i], src[3 * i + 1], src[3 * i + 2]};
  return cloud;
}

py::array_t<double> to_array(const pcs::PointCloud& cloud) {
  py::array_t<double> out({static_cast<py::ssize_t>(cloud.size()), py::ssize_t{3}});
  double* dst = out.mutable_data();
  for (std::size_t i = 0; i < cloud.size(); ++i)
    for (int a = 0; a < 3; ++a) dst[3 * i + a] = cloud.points[i][a];
  return out;
}

pcs::SeedPolicy policy_of(const std::string& first) {
  if (first == "random") return pcs::SeedPolicy::RandomFirstPoint;
  if (first == "fixed") return pcs::SeedPolicy::FixedFirstPoint;
  throw std::invalid_argument("first must be 'random' or 'fixed'");
}

pcs::Axis axis_of(const std::string& name) {
  const auto a = pcs::parse_axis(name);
  if (!a) throw std::invalid_argument("axis must be x, y, or z");
  return *a;
}

py::tuple to_tuple(const pcs::SampleResult& r) {
  const auto c = static_cast<py::ssize_t>(r.indices.size());
  py::array_t<std::int64_t> idx(c), sec(c);
  auto* pi = idx.mutable_data();
  auto* ps = sec.mutable_data();
  for (py::ssize_t i = 0; i < c; ++i) {
    pi[i] = static_cast<std::int64_t>(r.indices[i]);
    ps[i] = static_cast<std::int64_t>(r.sector_of[i]);
  }
  py::dict stats;
  stats["dist_evals"] = r.stats.dist_evals;
  stats["dist_writes"] = r.stats.dist_writes;
  stats["argmax_scans"] = r.stats.argmax_scans;
  stats["iterations"] = r.stats.iterations;
  return py::make_tuple(idx, sec, stats);
}

void check(int rc) {
  if (rc == PCS_OK) return;
  if (rc == PCS_ERR_INVALID_ARGUMENT) throw std::invalid_argument(pcs_last_error());
  throw std::runtime_error(pcs_last_error());
}

const double* xyz_of(const F64Array& a, std::int64_t* n) {
  const auto info = a.request();
  if (info.ndim != 2 || info.shape[1] != 3) throw std::invalid_argument("expected an (N, 3) array");
  *n = static_cast<std::int64_t>(info.shape[0]);
  return static_cast<const double*>(info.ptr);
}

// The samplers straight through the C-ABI host entry on the (forcecast,
// contiguous) array: the same validation order and messages as pcs::fps &
// co. (both use the C-ABI's checks), without the PointCloud copy -- a
// measurable share of a per-cloud call at 32K points.
py::tuple sample(const F64Array& points, int method, std::size_t c, std::size_t mm, std::size_t k,
                 pcs::SeedPolicy policy, std::uint64_t seed) {
  std::int64_t n = 0;
  const double* xyz = xyz_of(points, &n);
  // results are written only when c is feasible (c <= n)
  const auto cap = static_cast<py::ssize_t>(
      std::max<std::size_t>(1, std::min<std::size_t>(c, static_cast<std::size_t>(n))));
  py::array_t<std::int64_t> idx(cap), sec(cap);
  std::int64_t* pi = idx.mutable_data();
  std::int64_t* ps = sec.mutable_data();
  std::uint64_t st[4] = {0, 0, 0, 0};
  int rc;
  {
    py::gil_scoped_release nogil;
    rc = pcs_sample_host(method, xyz, n, static_cast<std::int64_t>(c), static_cast<std::int64_t>(mm),
                         static_cast<std::int64_t>(k),
                         policy == pcs::SeedPolicy::RandomFirstPoint ? PCS_RANDOM_FIRST_POINT
                                                                     : PCS_FIXED_FIRST_POINT,
                         seed, 1, pi, ps, st);
  }
  check(rc);
  py::dict stats;
  stats["dist_evals"] = st[0];
  stats["dist_writes"] = st[1];
  stats["argmax_scans"] = st[2];
  stats["iterations"] = st[3];
  return py::make_tuple(idx, sec, stats);
}

}  // namespace

PYBIND11_MODULE(_core, m) {
  m.doc() = "B200-native FPS / AFPS / NPDU-FPS / NPDU-AFPS sampling (arXiv 2208.08795)";

  m.def("fps",
        [](const F64Array& points, std::size_t c, std::uint64_t seed, const std::string& first) {
          const auto policy = policy_of(first);
          return sample(points, PCS_METHOD_FPS, c, 1, 0, policy, seed);
        },
        py::arg("points"), py::arg("c"), py::arg("seed") = 0, py::arg("first") = "random");
  m.def("afps",
        [](const F64Array& points, std::size_t c, std::size_t mm, std::uint64_t seed,
           const std::string& first, unsigned threads) {
          const auto policy = policy_of(first);
          (void)threads;  // accepted for the reference signature; the GPU schedule is fixed
          return sample(points, PCS_METHOD_AFPS, c, mm, 0, policy, seed);
        },
        py::arg("points"), py::arg("c"), py::arg("m"), py::arg("seed") = 0,
        py::arg("first") = "random", py::arg("threads") = 1);
  m.def("npdu_fps",
        [](const F64Array& points, std::size_t c, std::size_t k, std::uint64_t seed,
           const std::string& first) {
          const auto policy = policy_of(first);
          return sample(points, PCS_METHOD_NPDU_FPS, c, 1, k, policy, seed);
        },
        py::arg("points"), py::arg("c"), py::arg("k"), py::arg("seed") = 0,
        py::arg("first") = "random");
  m.def("npdu_afps",
        [](const F64Array& points, std::size_t c, std::size_t mm, std::size_t k, std::uint64_t seed,
           const std::string& first, unsigned threads) {
          const auto policy = policy_of(first);
          (void)threads;
          return sample(points, PCS_METHOD_NPDU_AFPS, c, mm, k, policy, seed);
        },
        py::arg("points"), py::arg("c"), py::arg("m"), py::arg("k"), py::arg("seed") = 0,
        py::arg("first") = "random", py::arg("threads") = 1);
  m.def("exact_sort",
        [](const F64Array& points, const std::string& axis) {
          const auto ax = axis_of(axis);
          std::int64_t n = 0;
          const double* xyz = xyz_of(points, &n);
          py::array_t<double> out({static_cast<py::ssize_t>(n), py::ssize_t{3}});
          double* dst = out.mutable_data();
          int rc = PCS_OK;
          if (n > 0) {
            py::gil_scoped_release nogil;
            rc = pcs_exact_sort_host(xyz, n, static_cast<int>(ax), dst, nullptr);
          }
          check(rc);
          return out;
        },
        py::arg("points"), py::arg("axis") = "x");
  m.def("local_fps",
        [](const F64Array& points, std::size_t begin, std::size_t end, std::size_t quota,
           std::optional<std::size_t> k, std::uint64_t seed, const std::string& first,
           bool trace) -> py::tuple {
          const auto policy = policy_of(first);
          const pcs::PointCloud cloud = to_cloud(points);
          pcs::DistanceTrace tr;
          pcs::SampleResult r;
          {
            py::gil_scoped_release nogil;
            r = pcs::detail::local_fps(cloud, {begin, end}, quota, k, policy, seed, trace ? &tr : nullptr);
          }
          py::tuple base = to_tuple(r);
          if (!trace) return base;
          const auto rows = static_cast<py::ssize_t>(tr.snapshots.size());
          py::array_t<double> snaps({rows, static_cast<py::ssize_t>(end - begin)});
          double* dst = snaps.mutable_data();
          for (py::ssize_t p = 0; p < rows; ++p)
            for (std::size_t j = 0; j < end - begin; ++j) dst[p * (end - begin) + j] = tr.snapshots[p][j];
          return py::tuple(py::make_tuple(base[0], base[1], base[2], snaps));
        },
        py::arg("points"), py::arg("begin"), py::arg("end"), py::arg("quota"),
        py::arg("k") = py::none(), py::arg("seed") = 0, py::arg("first") = "random",
        py::arg("trace") = false);

  // cloud files (proj/src/io.cpp); runtime_error -> RuntimeError
  auto format_of = [](const std::string& name) {
    const auto f = pcs::parse_format(name);
    if (!f) throw std::invalid_argument("format must be xyz_text or f32_bin");
    return *f;
  };
  m.def("read_cloud",
        [format_of](const std::string& path, const std::string& format) {
          const auto f = format_of(format);
          pcs::PointCloud cloud;
          {
            py::gil_scoped_release nogil;
            cloud = pcs::read_cloud(path, f);
          }
          return to_array(cloud);
        },
        py::arg("path"), py::arg("format") = "f32_bin");
  m.def("write_cloud",
        [format_of](const F64Array& points, const std::string& path, const std::string& format) {
          const auto f = format_of(format);
          const pcs::PointCloud cloud = to_cloud(points);
          py::gil_scoped_release nogil;
          pcs::write_cloud(cloud, path, f);
        },
        py::arg("points"), py::arg("path"), py::arg("format") = "f32_bin");

  // metrics (proj/bindings/pcsample_module.cpp:198-210)
  auto indices_of = [](const py::array_t<std::int64_t>& a) {
    const auto v = a.unchecked<1>();
    std::vector<std::size_t> out;
    out.reserve(static_cast<std::size_t>(v.shape(0)));
    for (py::ssize_t i = 0; i < v.shape(0); ++i) {
      if (v(i) < 0) throw std::invalid_argument("negative index");
      out.push_back(static_cast<std::size_t>(v(i)));
    }
    return out;
  };
  m.def("coverage_radius",
        [indices_of](const F64Array& points, const py::array_t<std::int64_t>& samples) {
          const pcs::PointCloud cloud = to_cloud(points);
          const auto idx = indices_of(samples);
          py::gil_scoped_release nogil;
          return pcs::coverage_radius(cloud, idx);
        },
        py::arg("points"), py::arg("samples"));
  m.def("separation",
        [indices_of](const F64Array& points, const py::array_t<std::int64_t>& samples) {
          const pcs::PointCloud cloud = to_cloud(points);
          const auto idx = indices_of(samples);
          py::gil_scoped_release nogil;
          return pcs::separation(cloud, idx);
        },
        py::arg("points"), py::arg("samples"));
  m.def("metric_device",
        [](int which, int coord_dtype, std::uintptr_t xyz, std::int64_t batch, std::int64_t n,
           int index_dtype, std::uintptr_t idx, std::int64_t c, std::uintptr_t out,
           std::uintptr_t stream) {
          auto fn = which == 0 ? pcs_gpu_coverage_radius : pcs_gpu_separation;
          check(fn(coord_dtype, reinterpret_cast<const void*>(xyz), batch, n, index_dtype,
                   reinterpret_cast<const void*>(idx), c, reinterpret_cast<double*>(out),
                   reinterpret_cast<void*>(stream)));
        });

  // Raw device-pointer entry points (torch tensors are unwrapped in Python).
  m.def("sample_device",
        [](int method, int coord_dtype, std::uintptr_t xyz, std::int64_t batch, std::int64_t n,
           std::int64_t c, std::int64_t mm, std::int64_t k, int seed_policy, std::uint64_t seed,
           std::uintptr_t seeds, int index_dtype, std::uintptr_t out_idx, std::uintptr_t out_sector,
           std::uintptr_t out_stats, std::uintptr_t stream, std::int64_t index_base,
           std::int64_t sector_base, std::uintptr_t perm) {
          pcs_gpu_args a{};
          a.index_base = index_base;
          a.sector_base = sector_base;
          a.method = method;
          a.coord_dtype = coord_dtype;
          a.xyz = reinterpret_cast<const void*>(xyz);
          a.batch = batch;
          a.n = n;
          a.c = c;
          a.m = mm;
          a.k = k;
          a.seed_policy = seed_policy;
          a.seed = seed;
          a.seeds = reinterpret_cast<const std::uint64_t*>(seeds);
          a.index_dtype = index_dtype;
          a.out_indices = reinterpret_cast<void*>(out_idx);
          a.out_sector = reinterpret_cast<std::int32_t*>(out_sector);
          a.out_stats = reinterpret_cast<std::uint64_t*>(out_stats);
          a.perm = reinterpret_cast<const std::int32_t*>(perm);
          check(pcs_gpu_sample(&a, reinterpret_cast<void*>(stream)));
        },
        py::arg("method"), py::arg("coord_dtype"), py::arg("xyz"), py::arg("batch"), py::arg("n"),
        py::arg("c"), py::arg("m"), py::arg("k"), py::arg("seed_policy"), py::arg("seed"),
        py::arg("seeds"), py::arg("index_dtype"), py::arg("out_idx"), py::arg("out_sector"),
        py::arg("out_stats"), py::arg("stream"), py::arg("index_base") = 0,
        py::arg("sector_base") = 0, py::arg("perm") = 0);
  // the dispatch decision of pcs_gpu_sample (no device work)
  m.def("kernel_family",
        [](int method, int coord_dtype, std::int64_t batch, std::int64_t n, std::int64_t c,
           std::int64_t mm, std::int64_t k) {
          pcs_gpu_args a{};
          a.method = method;
          a.coord_dtype = coord_dtype;
          a.batch = batch;
          a.n = n;
          a.c = c;
          a.m = mm;
          a.k = k;
          char name[128];
          check(pcs_kernel_family(&a, name, sizeof(name)));
          return std::string(name);
        },
        py::arg("method"), py::arg("coord_dtype"), py::arg("batch"), py::arg("n"), py::arg("c"),
        py::arg("m"), py::arg("k"));
  m.def("reload_knobs", []() { pcs_debug_reload_knobs(); });
  // the host-buffer batch entry (pointers into host memory, e.g. pinned
  // torch tensors); the GIL is released for the synchronous call
  m.def("sample_host_ptr",
        [](int method, int coord_dtype, std::uintptr_t xyz, std::int64_t batch, std::int64_t n,
           std::int64_t c, std::int64_t mm, std::int64_t k, int seed_policy, std::uint64_t seed,
           std::uintptr_t seeds, int index_dtype, std::uintptr_t out_idx, std::uintptr_t out_sector,
           std::uintptr_t out_stats, int sort_axis, std::uintptr_t out_perm, int chunks,
           std::int64_t index_base, std::int64_t sector_base, std::vector<int> devices) {
          pcs_gpu_args a{};
          a.index_base = index_base;
          a.sector_base = sector_base;
          a.method = method;
          a.coord_dtype = coord_dtype;
          a.xyz = reinterpret_cast<const void*>(xyz);
          a.batch = batch;
          a.n = n;
          a.c = c;
          a.m = mm;
          a.k = k;
          a.seed_policy = seed_policy;
          a.seed = seed;
          a.seeds = reinterpret_cast<const std::uint64_t*>(seeds);
          a.index_dtype = index_dtype;
          a.out_indices = reinterpret_cast<void*>(out_idx);
          a.out_sector = reinterpret_cast<std::int32_t*>(out_sector);
          a.out_stats = reinterpret_cast<std::uint64_t*>(out_stats);
          int rc;
          {
            py::gil_scoped_release nogil;
            if (devices.empty())
              rc = pcs_sample_host_batch(&a, sort_axis, reinterpret_cast<std::int32_t*>(out_perm),
                                         chunks);
            else
              rc = pcs_sample_host_multi(&a, sort_axis, reinterpret_cast<std::int32_t*>(out_perm),
                                         devices.data(), static_cast<std::int32_t>(devices.size()));
          }
          check(rc);
        },
        py::arg("method"), py::arg("coord_dtype"), py::arg("xyz"), py::arg("batch"), py::arg("n"),
        py::arg("c"), py::arg("m"), py::arg("k"), py::arg("seed_policy"), py::arg("seed"),
        py::arg("seeds"), py::arg("index_dtype"), py::arg("out_idx"), py::arg("out_sector"),
        py::arg("out_stats"), py::arg("sort_axis"), py::arg("out_perm"), py::arg("chunks") = 0,
        py::arg("index_base") = 0, py::arg("sector_base") = 0,
        py::arg("devices") = std::vector<int>{});
  m.def("sort_device",
        [](int coord_dtype, std::uintptr_t xyz, std::int64_t batch, std::int64_t n, int axis,
           std::uintptr_t out_xyz, std::uintptr_t out_perm, std::uintptr_t stream) {
          check(pcs_gpu_sort_axis(coord_dtype, reinterpret_cast<const void*>(xyz), batch, n, axis,
                                  reinterpret_cast<void*>(out_xyz),
                                  reinterpret_cast<std::int32_t*>(out_perm),
                                  reinterpret_cast<void*>(stream)));
        });
  m.def("validate",
        [](int method, std::int64_t n, std::int64_t c, std::int64_t mm, std::int64_t k) {
          // Host-side argument checks only (no device needed): raises the
          // reference's ValueError, or returns None.
          pcs_gpu_args a{};
          a.method = method;
          a.n = n;
          a.c = c;
          a.m = mm;
          a.k = k;
          a.batch = 0;  // batch 0: validated, nothing launched
          check(pcs_gpu_sample(&a, nullptr));
        });
  m.attr("ABI_VERSION") = pcs_abi_version();
}
