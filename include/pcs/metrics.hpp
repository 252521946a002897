// Drop-in for the sample-quality metrics of pcs/metrics.hpp
// (proj/include/pcs/metrics.hpp:16-22), served by GPU kernels
// (csrc/metrics_kernels.cu) and bit-identical to the reference's.
// compare() / report_csv() / report_json() (the QualityReport tooling) are
// outside the GPU path.
#pragma once

#include <cstddef>
#include <span>

#include "pcs/point_cloud.hpp"

namespace pcs {

// max over points of the distance to the nearest sample (fill distance)
double coverage_radius(const PointCloud& cloud, std::span<const std::size_t> samples);

// min pairwise distance among the samples
double separation(const PointCloud& cloud, std::span<const std::size_t> samples);

}  // namespace pcs
