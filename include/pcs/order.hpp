// Drop-in for pcs/order.hpp's exact_sort (proj/include/pcs/order.hpp:10),
// run as the device key sort (pcs_gpu_sort_axis).
#pragma once

#include "pcs/point_cloud.hpp"

namespace pcs {

// Stable ascending sort along `axis`; the result is tagged exactly_sorted.
PointCloud exact_sort(const PointCloud& cloud, Axis axis);

}  // namespace pcs
