// Drop-in for pcs/sampler.hpp (proj/include/pcs/sampler.hpp:16-77), served by
// the B200 kernels through the C-ABI in pcs_gpu.h. Same signatures, same
// results (indices, sector_of, OpStats), same std::invalid_argument
// messages; CUDA failures throw std::runtime_error. `threads` is accepted and
// ignored: every sector of the call runs in one launch.
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "pcs/point_cloud.hpp"
#include "pcs/sampler_spec.hpp"
#include "pcs/sectors.hpp"

namespace pcs {

// d[] after every update pass, for property tests.
struct DistanceTrace {
  std::vector<std::vector<double>> snapshots;
};

namespace detail {

// Greedy farthest-point loop over one contiguous storage range; window_k
// empty = update the whole range each iteration.
SampleResult local_fps(const PointCloud& cloud, IndexRange sector, std::size_t quota,
                       std::optional<std::size_t> window_k, SeedPolicy seed_policy,
                       std::uint64_t seed, DistanceTrace* trace = nullptr);

}  // namespace detail

SampleResult fps(const PointCloud& cloud, std::size_t c, SeedPolicy seed_policy,
                 std::uint64_t seed);

SampleResult afps(const PointCloud& cloud, std::size_t c, std::size_t m,
                  SeedPolicy seed_policy, std::uint64_t seed, unsigned threads = 1);

SampleResult npdu_fps(const PointCloud& cloud, std::size_t c, std::size_t k,
                      SeedPolicy seed_policy, std::uint64_t seed);

SampleResult npdu_afps(const PointCloud& cloud, std::size_t c, std::size_t m, std::size_t k,
                       SeedPolicy seed_policy, std::uint64_t seed, unsigned threads = 1);

// Fps / Afps / NpduFps / NpduAfps; Rps and GridVoxel throw
// std::invalid_argument (outside the GPU path, no CPU fallback).
SampleResult run_sampler(const PointCloud& cloud, const SamplerSpec& spec,
                         unsigned threads = 1);

}  // namespace pcs
