// Cloud file formats, the reference's semantics and messages
// (proj/src/io.cpp:32-122): xyz_text with '#' comments and blank lines,
// f32_bin little-endian fp32 widened exactly to double. Native host code;
// exposed as the C++ drop-in (pcs::read_cloud / write_cloud), through the
// C-ABI (pcs_read_cloud_host / pcs_write_cloud_host) and to Python.
#include <bit>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "internal.h"
#include "pcs/io.hpp"
#include "pcs_gpu.h"

static_assert(std::endian::native == std::endian::little, "f32_bin is little-endian");

namespace pcs {
namespace {

bool blank(const std::string& s) { return s.find_first_not_of(" \t\r\f\v") == std::string::npos; }

PointCloud read_text(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open " + path.string());
  PointCloud cloud;
  std::string line;
  for (std::size_t no = 1; std::getline(in, line); ++no) {
    const auto hash = line.find('#');
    if (hash != std::string::npos) line.erase(hash);
    if (blank(line)) continue;
    std::istringstream fields(line);
    Point p;
    if (!(fields >> p[0] >> p[1] >> p[2]))
      throw std::runtime_error(path.string() + ":" + std::to_string(no) + ": expected three coordinates");
    std::string extra;
    if (fields >> extra)
      throw std::runtime_error(path.string() + ":" + std::to_string(no) +
                               ": trailing data after three coordinates");
    cloud.points.push_back(p);
  }
  if (cloud.points.empty()) throw std::runtime_error(path.string() + ": no points (empty file)");
  return cloud;
}

PointCloud read_binary(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) throw std::runtime_error("cannot open " + path.string());
  const std::streamoff bytes = in.tellg();
  if (bytes == 0) throw std::runtime_error(path.string() + ": no points (empty file)");
  if (bytes % 12 != 0)
    throw std::runtime_error(path.string() + ": truncated binary cloud (" + std::to_string(bytes) +
                             " bytes, not a multiple of 12)");
  in.seekg(0);
  std::vector<float> raw(static_cast<std::size_t>(bytes) / 4);
  if (!in.read(reinterpret_cast<char*>(raw.data()), bytes))
    throw std::runtime_error(path.string() + ": read failure");
  PointCloud cloud;
  cloud.points.resize(raw.size() / 3);
  for (std::size_t i = 0; i < cloud.points.size(); ++i)
    cloud.points[i] = {raw[3 * i], raw[3 * i + 1], raw[3 * i + 2]};
  return cloud;
}

}  // namespace

const char* format_name(CloudFormat format) {
  return format == CloudFormat::XyzText ? "xyz_text" : "f32_bin";
}

std::optional<CloudFormat> parse_format(std::string_view name) {
  if (name == "xyz_text" || name == "xyz") return CloudFormat::XyzText;
  if (name == "f32_bin" || name == "f32") return CloudFormat::F32Bin;
  return std::nullopt;
}

PointCloud read_cloud(const std::filesystem::path& path, CloudFormat format) {
  PointCloud cloud = format == CloudFormat::XyzText ? read_text(path) : read_binary(path);
  cloud.order_tag = OrderTag::unsorted();  // storage order kept, not trusted
  return cloud;
}

void write_cloud(const PointCloud& cloud, const std::filesystem::path& path, CloudFormat format) {
  if (format == CloudFormat::XyzText) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot write " + path.string());
    char line[96];
    for (const Point& p : cloud.points) {
      std::snprintf(line, sizeof line, "%.17g %.17g %.17g\n", p[0], p[1], p[2]);
      out << line;
    }
    if (!out.flush()) throw std::runtime_error("write failed for " + path.string());
    return;
  }
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write " + path.string());
  std::vector<float> raw(cloud.points.size() * 3);
  for (std::size_t i = 0; i < cloud.points.size(); ++i)
    for (int a = 0; a < 3; ++a) raw[3 * i + a] = static_cast<float>(cloud.points[i][a]);
  out.write(reinterpret_cast<const char*>(raw.data()), static_cast<std::streamsize>(raw.size() * 4));
  if (!out.flush()) throw std::runtime_error("write failed for " + path.string());
}

}  // namespace pcs

extern "C" {

long long pcs_read_cloud_host(const char* path, int32_t format, double* out_xyz, int64_t capacity) {
  pcs_internal::clear_error();
  try {
    const auto cloud = pcs::read_cloud(path, format == 0 ? pcs::CloudFormat::XyzText
                                                         : pcs::CloudFormat::F32Bin);
    const int64_t n = static_cast<int64_t>(cloud.size());
    if (out_xyz)
      for (int64_t i = 0; i < n && i < capacity; ++i)
        std::memcpy(out_xyz + 3 * i, cloud.points[static_cast<std::size_t>(i)].data(), 24);
    return n;
  } catch (const std::exception& e) {
    pcs_internal::set_error(e.what());
    return -1;
  }
}

int pcs_write_cloud_host(const char* path, int32_t format, const double* xyz, int64_t n) {
  pcs_internal::clear_error();
  try {
    pcs::PointCloud cloud;
    cloud.points.resize(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) std::memcpy(cloud.points[static_cast<std::size_t>(i)].data(), xyz + 3 * i, 24);
    pcs::write_cloud(cloud, path, format == 0 ? pcs::CloudFormat::XyzText : pcs::CloudFormat::F32Bin);
    return PCS_OK;
  } catch (const std::exception& e) {
    pcs_internal::set_error(e.what());
    return PCS_ERR_INVALID_ARGUMENT;
  }
}

}  // extern "C"
