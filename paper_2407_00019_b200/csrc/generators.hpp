// generators.hpp -- host-side matrix generators (see generators.cpp).
#pragma once

#include <cstdint>
#include <vector>

namespace spmvtk::gen {

// A host CRS in either index width: the reference generators produce int64
// 1-based arrays (row_ptr / col_idx), the BASELINE workloads int32 0-based
// (row_ptr32 / col32) to halve host memory for 67M-entry matrices.
struct HostCrs {
  std::int64_t n = 0;
  int base = 1;
  std::vector<std::int64_t> row_ptr, col_idx;
  std::vector<std::int32_t> row_ptr32, col32;
  std::vector<double> values;
  bool wide() const { return !row_ptr.empty(); }
  std::int64_t nnz() const { return static_cast<std::int64_t>(values.size()); }
};

HostCrs banded(std::int64_t n, std::int64_t half_width);
HostCrs skewed(std::int64_t n, std::int64_t base_deg, std::int64_t heavy_rows,
               std::int64_t heavy_deg, std::uint64_t seed);
HostCrs cv_target(std::int64_t n, double mean_deg, double target_dmat, std::uint64_t seed);
HostCrs baseline(int config, std::int64_t param, double dparam, std::uint64_t seed);
void vector_u11(std::int64_t n, std::uint64_t seed, double* out);

}  // namespace spmvtk::gen
