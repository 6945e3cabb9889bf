// generators.hpp -- host-side matrix generators (see generators.cpp).
#pragma once

#include <cstdint>
#include <vector>

namespace spmvtk::gen {

// A host CRS in either index width: the reference generators produce int64
// 1-based arrays (row_ptr / col_idx), the BASELINE workloads int32 0-based
// (row_ptr32 / col32) to halve host memory for 67M-entry matrices.
struct HostCrs {
  std::int64_t n = 0;           // rows held (a row-block shard: the block's rows)
  std::int64_t ncols = -1;      // columns (-1: n, a square matrix)
  std::int64_t row_offset = 0;  // global index of row 0 (shards)
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
// Rank `rank` of `world`'s row block of the same matrix, generated alone
// (only the RNG blocks overlapping the rows are filled): rows [r0, r1) of the
// entry-balanced partition (partition_rows), global columns, ncols = n.
HostCrs baseline_shard(int config, std::int64_t param, double dparam, std::uint64_t seed,
                       int rank, int world);
// Entry-balanced contiguous row blocks: begin[k] = first row whose start is
// at least k*nnz/world (begin[0] = 0, begin[world] = n).  row_ptr: n + 1
// offsets (any base: only differences are used).
std::vector<std::int64_t> partition_rows(const std::int64_t* row_ptr, std::int64_t n, int world);
void vector_u11(std::int64_t n, std::uint64_t seed, double* out);

}  // namespace spmvtk::gen
