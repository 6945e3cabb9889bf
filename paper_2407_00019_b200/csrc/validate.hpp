// validate.hpp -- structural validation on the GPU (kernels_validate.cu),
// behind the reference's validate() overloads (formats.cpp:75-182).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace spmvtk::dev {

// CRS (seg_kind "row") / CCS (seg_kind "column")
std::vector<std::string> validate_segments(std::int64_t n, const std::vector<std::int64_t>& ptr,
                                           const std::vector<std::int64_t>& idx,
                                           std::size_t nvalues, const char* ptr_name,
                                           const char* idx_name, const char* idx_kind,
                                           const char* seg_kind);
// COO; ordering 0 row-major, 1 column-major, 2 unordered
std::vector<std::string> validate_triplets(std::int64_t n, const std::vector<std::int64_t>& row,
                                           const std::vector<std::int64_t>& col,
                                           std::size_t nvalues, int ordering);
std::vector<std::string> validate_ell(std::int64_t n, std::int64_t bc,
                                      const std::vector<double>& values,
                                      const std::vector<std::int64_t>& col,
                                      const std::vector<std::int64_t>& count,
                                      std::int64_t stored_nnz);

}  // namespace spmvtk::dev
