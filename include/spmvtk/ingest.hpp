// ingest.hpp -- Matrix Market I/O and generators (drop-in for
// /root/reference/proj/include/spmvtk/ingest.hpp:12-29).  Host-side; the
// generators reproduce the reference's matrices byte for byte per seed.
#pragma once

#include <cstdint>
#include <filesystem>

#include "spmvtk/formats.hpp"

namespace spmvtk {

CrsMatrix read_matrix_market(const std::filesystem::path& path);
void write_matrix_market(const CrsMatrix& m, const std::filesystem::path& path);

CrsMatrix gen_banded(index_t n, index_t half_width);
CrsMatrix gen_skewed(index_t n, index_t base_deg, index_t heavy_rows, index_t heavy_deg,
                     std::uint64_t seed);
CrsMatrix gen_cv_target(index_t n, double mean_deg, double target_dmat, std::uint64_t seed);

}  // namespace spmvtk
