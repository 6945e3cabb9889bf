// convert.hpp -- C++ transform entry points (drop-in for
// /root/reference/proj/include/spmvtk/convert.hpp:9-33).  The forward
// transforms run on the GPU (upload, sm_100a kernels, download); results are
// bit-identical to the reference.  coo_to_crs / ell_to_crs / canonicalize
// rebuild canonical CRS on the device too (kernels_inverse.cu).
#pragma once

#include <cstdint>

#include "spmvtk/formats.hpp"

namespace spmvtk {

inline constexpr std::uint64_t kNoByteLimit = 0;

CooMatrix crs_to_coo_row(const CrsMatrix& m);
CcsMatrix crs_to_ccs(const CrsMatrix& m);          // rows ascend in each column
CooMatrix ccs_to_coo_col(const CcsMatrix& m);
CooMatrix crs_to_coo_col(const CrsMatrix& m);      // CRS -> CCS -> COO (column-major)

std::uint64_t estimate_ell_bytes(const CrsMatrix& m, int value_bytes = 8, int index_bytes = 8);
// throws Error(MemoryLimit) when the 16-byte/slot estimate exceeds max_bytes
EllMatrix crs_to_ell(const CrsMatrix& m, std::uint64_t max_bytes = kNoByteLimit);

CrsMatrix coo_to_crs(const CooMatrix& m);  // canonical; refuses duplicate positions
CrsMatrix ell_to_crs(const EllMatrix& m);  // drops exactly the padding slots

}  // namespace spmvtk
