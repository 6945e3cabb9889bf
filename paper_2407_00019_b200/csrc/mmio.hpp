// mmio.hpp -- Matrix Market read / write (see mmio.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "generators.hpp"

namespace spmvtk::mm {

gen::HostCrs read(const std::string& path);  // int64, 1-based
// 1-based triplets in any order; written canonical (row, then column)
void write(std::int64_t n, std::vector<std::int64_t> rows, std::vector<std::int64_t> cols,
           std::vector<double> vals, bool refuse_duplicates, const std::string& path);

}  // namespace spmvtk::mm
