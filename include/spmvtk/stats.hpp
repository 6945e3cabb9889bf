// stats.hpp -- D_mat row statistics (drop-in for
// /root/reference/proj/include/spmvtk/stats.hpp:9-19).  row_stats reduces the
// row pointer array on the GPU; both compute exact integer moments and round
// once (agrees with the reference's Welford to <= 1e-12, exact on the
// reference's special cases).
#pragma once

#include "spmvtk/formats.hpp"

namespace spmvtk {

struct RowStats {
  double mu = 0.0;
  double sigma = 0.0;  // population standard deviation of row counts
  double d_mat = 0.0;  // sigma / mu
};

RowStats stats_from_histogram(const RowHistogram& h);
RowStats row_stats(const CrsMatrix& m);

}  // namespace spmvtk
