// cxx_api.cpp -- host-side helpers of the C++ API (formats.hpp).
// Semantics of /root/reference/proj/src/formats.cpp:75-249.
#include <algorithm>
#include <numeric>
#include <string>
#include <unordered_set>

#include "spmvtk/error.hpp"
#include "spmvtk/formats.hpp"

namespace spmvtk {

std::vector<std::string> validate(const CrsMatrix& m) {
  std::vector<std::string> out;
  if (m.n < 0) out.push_back("negative dimension");
  if (m.values.size() != m.col_idx.size()) out.push_back("values / col_idx length mismatch");
  if (static_cast<index_t>(m.row_ptr.size()) != m.n + 1) {
    out.push_back("pointer array length " + std::to_string(m.row_ptr.size()) + ", expected " +
                  std::to_string(m.n + 1));
    return out;
  }
  if (m.row_ptr.front() != 1) out.push_back("row_ptr[1] != 1");
  if (m.row_ptr.back() != m.nnz() + 1)
    out.push_back("pointer array end " + std::to_string(m.row_ptr.back()) +
                  ", expected nnz+1 = " + std::to_string(m.nnz() + 1));
  for (std::size_t i = 1; i < m.row_ptr.size(); ++i)
    if (m.row_ptr[i] < m.row_ptr[i - 1]) {
      out.push_back("row_ptr not nondecreasing at position " + std::to_string(i + 1));
      break;
    }
  for (std::size_t p = 0; p < m.col_idx.size(); ++p)
    if (m.col_idx[p] < 1 || m.col_idx[p] > m.n)
      out.push_back("column index " + std::to_string(m.col_idx[p]) + " out of range at entry " +
                    std::to_string(p + 1));
  if (!out.empty()) return out;
  std::unordered_set<index_t> seen;
  for (index_t i = 1; i <= m.n; ++i) {
    seen.clear();
    for (index_t p = m.row_ptr[i - 1]; p < m.row_ptr[i]; ++p)
      if (!seen.insert(m.col_idx[p - 1]).second)
        out.push_back("duplicate index in row " + std::to_string(i) + " (index " +
                      std::to_string(m.col_idx[p - 1]) + ")");
  }
  return out;
}

RowHistogram row_histogram(const CrsMatrix& m) {
  RowHistogram h;
  h.counts.resize(static_cast<std::size_t>(m.n));
  for (index_t i = 0; i < m.n; ++i)
    h.counts[static_cast<std::size_t>(i)] = m.row_ptr[i + 1] - m.row_ptr[i];
  return h;
}

DenseMatrix dense_from_crs(const CrsMatrix& m) {
  if (m.n > kDenseOracleCap)
    throw Error(ErrorCode::InvalidArgument,
                "dense oracle capped at n = " + std::to_string(kDenseOracleCap));
  DenseMatrix d;
  d.n = m.n;
  d.entries.assign(static_cast<std::size_t>(m.n * m.n), 0.0);
  for (index_t i = 1; i <= m.n; ++i)
    for (index_t p = m.row_ptr[i - 1]; p < m.row_ptr[i]; ++p) d.at(i, m.col_idx[p - 1]) = m.values[p - 1];
  return d;
}

CrsMatrix canonicalize(const CrsMatrix& m) {
  CrsMatrix out = m;
  std::vector<std::size_t> idx;
  for (index_t i = 1; i <= m.n; ++i) {
    const std::size_t lo = static_cast<std::size_t>(m.row_ptr[i - 1] - 1);
    const std::size_t hi = static_cast<std::size_t>(m.row_ptr[i] - 1);
    idx.resize(hi - lo);
    std::iota(idx.begin(), idx.end(), lo);
    std::sort(idx.begin(), idx.end(),
              [&](std::size_t a, std::size_t b) { return m.col_idx[a] < m.col_idx[b]; });
    for (std::size_t k = 0; k < idx.size(); ++k) {
      out.col_idx[lo + k] = m.col_idx[idx[k]];
      out.values[lo + k] = m.values[idx[k]];
    }
  }
  return out;
}

bool structurally_equal(const CrsMatrix& a, const CrsMatrix& b) {
  return a.n == b.n && a.row_ptr == b.row_ptr && a.col_idx == b.col_idx && a.values == b.values;
}

}  // namespace spmvtk
