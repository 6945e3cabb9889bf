// mmio.cpp -- Matrix Market ingest / export (host side of the boundary).
//
// Behaviour of /root/reference/proj/src/ingest.cpp:95-232: coordinate real,
// general or symmetric (mirrored on read), square only, refusals name the
// offending line, duplicates refused, entries grouped by row in file order;
// the writer emits canonical (column-sorted) general format with %.17g.
#include "mmio.hpp"

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <fstream>
#include <numeric>
#include <sstream>

#include "spmvtk/error.hpp"

namespace spmvtk::mm {

namespace {
[[noreturn]] void fail(const std::string& path, long line, const std::string& what) {
  throw Error(ErrorCode::Parse, path + ":" + std::to_string(line) + ": " + what);
}
bool blank(const std::string& s) { return s.find_first_not_of(" \t\r") == std::string::npos; }
}  // namespace

gen::HostCrs read(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw Error(ErrorCode::Io, "cannot open " + path);
  long ln = 1;
  std::string line;
  if (!std::getline(in, line)) fail(path, ln, "empty file");
  std::string lowered = line;
  for (char& ch : lowered) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  std::istringstream hs(lowered);
  std::string banner, object, format, field, symmetry;
  hs >> banner >> object >> format >> field >> symmetry;
  if (banner != "%%matrixmarket" || object != "matrix") fail(path, ln, "not a Matrix Market file");
  if (format != "coordinate") fail(path, ln, "only coordinate format is supported");
  if (field != "real")
    fail(path, ln, "only real-valued matrices are supported (got \"" + field + "\")");
  const bool sym = symmetry == "symmetric";
  if (!sym && symmetry != "general") fail(path, ln, "unsupported symmetry kind \"" + symmetry + "\"");

  std::int64_t rows = 0, cols = 0;
  long long declared = 0;
  for (;;) {
    ++ln;
    if (!std::getline(in, line)) fail(path, ln, "missing size line");
    if ((!line.empty() && line[0] == '%') || blank(line)) continue;
    std::istringstream ss(line);
    if (!(ss >> rows >> cols >> declared)) fail(path, ln, "malformed size line");
    break;
  }
  if (rows != cols)
    fail(path, ln, "non-square matrix (" + std::to_string(rows) + " x " + std::to_string(cols) + ")");
  const std::int64_t n = rows;

  std::vector<std::int64_t> ri, ci;
  std::vector<double> vv;
  std::vector<long> at;
  for (long long seen = 0; seen < declared;) {
    ++ln;
    if (!std::getline(in, line))
      fail(path, ln, "unexpected end of file, expected " + std::to_string(declared) + " entries");
    if ((!line.empty() && line[0] == '%') || blank(line)) continue;
    std::istringstream es(line);
    std::int64_t i = 0, j = 0;
    double v = 0;
    if (!(es >> i >> j >> v)) fail(path, ln, "malformed entry line");
    if (i < 1 || i > n) fail(path, ln, "row index " + std::to_string(i) + " out of range");
    if (j < 1 || j > n) fail(path, ln, "column index " + std::to_string(j) + " out of range");
    ri.push_back(i);
    ci.push_back(j);
    vv.push_back(v);
    at.push_back(ln);
    if (sym && i != j) {
      ri.push_back(j);
      ci.push_back(i);
      vv.push_back(v);
      at.push_back(ln);
    }
    ++seen;
  }
  std::vector<std::size_t> ord(ri.size());
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](std::size_t a, std::size_t b) {
    return ri[a] != ri[b] ? ri[a] < ri[b] : ci[a] < ci[b];
  });
  for (std::size_t k = 1; k < ord.size(); ++k) {
    std::size_t a = ord[k - 1], b = ord[k];
    if (ri[a] == ri[b] && ci[a] == ci[b])
      fail(path, std::max(at[a], at[b]),
           "duplicate entry (" + std::to_string(ri[a]) + ", " + std::to_string(ci[a]) + ")");
  }
  // group by row, file order within a row (stable counting placement)
  gen::HostCrs m;
  m.n = n;
  m.base = 1;
  m.row_ptr.assign(static_cast<std::size_t>(n) + 1, 0);
  m.row_ptr[0] = 1;
  for (std::int64_t r : ri) ++m.row_ptr[static_cast<std::size_t>(r)];
  for (std::int64_t i = 1; i <= n; ++i)
    m.row_ptr[static_cast<std::size_t>(i)] += m.row_ptr[static_cast<std::size_t>(i - 1)];
  m.values.resize(vv.size());
  m.col_idx.resize(vv.size());
  std::vector<std::int64_t> next(m.row_ptr.begin(), m.row_ptr.end() - 1);
  for (std::size_t p = 0; p < ri.size(); ++p) {
    std::int64_t slot = next[static_cast<std::size_t>(ri[p] - 1)]++;
    m.values[static_cast<std::size_t>(slot - 1)] = vv[p];
    m.col_idx[static_cast<std::size_t>(slot - 1)] = ci[p];
  }
  return m;
}

void write(std::int64_t n, std::vector<std::int64_t> rows, std::vector<std::int64_t> cols,
           std::vector<double> vals, bool refuse_duplicates, const std::string& path) {
  std::vector<std::size_t> ord(vals.size());
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](std::size_t a, std::size_t b) {
    return rows[a] != rows[b] ? rows[a] < rows[b] : cols[a] < cols[b];
  });
  if (refuse_duplicates)
    for (std::size_t k = 1; k < ord.size(); ++k) {
      std::size_t a = ord[k - 1], b = ord[k];
      if (rows[a] == rows[b] && cols[a] == cols[b])
        throw Error(ErrorCode::Validation, "duplicate (row, col) pair (" + std::to_string(rows[a]) +
                                               ", " + std::to_string(cols[a]) + ")");
    }
  std::ofstream out(path);
  if (!out) throw Error(ErrorCode::Io, "cannot open " + path + " for writing");
  out << "%%MatrixMarket matrix coordinate real general\n";
  out << n << ' ' << n << ' ' << vals.size() << '\n';
  char buf[96];
  for (std::size_t k : ord) {
    std::snprintf(buf, sizeof(buf), "%lld %lld %.17g\n", static_cast<long long>(rows[k]),
                  static_cast<long long>(cols[k]), vals[k]);
    out << buf;
  }
  if (!out) throw Error(ErrorCode::Io, "write failed: " + path);
}

}  // namespace spmvtk::mm
