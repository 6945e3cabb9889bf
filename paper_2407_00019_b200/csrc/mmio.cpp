// mmio.cpp -- Matrix Market ingest / export (host side of the boundary).
//
// Behaviour of /root/reference/proj/src/ingest.cpp:95-232: coordinate real,
// general or symmetric (mirrored on read), square only, refusals name the
// offending line, duplicates refused, entries grouped by row in file order;
// the writer emits canonical (column-sorted) general format with %.17g.
//
// Unlike the reference (one istringstream per line, one global sort), the
// file is read whole and parsed by all host threads: the entry region is cut
// at line boundaries, every thread parses its lines with std::from_chars
// (lines outside the plain "int int number" grammar fall back to the
// reference's istringstream extraction, so odd tokens parse identically),
// the first error in FILE order wins, and duplicates are found per row after
// grouping.  The writer formats row ranges in parallel.
#include "mmio.hpp"

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>
#include <thread>

#include "spmvtk/error.hpp"

namespace spmvtk::mm {

namespace {
[[noreturn]] void fail(const std::string& path, long line, const std::string& what) {
  throw Error(ErrorCode::Parse, path + ":" + std::to_string(line) + ": " + what);
}
bool blank(const char* b, const char* e) {
  for (; b < e; ++b)
    if (*b != ' ' && *b != '\t' && *b != '\r') return false;
  return true;
}
unsigned threads_for(std::size_t work) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  return static_cast<unsigned>(std::max<std::size_t>(1, std::min<std::size_t>(hw, work / 65536 + 1)));
}

// one entry line: "i j v" with optional surrounding blanks.  Returns 0 on
// success, 1 malformed; the fast path accepts [-]digits for the indices and
// [-](digits[.digits]|.digits)([eE][+-]digits)? for the value followed by a
// blank or the line end -- anything else goes through istringstream exactly
// as the reference extracts it.
bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }

int parse_entry(const char* b, const char* e, std::int64_t& i, std::int64_t& j, double& v) {
  const char* p = b;
  auto skip = [&] {
    while (p < e && is_ws(*p)) ++p;
  };
  auto fast_int = [&](std::int64_t& out) -> bool {
    skip();
    const char* s = p;
    if (p < e && *p == '-') ++p;
    const char* d = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    if (p == d || p - d > 18 || (p < e && !is_ws(*p))) return false;
    return std::from_chars(s, p, out).ec == std::errc();
  };
  auto fast_real = [&](double& out) -> bool {
    skip();
    const char* s = p;
    if (p < e && *p == '-') ++p;
    const char* d = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    bool digits = p > d;
    if (p < e && *p == '.') {
      ++p;
      const char* f = p;
      while (p < e && *p >= '0' && *p <= '9') ++p;
      digits = digits || p > f;
    }
    if (!digits) return false;
    if (p < e && (*p == 'e' || *p == 'E')) {
      ++p;
      if (p < e && (*p == '+' || *p == '-')) ++p;
      const char* x = p;
      while (p < e && *p >= '0' && *p <= '9') ++p;
      if (p == x) return false;
    }
    if (p < e && !is_ws(*p)) return false;
    return std::from_chars(s, p, out).ec == std::errc();
  };
  if (fast_int(i) && fast_int(j) && fast_real(v)) return 0;
  // the reference's extraction, byte for byte
  std::istringstream es(std::string(b, e));
  i = j = 0;
  v = 0.0;
  return (es >> i >> j >> v) ? 0 : 1;
}

struct Chunk {
  // parsed entries of one slice of the entry region, in file order
  std::vector<std::int64_t> ri, ci;
  std::vector<double> vv;
  std::vector<long> at;       // local line index (0-based within the chunk)
  long lines = 0;             // lines in the chunk
  long err_line = -1;         // local index of the first bad line
  std::string err;
  std::int64_t entries = 0;   // file entries seen (before mirroring)
};
}  // namespace

gen::HostCrs read(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error(ErrorCode::Io, "cannot open " + path);
  std::string buf((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  const char* const begin = buf.data();
  const char* const end = begin + buf.size();
  // line iterator with std::getline semantics (no empty line after a final '\n')
  const char* cur = begin;
  auto next_line = [&](const char*& lb, const char*& le) -> bool {
    if (cur >= end) return false;
    lb = cur;
    const char* nl = static_cast<const char*>(std::memchr(cur, '\n', end - cur));
    le = nl ? nl : end;
    cur = nl ? nl + 1 : end;
    return true;
  };

  long ln = 1;
  const char *lb, *le;
  if (!next_line(lb, le)) fail(path, ln, "empty file");
  std::string lowered(lb, le);
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
    if (!next_line(lb, le)) fail(path, ln, "missing size line");
    if ((lb < le && lb[0] == '%') || blank(lb, le)) continue;
    std::istringstream ss(std::string(lb, le));
    if (!(ss >> rows >> cols >> declared)) fail(path, ln, "malformed size line");
    break;
  }
  if (rows != cols)
    fail(path, ln, "non-square matrix (" + std::to_string(rows) + " x " + std::to_string(cols) + ")");
  const std::int64_t n = rows;
  const long header_lines = ln;  // the entry region starts at line header_lines + 1

  // cut the entry region at line starts, one slice per thread
  const std::size_t region = static_cast<std::size_t>(end - cur);
  const unsigned T = threads_for(region / 16);
  std::vector<const char*> cut(T + 1);
  cut[0] = cur;
  cut[T] = end;
  for (unsigned t = 1; t < T; ++t) {
    const char* p = cur + region * t / T;
    if (p < cut[t - 1]) p = cut[t - 1];
    const char* nl = p < end ? static_cast<const char*>(std::memchr(p, '\n', end - p)) : nullptr;
    cut[t] = nl ? nl + 1 : end;
  }
  std::vector<Chunk> chunks(T);
  auto parse_chunk = [&](unsigned t) {
    Chunk& c = chunks[t];
    const char* p = cut[t];
    const char* stop = cut[t + 1];
    const std::size_t guess = static_cast<std::size_t>(stop - p) / 24 + 16;
    c.ri.reserve(sym ? 2 * guess : guess);
    c.ci.reserve(sym ? 2 * guess : guess);
    c.vv.reserve(sym ? 2 * guess : guess);
    c.at.reserve(sym ? 2 * guess : guess);
    while (p < stop) {
      const char* b = p;
      const char* nl = static_cast<const char*>(std::memchr(p, '\n', stop - p));
      const char* e = nl ? nl : stop;
      p = nl ? nl + 1 : stop;
      const long idx = c.lines++;
      if ((b < e && b[0] == '%') || blank(b, e)) continue;
      std::int64_t i = 0, j = 0;
      double v = 0.0;
      ++c.entries;
      if (parse_entry(b, e, i, j, v)) {
        c.err_line = idx;
        c.err = "malformed entry line";
        return;
      }
      if (i < 1 || i > n) {
        c.err_line = idx;
        c.err = "row index " + std::to_string(i) + " out of range";
        return;
      }
      if (j < 1 || j > n) {
        c.err_line = idx;
        c.err = "column index " + std::to_string(j) + " out of range";
        return;
      }
      c.ri.push_back(i);
      c.ci.push_back(j);
      c.vv.push_back(v);
      c.at.push_back(idx);
      if (sym && i != j) {
        c.ri.push_back(j);
        c.ci.push_back(i);
        c.vv.push_back(v);
        c.at.push_back(idx);
      }
    }
  };
  {
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < T; ++t) pool.emplace_back(parse_chunk, t);
    parse_chunk(0);
    for (auto& th : pool) th.join();
  }

  // walk the chunks in file order: the reference stops after `declared`
  // entries, so neither errors nor entries past that point count
  std::vector<std::size_t> keep(T, 0);  // entries (post-mirroring) kept per chunk
  std::vector<long> base_line(T, 0);
  long long seen = 0;
  long lines_before = header_lines;
  unsigned last = T;
  for (unsigned t = 0; t < T && seen < declared; ++t) {
    Chunk& c = chunks[t];
    base_line[t] = lines_before;
    // entries of this chunk, in order, until `declared` is reached or its error
    std::size_t k = 0;
    long long taken = 0;
    while (k < c.ri.size() && seen + taken < declared) {
      const long line = c.at[k];
      std::size_t m = k + 1;
      while (m < c.ri.size() && c.at[m] == line) ++m;  // mirrored twin
      ++taken;
      k = m;
    }
    const long long errors_before = c.err_line >= 0 ? 1 : 0;
    if (seen + taken < declared && errors_before) {
      fail(path, lines_before + 1 + c.err_line, c.err);
    }
    keep[t] = k;
    seen += taken;
    lines_before += c.lines;
    last = t;
  }
  if (seen < declared)
    fail(path, lines_before + 1,
         "unexpected end of file, expected " + std::to_string(declared) + " entries");
  (void)last;

  // group by row, file order within a row (stable counting placement)
  std::size_t total = 0;
  for (unsigned t = 0; t < T; ++t) total += keep[t];
  gen::HostCrs m;
  m.n = n;
  m.base = 1;
  m.row_ptr.assign(static_cast<std::size_t>(n) + 1, 0);
  m.row_ptr[0] = 1;
  for (unsigned t = 0; t < T; ++t)
    for (std::size_t k = 0; k < keep[t]; ++k) ++m.row_ptr[static_cast<std::size_t>(chunks[t].ri[k])];
  for (std::int64_t i = 1; i <= n; ++i)
    m.row_ptr[static_cast<std::size_t>(i)] += m.row_ptr[static_cast<std::size_t>(i - 1)];
  m.values.resize(total);
  m.col_idx.resize(total);
  std::vector<long> line_of(total);
  {
    std::vector<std::int64_t> next(m.row_ptr.begin(), m.row_ptr.end() - 1);
    for (unsigned t = 0; t < T; ++t) {
      const Chunk& c = chunks[t];
      for (std::size_t k = 0; k < keep[t]; ++k) {
        const std::size_t slot = static_cast<std::size_t>(next[static_cast<std::size_t>(c.ri[k] - 1)]++ - 1);
        m.values[slot] = c.vv[k];
        m.col_idx[slot] = c.ci[k];
        line_of[slot] = base_line[t] + 1 + c.at[k];
      }
    }
  }
  chunks.clear();

  // duplicates: per row, the smallest repeated column; the first such row
  // (row-major order, as the reference's sorted scan finds it) is reported
  // with the later of the two lines
  {
    const unsigned TT = threads_for(total);
    std::vector<std::int64_t> dup_row(TT, -1), dup_col(TT, 0);
    std::vector<long> dup_line(TT, 0);
    auto scan = [&](unsigned t) {
      const std::int64_t r0 = n * t / TT, r1 = n * (t + 1) / TT;
      std::vector<std::pair<std::int64_t, long>> row;
      for (std::int64_t r = r0; r < r1; ++r) {
        const std::size_t a = static_cast<std::size_t>(m.row_ptr[r] - 1);
        const std::size_t b = static_cast<std::size_t>(m.row_ptr[r + 1] - 1);
        if (b - a < 2) continue;
        row.clear();
        for (std::size_t p = a; p < b; ++p) row.emplace_back(m.col_idx[p], line_of[p]);
        std::sort(row.begin(), row.end());
        for (std::size_t k = 1; k < row.size(); ++k)
          if (row[k].first == row[k - 1].first) {
            dup_row[t] = r + 1;
            dup_col[t] = row[k].first;
            dup_line[t] = std::max(row[k].second, row[k - 1].second);
            return;
          }
      }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < TT; ++t) pool.emplace_back(scan, t);
    scan(0);
    for (auto& th : pool) th.join();
    for (unsigned t = 0; t < TT; ++t)
      if (dup_row[t] >= 0)
        fail(path, dup_line[t],
             "duplicate entry (" + std::to_string(dup_row[t]) + ", " + std::to_string(dup_col[t]) +
                 ")");
  }
  return m;
}

void write(std::int64_t n, std::vector<std::int64_t> rows, std::vector<std::int64_t> cols,
           std::vector<double> vals, bool refuse_duplicates, const std::string& path) {
  // group by row (stable), then sort each row by column in parallel
  const std::size_t nnz = vals.size();
  std::vector<std::int64_t> ptr(static_cast<std::size_t>(n) + 1, 0);
  for (std::int64_t r : rows) ++ptr[static_cast<std::size_t>(r)];
  for (std::int64_t i = 1; i <= n; ++i) ptr[static_cast<std::size_t>(i)] += ptr[static_cast<std::size_t>(i - 1)];
  std::vector<std::size_t> ord(nnz);
  {
    std::vector<std::int64_t> next(ptr.begin(), ptr.end() - 1);
    for (std::size_t k = 0; k < nnz; ++k) ord[static_cast<std::size_t>(next[static_cast<std::size_t>(rows[k] - 1)]++)] = k;
  }
  const unsigned T = threads_for(nnz);
  std::vector<std::string> text(T);
  std::vector<std::int64_t> dup_row(T, -1), dup_col(T, 0);
  auto work = [&](unsigned t) {
    const std::int64_t r0 = n * t / T, r1 = n * (t + 1) / T;
    std::string& out = text[t];
    out.reserve(static_cast<std::size_t>(ptr[static_cast<std::size_t>(r1)] - ptr[static_cast<std::size_t>(r0)]) * 32);
    char buf[96];
    for (std::int64_t r = r0; r < r1; ++r) {
      auto b = ord.begin() + ptr[static_cast<std::size_t>(r)];
      auto e = ord.begin() + ptr[static_cast<std::size_t>(r) + 1];
      std::stable_sort(b, e, [&](std::size_t x, std::size_t y) { return cols[x] < cols[y]; });
      for (auto it = b; it != e; ++it) {
        if (refuse_duplicates && it != b && cols[*it] == cols[*(it - 1)] && dup_row[t] < 0) {
          dup_row[t] = r + 1;
          dup_col[t] = cols[*it];
        }
        const int len = std::snprintf(buf, sizeof(buf), "%lld %lld %.17g\n",
                                      static_cast<long long>(r + 1),
                                      static_cast<long long>(cols[*it]), vals[*it]);
        out.append(buf, static_cast<std::size_t>(len));
      }
    }
  };
  {
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < T; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
  }
  for (unsigned t = 0; t < T; ++t)
    if (dup_row[t] >= 0)
      throw Error(ErrorCode::Validation, "duplicate (row, col) pair (" + std::to_string(dup_row[t]) +
                                             ", " + std::to_string(dup_col[t]) + ")");
  std::ofstream out(path, std::ios::binary);
  if (!out) throw Error(ErrorCode::Io, "cannot open " + path + " for writing");
  out << "%%MatrixMarket matrix coordinate real general\n";
  out << n << ' ' << n << ' ' << nnz << '\n';
  for (const std::string& s : text) out.write(s.data(), static_cast<std::streamsize>(s.size()));
  if (!out) throw Error(ErrorCode::Io, "write failed: " + path);
}

}  // namespace spmvtk::mm
