// cxx_api.cpp -- the reference's C++ entry points, B200-backed.
//
// Drop-in for /root/reference/proj/include/spmvtk/{formats,convert,spmv,
// stats,autotune,ingest}.hpp: same names, signatures, value semantics
// (inputs const&, fresh results returned) and error codes / message
// substrings.  The work runs on the GPU: arguments are uploaded into device
// handles (int64 1-based -> int32 0-based on the device), the sm_100a kernels
// run, results are copied back into the reference's host types.  Host-only
// helpers (validate, canonicalize, the dense oracle, the inverse conversions)
// keep the reference's semantics (formats.cpp:75-249, convert.cpp:117-183).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <fstream>
#include <functional>
#include <iterator>
#include <memory>
#include <numeric>
#include <string>
#include <unordered_set>

#include "autotune.hpp"
#include "generators.hpp"
#include "matrix.hpp"
#include "mmio.hpp"
#include "runtime.hpp"
#include "spmvtk/autotune.hpp"
#include "spmvtk/convert.hpp"
#include "spmvtk/error.hpp"
#include "spmvtk/formats.hpp"
#include "spmvtk/ingest.hpp"
#include "spmvtk/spmv.hpp"
#include "spmvtk/spmvtk_kernels.h"
#include "spmvtk/stats.hpp"
#include "validate.hpp"

namespace spmvtk {

namespace {

using Handle = std::unique_ptr<dev::Matrix>;

Handle up(const CrsMatrix& m) {
  return Handle(dev::crs_from_arrays(m.n, m.nnz(), m.row_ptr.data(), m.col_idx.data(),
                                     m.values.data(), 8, 1, false));
}

Handle up(const CooMatrix& m) {
  if (m.ordering == CooOrdering::Unordered)
    throw Error(ErrorCode::InvalidArgument, "COO kernels require an ordered COO matrix");
  return Handle(dev::coo_from_arrays(m.n, m.nnz(), m.row_idx.data(), m.col_idx.data(),
                                     m.values.data(), 8, 1,
                                     m.ordering == CooOrdering::RowMajor ? 0 : 1));
}

Handle up(const EllMatrix& m) {
  return Handle(dev::ell_from_arrays(m.n, m.band_count, m.col_idx.data(), m.values.data(),
                                     m.row_entry_count.data(), m.stored_nnz));
}

std::vector<index_t> idx_of(const dev::Matrix& h, spmvtk_array a, int base = 1) {
  std::vector<index_t> out(static_cast<std::size_t>(dev::copy_array(h, a, nullptr, 0, 8, base)));
  dev::copy_array(h, a, out.data(), static_cast<std::int64_t>(out.size()), 8, base);
  return out;
}

std::vector<double> vals_of(const dev::Matrix& h) {
  std::vector<double> out(
      static_cast<std::size_t>(dev::copy_array(h, SPMVTK_ARRAY_VALUES, nullptr, 0, 8, 0)));
  dev::copy_array(h, SPMVTK_ARRAY_VALUES, out.data(), static_cast<std::int64_t>(out.size()), 8, 0);
  return out;
}

EllMatrix down_ell(const dev::Matrix& h) {
  EllMatrix e;
  e.n = h.n;
  e.band_count = h.band_count;
  e.stored_nnz = h.nnz;
  e.values = vals_of(h);
  e.col_idx = idx_of(h, SPMVTK_ARRAY_COL_IDX);
  e.row_entry_count = idx_of(h, SPMVTK_ARRAY_ROW_ENTRY_COUNT, 0);
  return e;
}

CrsMatrix down_crs(const dev::Matrix& h) {
  CrsMatrix out;
  out.n = h.n;
  out.values = vals_of(h);
  out.col_idx = idx_of(h, SPMVTK_ARRAY_COL_IDX);
  out.row_ptr = idx_of(h, SPMVTK_ARRAY_POINTER);
  return out;
}

void require_dim(index_t n, std::size_t len) {
  if (static_cast<index_t>(len) != n)
    throw Error(ErrorCode::InvalidArgument, "vector length " + std::to_string(len) +
                                                " does not match matrix dimension " +
                                                std::to_string(n));
}

void require_lanes(int lanes) {
  if (lanes < 1) throw Error(ErrorCode::InvalidArgument, "lane count must be at least 1");
}

std::vector<double> run(const dev::Matrix& h, spmvtk_kernel k, std::span<const double> x) {
  const std::size_t n = static_cast<std::size_t>(h.n);
  std::vector<double> y(n);
  rt::DevArray<double> dx(std::max<std::size_t>(x.size(), 1), "x");
  rt::DevArray<double> dy(std::max<std::size_t>(n, 1), "y");
  rt::copy_to_device(dx.get(), x.data(), x.size() * sizeof(double));
  dev::spmv_device(h, k, dx.get(), dy.get());
  rt::copy_to_host(y.data(), dy.get(), n * sizeof(double));
  return y;
}

spmvtk_kernel to_c(Kernel k) { return static_cast<spmvtk_kernel>(static_cast<int>(k)); }

RowStats stats_of(const rt::Moments& mo, index_t n) {
  rt::RowStatsD s = rt::stats_from_moments(mo, n);
  return RowStats{s.mu, s.sigma, s.d_mat};
}

CrsMatrix canonical_from_triplets(index_t n, std::vector<index_t> rows, std::vector<index_t> cols,
                                  std::vector<double> vals) {
  std::vector<std::size_t> ord(vals.size());
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](std::size_t a, std::size_t b) {
    return rows[a] != rows[b] ? rows[a] < rows[b] : cols[a] < cols[b];
  });
  for (std::size_t k = 1; k < ord.size(); ++k)
    if (rows[ord[k]] == rows[ord[k - 1]] && cols[ord[k]] == cols[ord[k - 1]])
      throw Error(ErrorCode::Validation, "duplicate (row, col) pair (" +
                                             std::to_string(rows[ord[k]]) + ", " +
                                             std::to_string(cols[ord[k]]) + ")");
  CrsMatrix out;
  out.n = n;
  out.row_ptr.assign(static_cast<std::size_t>(n) + 1, 0);
  out.row_ptr[0] = 1;
  for (index_t r : rows) ++out.row_ptr[static_cast<std::size_t>(r)];
  for (index_t i = 1; i <= n; ++i) out.row_ptr[i] += out.row_ptr[i - 1];
  out.values.reserve(vals.size());
  out.col_idx.reserve(vals.size());
  for (std::size_t k : ord) {
    out.values.push_back(vals[k]);
    out.col_idx.push_back(cols[k]);
  }
  return out;
}

}  // namespace

// ---------------------------------------------------------------- formats
// The structural rules and messages are the reference's (formats.cpp:75-182);
// the O(nnz) checks run on the GPU (kernels_validate.cu).
std::vector<std::string> validate(const CrsMatrix& m) {
  return dev::validate_segments(m.n, m.row_ptr, m.col_idx, m.values.size(), "row_ptr", "col_idx",
                                "column", "row");
}

std::vector<std::string> validate(const CcsMatrix& m) {
  return dev::validate_segments(m.n, m.col_ptr, m.row_idx, m.values.size(), "col_ptr", "row_idx",
                                "row", "column");
}

std::vector<std::string> validate(const CooMatrix& m) {
  const int ordering = m.ordering == CooOrdering::RowMajor   ? 0
                       : m.ordering == CooOrdering::ColMajor ? 1
                                                             : 2;
  return dev::validate_triplets(m.n, m.row_idx, m.col_idx, m.values.size(), ordering);
}

std::vector<std::string> validate(const EllMatrix& m) {
  return dev::validate_ell(m.n, m.band_count, m.values, m.col_idx, m.row_entry_count,
                           m.stored_nnz);
}

RowHistogram row_histogram(const CrsMatrix& m) {
  // counts[i] = row_ptr[i+1] - row_ptr[i] (formats.cpp:184-192)
  RowHistogram h;
  h.counts.resize(static_cast<std::size_t>(std::max<index_t>(m.n, 0)));
  if (m.n > 0)
    std::transform(m.row_ptr.begin() + 1, m.row_ptr.begin() + 1 + m.n, m.row_ptr.begin(),
                   h.counts.begin(), std::minus<index_t>());
  return h;
}

namespace {
void dense_cap(index_t n) {
  if (n > kDenseOracleCap)
    throw Error(ErrorCode::InvalidArgument,
                "dense oracle capped at n = " + std::to_string(kDenseOracleCap));
}
}  // namespace

DenseMatrix dense_from_crs(const CrsMatrix& m) {
  dense_cap(m.n);
  DenseMatrix d;
  d.n = m.n;
  d.entries.assign(static_cast<std::size_t>(m.n * m.n), 0.0);
  // entries in storage order; the row advances past every segment end
  index_t row = 1;
  for (index_t p = 1; p <= m.nnz(); ++p) {
    while (m.row_ptr[static_cast<std::size_t>(row)] <= p) ++row;
    d.at(row, m.col_idx[static_cast<std::size_t>(p - 1)]) = m.values[static_cast<std::size_t>(p - 1)];
  }
  return d;
}

CrsMatrix crs_from_dense(const DenseMatrix& d, double drop_tol) {
  dense_cap(d.n);
  CrsMatrix m;
  m.n = d.n;
  m.row_ptr.assign(static_cast<std::size_t>(d.n) + 1, 1);
  for (index_t i = 0; i < d.n; ++i) {
    const double* rowv = d.entries.data() + static_cast<std::size_t>(i * d.n);
    for (index_t j = 0; j < d.n; ++j)
      if (std::abs(rowv[j]) > drop_tol) {
        m.col_idx.push_back(j + 1);
        m.values.push_back(rowv[j]);
      }
    m.row_ptr[static_cast<std::size_t>(i) + 1] = static_cast<index_t>(m.values.size()) + 1;
  }
  return m;
}

CrsMatrix canonicalize(const CrsMatrix& m) {
  if (m.n > 0 && m.nnz() > 0) {  // per-row sort on the device
    Handle h = up(m);
    Handle c(dev::to_crs(*h));
    return down_crs(*c);
  }
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

// ---------------------------------------------------------------- convert
CooMatrix crs_to_coo_row(const CrsMatrix& m) {
  Handle h = up(m);
  Handle c(dev::convert(*h, SPMVTK_FORMAT_COO_ROW, 0));
  CooMatrix out;
  out.n = m.n;
  out.ordering = CooOrdering::RowMajor;
  out.values = vals_of(*c);
  out.row_idx = idx_of(*c, SPMVTK_ARRAY_ROW_IDX);
  out.col_idx = idx_of(*c, SPMVTK_ARRAY_COL_IDX);
  return out;
}

CcsMatrix crs_to_ccs(const CrsMatrix& m) {
  Handle h = up(m);
  Handle c(dev::convert(*h, SPMVTK_FORMAT_CCS, 0));
  CcsMatrix out;
  out.n = m.n;
  out.values = vals_of(*c);
  out.row_idx = idx_of(*c, SPMVTK_ARRAY_ROW_IDX);
  out.col_ptr = idx_of(*c, SPMVTK_ARRAY_POINTER);
  return out;
}

CooMatrix ccs_to_coo_col(const CcsMatrix& m) {
  // convert.cpp:55-66: copy values / row_idx, expand col_ptr on the GPU
  Handle h(dev::crs_from_arrays(m.n, m.nnz(), m.col_ptr.data(), m.row_idx.data(),
                                m.values.data(), 8, 1, false));
  Handle c(dev::convert(*h, SPMVTK_FORMAT_COO_ROW, 0));  // segments = columns here
  CooMatrix out;
  out.n = m.n;
  out.ordering = CooOrdering::ColMajor;
  out.values = vals_of(*c);
  out.row_idx = idx_of(*c, SPMVTK_ARRAY_COL_IDX);
  out.col_idx = idx_of(*c, SPMVTK_ARRAY_ROW_IDX);
  return out;
}

CooMatrix crs_to_coo_col(const CrsMatrix& m) {
  Handle h = up(m);
  Handle c(dev::convert(*h, SPMVTK_FORMAT_COO_COL, 0));
  CooMatrix out;
  out.n = m.n;
  out.ordering = CooOrdering::ColMajor;
  out.values = vals_of(*c);
  out.row_idx = idx_of(*c, SPMVTK_ARRAY_ROW_IDX);
  out.col_idx = idx_of(*c, SPMVTK_ARRAY_COL_IDX);
  return out;
}

std::uint64_t estimate_ell_bytes(const CrsMatrix& m, int value_bytes, int index_bytes) {
  index_t max_row = 0;
  for (index_t i = 1; i <= m.n; ++i) max_row = std::max(max_row, m.row_ptr[i] - m.row_ptr[i - 1]);
  return static_cast<std::uint64_t>(m.n) * static_cast<std::uint64_t>(max_row) *
         static_cast<std::uint64_t>(value_bytes + index_bytes);
}

EllMatrix crs_to_ell(const CrsMatrix& m, std::uint64_t max_bytes) {
  if (max_bytes != kNoByteLimit) {  // refuse before touching the device
    const std::uint64_t est = estimate_ell_bytes(m);
    if (est > max_bytes)
      throw Error(ErrorCode::MemoryLimit, "ELL footprint estimate " + std::to_string(est) +
                                              " bytes exceeds limit " + std::to_string(max_bytes));
  }
  Handle h = up(m);
  Handle e(dev::convert(*h, SPMVTK_FORMAT_ELL, 0));
  return down_ell(*e);
}

// convert.cpp:158-164 -- on the device: row histogram, scan, cursor scatter,
// per-row sort on the column, duplicate refusal
CrsMatrix coo_to_crs(const CooMatrix& m) {
  if (m.n <= 0) return canonical_from_triplets(m.n, m.row_idx, m.col_idx, m.values);
  Handle h(dev::coo_from_arrays(m.n, m.nnz(), m.row_idx.data(), m.col_idx.data(),
                                m.values.data(), 8, 1,
                                m.ordering == CooOrdering::ColMajor ? 1 : 0));
  Handle c(dev::to_crs(*h));
  return down_crs(*c);
}

// convert.cpp:166-183 -- padding dropped by row_entry_count, on the device
CrsMatrix ell_to_crs(const EllMatrix& m) {
  if (m.n <= 0) return canonical_from_triplets(m.n, {}, {}, {});
  Handle h = up(m);
  Handle c(dev::to_crs(*h));
  return down_crs(*c);
}

// ---------------------------------------------------------------- spmv
ThreadPartition partition_range(index_t range_len, int lanes) {
  require_lanes(lanes);
  ThreadPartition p;
  p.lanes = lanes;
  p.range_len = range_len;
  const index_t base = range_len / lanes, rem = range_len % lanes;
  index_t pos = 1;
  for (int k = 0; k < lanes; ++k) {
    const index_t size = base + (k < rem ? 1 : 0);
    p.istart.push_back(pos);
    p.iend.push_back(pos + size - 1);
    pos += size;
  }
  return p;
}

std::vector<double> reduce_partials(const PartialResults& pr) {
  std::vector<double> y(static_cast<std::size_t>(pr.n), 0.0);
  for (int k = 0; k < pr.lanes; ++k)
    for (index_t i = 1; i <= pr.n; ++i) y[i - 1] += pr.at(i, k);
  return y;
}

std::vector<double> spmv_crs(const CrsMatrix& m, std::span<const double> x) {
  require_dim(m.n, x.size());
  return run(*up(m), SPMVTK_KERNEL_CRS, x);
}

std::vector<double> spmv_coo_col_outer(const CooMatrix& m, std::span<const double> x, int lanes) {
  if (m.ordering != CooOrdering::ColMajor)
    throw Error(ErrorCode::InvalidArgument,
                "spmv_coo_col_outer requires the matching COO ordering");
  require_dim(m.n, x.size());
  require_lanes(lanes);
  return run(*up(m), SPMVTK_KERNEL_COO_COL_OUTER, x);
}

std::vector<double> spmv_coo_row_outer(const CooMatrix& m, std::span<const double> x, int lanes) {
  if (m.ordering != CooOrdering::RowMajor)
    throw Error(ErrorCode::InvalidArgument,
                "spmv_coo_row_outer requires the matching COO ordering");
  require_dim(m.n, x.size());
  require_lanes(lanes);
  return run(*up(m), SPMVTK_KERNEL_COO_ROW_OUTER, x);
}

std::vector<double> spmv_ell_inner(const EllMatrix& m, std::span<const double> x, int lanes) {
  require_dim(m.n, x.size());
  require_lanes(lanes);
  return run(*up(m), SPMVTK_KERNEL_ELL_INNER, x);
}

std::vector<double> spmv_ell_outer(const EllMatrix& m, std::span<const double> x, int lanes) {
  require_dim(m.n, x.size());
  require_lanes(lanes);
  return run(*up(m), SPMVTK_KERNEL_ELL_OUTER, x);
}

// ---------------------------------------------------------------- stats
RowStats stats_from_histogram(const RowHistogram& h) {
  if (h.counts.empty()) throw Error(ErrorCode::InvalidArgument, "empty histogram");
  rt::Moments mo;
  for (index_t c : h.counts) {
    const std::uint64_t u = static_cast<std::uint64_t>(std::max<index_t>(c, 0));
    mo.max = std::max(mo.max, u);
    mo.sum += u;
    mo.sumsq += u * u;
  }
  return stats_of(mo, static_cast<index_t>(h.counts.size()));
}

RowStats row_stats(const CrsMatrix& m) {
  if (m.nnz() == 0)
    throw Error(ErrorCode::InvalidArgument,
                "row statistics undefined for an empty matrix (mu = 0)");
  rt::init();
  // only the pointer array goes to the device
  rt::DevArray<std::int64_t> wide(m.row_ptr.size(), "row_ptr upload");
  rt::DevArray<std::int32_t> ptr(m.row_ptr.size(), "row_ptr upload");
  rt::copy_to_device(wide.get(), m.row_ptr.data(), m.row_ptr.size() * 8);
  rt::check_launch(spmvtk_k_narrow_index(wide.get(), ptr.get(),
                                         static_cast<std::int64_t>(m.row_ptr.size()), 1,
                                         rt::stream()),
                   "row_ptr upload");
  return stats_of(rt::row_moments(ptr.get(), m.n), m.n);
}

// ---------------------------------------------------------------- autotune
std::string kernel_name(Kernel k) { return at::kernel_name(to_c(k)); }

Kernel kernel_from_name(const std::string& name) {
  spmvtk_kernel k = at::kernel_from_name(name);
  if (k == SPMVTK_KERNEL_ELL_ROWMAJOR)
    throw Error(ErrorCode::InvalidArgument, "unknown kernel name: " + name);
  return static_cast<Kernel>(static_cast<int>(k));
}

CostMetrics compute_metrics(const Timings& t) {
  at::Metrics m = at::compute_metrics(at::Timings{t.t_crs, t.t_ell, t.t_trans});
  return CostMetrics{m.sp, m.tt, m.r};
}

std::optional<std::int64_t> amortization_iterations(const Timings& t) {
  return at::amortization(at::Timings{t.t_crs, t.t_ell, t.t_trans});
}

double measure_spmv(Kernel kernel, MatrixRef m, std::span<const double> x, int lanes,
                    int repeats) {
  if (repeats < 1) throw Error(ErrorCode::InvalidArgument, "repeats must be at least 1");
  Handle h;
  bool ok = false;
  switch (kernel) {
    case Kernel::Crs:
      if (auto* p = std::get_if<const CrsMatrix*>(&m)) {
        require_dim((*p)->n, x.size());
        h = up(**p);
        ok = true;
      }
      break;
    case Kernel::CooRowOuter:
    case Kernel::CooColOuter:
      if (auto* p = std::get_if<const CooMatrix*>(&m)) {
        const CooOrdering want =
            kernel == Kernel::CooRowOuter ? CooOrdering::RowMajor : CooOrdering::ColMajor;
        if ((*p)->ordering != want)
          throw Error(ErrorCode::InvalidArgument,
                      std::string(kernel == Kernel::CooRowOuter ? "spmv_coo_row_outer"
                                                                : "spmv_coo_col_outer") +
                          " requires the matching COO ordering");
        require_dim((*p)->n, x.size());
        require_lanes(lanes);
        h = up(**p);
        ok = true;
      }
      break;
    case Kernel::EllInner:
    case Kernel::EllOuter:
      if (auto* p = std::get_if<const EllMatrix*>(&m)) {
        require_dim((*p)->n, x.size());
        require_lanes(lanes);
        h = up(**p);
        ok = true;
      }
      break;
  }
  if (!ok)
    throw Error(ErrorCode::InvalidArgument,
                "matrix format does not match kernel " + kernel_name(kernel));
  // the caller's x, not ones: measure exactly what was asked
  rt::DevArray<double> dx(std::max<std::size_t>(x.size(), 1), "x");
  rt::DevArray<double> dy(static_cast<std::size_t>(std::max<std::int64_t>(h->n, 1)), "y");
  rt::copy_to_device(dx.get(), x.data(), x.size() * sizeof(double));
  dev::spmv_device(*h, to_c(kernel), dx.get(), dy.get());
  rt::sync();
  std::vector<double> samples;
  rt::EventTimer timer;
  for (int r = 0; r < repeats; ++r) {
    timer.start();
    dev::spmv_device(*h, to_c(kernel), dx.get(), dy.get());
    samples.push_back(timer.stop_seconds());
  }
  std::sort(samples.begin(), samples.end());
  const std::size_t mid = samples.size() / 2;
  return samples.size() % 2 ? samples[mid] : 0.5 * (samples[mid - 1] + samples[mid]);
}

std::pair<EllMatrix, double> measure_transformation(const CrsMatrix& m, std::uint64_t max_bytes) {
  if (max_bytes != kNoByteLimit) {
    const std::uint64_t est = estimate_ell_bytes(m);
    if (est > max_bytes)
      throw Error(ErrorCode::MemoryLimit, "ELL footprint estimate " + std::to_string(est) +
                                              " bytes exceeds limit " + std::to_string(max_bytes));
  }
  Handle h = up(m);  // the upload is not part of the transformation
  auto [conv, secs] = at::measure_transformation(*h, SPMVTK_FORMAT_ELL, max_bytes);
  Handle e(conv);
  return {down_ell(*e), secs};
}

double find_d_star(std::span<const std::pair<double, double>> records, double c) {
  return at::find_d_star(std::vector<std::pair<double, double>>(records.begin(), records.end()),
                         c);
}

double find_d_star(const std::vector<BenchRecord>& records, double c) {
  std::vector<std::pair<double, double>> pts;
  for (const auto& r : records)
    if (!r.excluded && r.metrics) pts.emplace_back(r.stats.d_mat, r.metrics->r);
  return at::find_d_star(std::move(pts), c);
}

namespace {
Profile from_internal(const at::Profile& q) {
  Profile p;
  p.machine_label = q.machine_label;
  p.kernel_variant = static_cast<Kernel>(static_cast<int>(q.kernel));
  p.lanes = q.lanes;
  p.c = q.c;
  p.d_star = q.d_star;
  for (const auto& r : q.records) {
    BenchRecord b;
    b.matrix_id = r.matrix_id;
    b.n = r.n;
    b.nnz = r.nnz;
    b.stats = RowStats{r.mu, r.sigma, r.d_mat};
    b.kernel_variant = p.kernel_variant;
    b.lanes = p.lanes;
    if (r.timings) b.timings = Timings{r.timings->t_crs, r.timings->t_ell, r.timings->t_trans};
    if (r.metrics) b.metrics = CostMetrics{r.metrics->sp, r.metrics->tt, r.metrics->r};
    b.excluded = r.excluded;
    b.exclusion_reason = r.exclusion_reason;
    p.records.push_back(std::move(b));
  }
  return p;
}

at::Profile to_internal(const Profile& p) {
  at::Profile q;
  q.machine_label = p.machine_label;
  q.kernel = to_c(p.kernel_variant);
  q.lanes = p.lanes;
  q.c = p.c;
  q.d_star = p.d_star;
  for (const auto& b : p.records) {
    at::Record r;
    r.matrix_id = b.matrix_id;
    r.n = b.n;
    r.nnz = b.nnz;
    r.mu = b.stats.mu;
    r.sigma = b.stats.sigma;
    r.d_mat = b.stats.d_mat;
    if (b.timings) r.timings = at::Timings{b.timings->t_crs, b.timings->t_ell, b.timings->t_trans};
    if (b.metrics) r.metrics = at::Metrics{b.metrics->sp, b.metrics->tt, b.metrics->r};
    r.excluded = b.excluded;
    r.exclusion_reason = b.exclusion_reason;
    q.records.push_back(std::move(r));
  }
  return q;
}
}  // namespace

Profile offline_profile(std::span<const std::pair<std::string, const CrsMatrix*>> matrix_set,
                        const ProfileOptions& opts) {
  if (matrix_set.empty()) throw Error(ErrorCode::InvalidArgument, "empty benchmark matrix set");
  std::vector<Handle> owned;
  std::vector<std::pair<std::string, const dev::Matrix*>> set;
  for (const auto& [id, mat] : matrix_set) {
    owned.push_back(up(*mat));
    set.emplace_back(id, owned.back().get());
  }
  return from_internal(at::offline_profile(set, to_c(opts.kernel_variant), opts.lanes, opts.c,
                                           opts.repeats, opts.max_bytes, opts.machine_label));
}

Selection online_select(const CrsMatrix& m, const Profile& p) {
  Selection s;
  s.d_mat = row_stats(m).d_mat;
  s.decision = s.d_mat < p.d_star ? Decision::UseEll : Decision::UseCrs;
  return s;
}

std::string profile_to_json(const Profile& p) { return at::profile_to_json(to_internal(p)); }

Profile profile_from_json(const std::string& text) {
  return from_internal(at::profile_from_json(text));
}

void write_profile(const Profile& p, const std::filesystem::path& path) {
  std::ofstream out(path);
  if (!out) throw Error(ErrorCode::Io, "cannot open " + path.string() + " for writing");
  out << profile_to_json(p) << '\n';
  if (!out) throw Error(ErrorCode::Io, "write failed: " + path.string());
}

Profile read_profile(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw Error(ErrorCode::Io, "cannot open " + path.string());
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  return profile_from_json(text);
}

// ---------------------------------------------------------------- ingest
namespace {
CrsMatrix to_crs(gen::HostCrs&& h) {
  CrsMatrix m;
  m.n = h.n;
  if (h.wide()) {
    m.row_ptr = std::move(h.row_ptr);
    m.col_idx = std::move(h.col_idx);
  } else {
    m.row_ptr.assign(h.row_ptr32.begin(), h.row_ptr32.end());
    m.col_idx.assign(h.col32.begin(), h.col32.end());
    for (auto& v : m.row_ptr) v += 1 - h.base;
    for (auto& v : m.col_idx) v += 1 - h.base;
  }
  m.values = std::move(h.values);
  return m;
}
}  // namespace

CrsMatrix read_matrix_market(const std::filesystem::path& path) {
  return to_crs(mm::read(path.string()));
}

void write_matrix_market(const CrsMatrix& m, const std::filesystem::path& path) {
  std::vector<index_t> rows(static_cast<std::size_t>(m.nnz()));
  for (index_t i = 1; i <= m.n; ++i)
    for (index_t p = m.row_ptr[i - 1]; p < m.row_ptr[i]; ++p) rows[p - 1] = i;
  mm::write(m.n, std::move(rows), m.col_idx, m.values, false, path.string());
}

CrsMatrix gen_banded(index_t n, index_t half_width) { return to_crs(gen::banded(n, half_width)); }

CrsMatrix gen_skewed(index_t n, index_t base_deg, index_t heavy_rows, index_t heavy_deg,
                     std::uint64_t seed) {
  return to_crs(gen::skewed(n, base_deg, heavy_rows, heavy_deg, seed));
}

CrsMatrix gen_cv_target(index_t n, double mean_deg, double target_dmat, std::uint64_t seed) {
  return to_crs(gen::cv_target(n, mean_deg, target_dmat, seed));
}

}  // namespace spmvtk
