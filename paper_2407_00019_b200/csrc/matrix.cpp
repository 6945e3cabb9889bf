// matrix.cpp -- handle construction, conversions and SpMV dispatch.
#include "matrix.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "spmvtk/spmvtk_kernels.h"

namespace spmvtk::dev {

using rt::DevArray;

namespace {

void* s() { return rt::stream(); }

std::int64_t round_up(std::int64_t v, std::int64_t a) { return (v + a - 1) / a * a; }

void require_int32_range(std::int64_t n, std::int64_t nnz) {
  if (n < 0) throw Error(ErrorCode::InvalidArgument, "negative dimension");
  if (n >= INT32_MAX || nnz >= INT32_MAX)
    throw Error(ErrorCode::InvalidArgument,
                "matrix exceeds the int32 device index range (n or nnz >= 2^31-1)");
}

// Copies an index array given in (width, base, location) into an int32
// 0-based device array; narrowing / rebasing runs on the GPU.
void upload_index(DevArray<std::int32_t>& dst, const void* src, std::int64_t len, int width,
                  int base, bool on_device, const char* what) {
  dst.reset(static_cast<std::size_t>(len), what);
  if (len == 0) return;
  if (width == 4) {
    if (on_device)
      rt::check(cudaMemcpyAsync(dst.get(), src, len * 4, cudaMemcpyDeviceToDevice, rt::stream()),
                what);
    else
      rt::copy_to_device(dst.get(), src, len * 4);
    if (base != 0) {
      // rebase in place through the widening kernels' int32 path
      DevArray<std::int64_t> tmp(static_cast<std::size_t>(len), what);
      rt::check_launch(spmvtk_k_widen_index(dst.get(), tmp.get(), len, 0, s()), what);
      rt::check_launch(spmvtk_k_narrow_index(tmp.get(), dst.get(), len, base, s()), what);
    }
  } else {
    DevArray<std::int64_t> tmp(static_cast<std::size_t>(len), what);
    if (on_device)
      rt::check(cudaMemcpyAsync(tmp.get(), src, len * 8, cudaMemcpyDeviceToDevice, rt::stream()),
                what);
    else
      rt::copy_to_device(tmp.get(), src, len * 8);
    rt::check_launch(spmvtk_k_narrow_index(tmp.get(), dst.get(), len, base, s()), what);
  }
}

unsigned long long count_bad_indices(const std::int32_t* idx, std::int64_t len, std::int64_t n) {
  DevArray<unsigned long long> bad(1, "validation");
  rt::check_launch(spmvtk_k_count_out_of_range(idx, len, n, bad.get(), s()), "validation");
  unsigned long long h = 0;
  rt::copy_to_host(&h, bad.get(), sizeof(h));
  return h;
}

Matrix* new_matrix(spmvtk_format f, std::int64_t n, std::int64_t nnz) {
  auto* m = new Matrix;
  m->format = f;
  m->n = n;
  m->nnz = nnz;
  m->ncols = n;
  cudaGetDevice(&m->device);
  return m;
}

// conversions inherit the shape of their source (row-block shards)
Matrix* derived(const Matrix& src, spmvtk_format f, std::int64_t nnz) {
  Matrix* m = new_matrix(f, src.n, nnz);
  m->ncols = src.ncols;
  m->row_offset = src.row_offset;
  return m;
}

int ell_splits(std::int64_t n, std::int32_t nz) {
  if (const int forced = spmvtk_k_ell_splits_forced(); forced > 0)
    return std::max(1, std::min<int>(forced, nz));
  // band split only pays when row pairs alone cannot fill 148 SMs x 2048
  const std::int64_t want = 148LL * 2048;
  const std::int64_t pairs = (n + 1) / 2;
  if (nz <= 1 || pairs >= want) return 1;
  std::int64_t sp = (want + pairs - 1) / pairs;
  return static_cast<int>(std::min<std::int64_t>(sp, nz));
}

}  // namespace

const char* kernel_label(spmvtk_kernel k) {
  switch (k) {
    case SPMVTK_KERNEL_CRS: return "crs";
    case SPMVTK_KERNEL_COO_ROW_OUTER: return "coo-row";
    case SPMVTK_KERNEL_COO_COL_OUTER: return "coo-col";
    case SPMVTK_KERNEL_ELL_INNER: return "ell-inner";
    case SPMVTK_KERNEL_ELL_OUTER: return "ell-outer";
    case SPMVTK_KERNEL_ELL_ROWMAJOR: return "ell-row";
  }
  return "unknown";
}

rt::Moments crs_moments(const Matrix& m) {
  std::lock_guard<std::mutex> lk(m.mu);
  if (!m.moments) m.moments = rt::row_moments(m.ptr.get(), m.n);
  return *m.moments;
}

const std::vector<std::int32_t>& crs_seg_plan(const Matrix& m, const std::int32_t** dev) {
  std::lock_guard<std::mutex> lk(m.mu);
  const std::int32_t chunk = spmvtk_k_seg_chunk();
  if (m.seg_plan_host.empty() || m.seg_plan_chunk != chunk) {
    const std::int32_t nw = spmvtk_k_seg_plan_warps(m.nnz, chunk);
    DevArray<std::int32_t> plan(static_cast<std::size_t>(nw) + 1, "SpMV plan");
    rt::check_launch(spmvtk_k_seg_plan(m.n, m.nnz, m.ptr.get(), chunk, plan.get(),
                                       rt::stream()),
                     "SpMV plan");
    std::vector<std::int32_t> host(static_cast<std::size_t>(nw) + 1);
    rt::copy_to_host(host.data(), plan.get(), host.size() * sizeof(std::int32_t));  // synchronises
    m.seg_plan = std::move(plan);
    m.seg_plan_host = std::move(host);
    m.seg_plan_chunk = chunk;
  }
  *dev = m.seg_plan.get();
  return m.seg_plan_host;
}

namespace {
// warps whose rows intersect [r0, r1): plan[w] < r1 and plan[w+1] > r0
std::pair<std::int32_t, std::int32_t> plan_warps_for(const std::vector<std::int32_t>& plan,
                                                     std::int64_t r0, std::int64_t r1) {
  const std::int32_t nw = static_cast<std::int32_t>(plan.size()) - 1;
  // first w with plan[w+1] > r0
  const auto lo = std::upper_bound(plan.begin() + 1, plan.end(), static_cast<std::int32_t>(r0));
  const std::int32_t w0 = static_cast<std::int32_t>(lo - (plan.begin() + 1));
  // first w with plan[w] >= r1
  const auto hi = std::lower_bound(plan.begin(), plan.begin() + nw, static_cast<std::int32_t>(r1));
  const std::int32_t w1 = static_cast<std::int32_t>(hi - plan.begin());
  return {w0, std::max(w0, w1)};
}

void spmv_crs_rows(const Matrix& m, const double* x, double* y, std::int64_t r0, std::int64_t r1,
                   cudaStream_t st) {
  rt::Moments mo = crs_moments(m);
  const double mean = m.n > 0 ? static_cast<double>(mo.sum) / static_cast<double>(m.n) : 0;
  if (spmvtk_k_crs_use_seg(mean, static_cast<std::int64_t>(mo.max))) {
    const std::int32_t* plan = nullptr;
    const auto& hp = crs_seg_plan(m, &plan);
    auto [w0, w1] = plan_warps_for(hp, r0, r1);
    rt::check_launch(spmvtk_k_spmv_crs_seg(m.ptr.get(), m.col.get(), m.val.get(), x, y, plan, w0,
                                           w1, r0, r1, m.nnz, st),
                     "spmv crs");
    return;
  }
  const std::int64_t rows = r1 - r0;
  DevArray<std::int32_t> long_rows;
  if (static_cast<std::int64_t>(mo.max) > spmvtk_k_crs_long_limit(mean))
    long_rows.reset(rows + 1, "CRS long-row queue");
  // row pointers stay absolute, so offsetting irp and y is enough
  rt::check_launch(spmvtk_k_spmv_crs(rows, m.ptr.get() + r0, m.col.get(), m.val.get(), x, y + r0,
                                     mean,
                                     static_cast<std::int32_t>(std::min<std::uint64_t>(mo.max, INT32_MAX)),
                                     long_rows.get(), st),
                   "spmv crs");
}
}  // namespace

bool pairs_ascending(const Matrix& m) {
  std::lock_guard<std::mutex> lk(m.mu);
  if (!m.pairs_ascending) {
    // one pass: ordering (the fast CCS pipeline's precondition) and, for a
    // CRS, the band shape (the SM-local ELL kernel's)
    const DevArray<std::int32_t>& idx = m.format == SPMVTK_FORMAT_CCS ? m.row : m.col;
    DevArray<unsigned long long> out(4, "ordering check");
    rt::check_launch(spmvtk_k_row_order_stats(m.ptr.get(), m.n, m.row_offset, idx.get(),
                                              out.get(), s()),
                     "ordering check");
    unsigned long long h[4] = {0, 0, 0, 0};
    rt::copy_to_host(h, out.get(), sizeof(h));
    m.pairs_ascending = h[0] == 0;
    if (m.format == SPMVTK_FORMAT_CRS && h[2] != 0 && h[3] != 0) {
      const long long off = 1LL << 32;
      m.band = Matrix::BandShape{static_cast<long long>(h[2]) - off,
                                 static_cast<long long>(h[3]) - off, h[1]};
    }
  }
  return *m.pairs_ascending;
}

// Band-major ELL of a banded matrix whose columns scatter inside the band:
// the SM-local kernel (one CTA per SM sweeping a row region) keeps each SM's
// x gathers inside one band window that L1 holds.  Measured on configs 1-5
// (profiles/r02_ell_banded.txt): config 5 at D = 0 240 -> 157 us, at D = 0.1
// 274 -> 238 us; slower where the interleaved grid already has locality
// (stencil runs of adjacent columns, config 3), where padding makes the
// product a stream (D >= 0.2), on random columns (config 2) and small n.
bool ell_banded(const Matrix& m) {
  const int forced = spmvtk_k_ell_banded_forced();
  if (forced >= 0) return forced == 1;
  if (!m.band) return false;
  const Matrix::BandShape& b = *m.band;
  const std::int64_t window = b.right + b.left + 1;
  const double slots = static_cast<double>(m.n) * m.band_count;
  return m.n >= std::int64_t(148) * 2048 && window > 4096 &&
         window <= (std::int64_t(1) << 17) &&
         b.adjacent * 8 < static_cast<std::uint64_t>(m.nnz) &&
         slots <= 1.6 * static_cast<double>(m.nnz);
}

namespace {
// CRS (or CCS read as the CRS of the transpose) -> CCS / COO-col: the
// rank-by-row pipeline when every segment's indices ascend strictly (no
// duplicate pairs), else the stable partition that keeps duplicates in CRS
// order (convert.cpp:43-51 semantics either way).
void launch_ccs(const Matrix& a, const std::int32_t* seg_idx, std::int32_t* col_ptr,
                std::int32_t* row_out, std::int32_t* col_out, double* val_out, void* scratch,
                cudaStream_t st) {
  const bool stable = spmvtk_k_ccs_force_stable() || !pairs_ascending(a);
  const std::int64_t n = a.n, nnz = a.nnz;
  int rc;
  if (col_out)
    rc = stable ? spmvtk_k_crs_to_coo_col_stable(n, nnz, a.ptr.get(), seg_idx, a.val.get(),
                                                 col_ptr, row_out, col_out, val_out, scratch, st)
                : spmvtk_k_crs_to_coo_col(n, nnz, a.ptr.get(), seg_idx, a.val.get(), col_ptr,
                                          row_out, col_out, val_out, scratch, st);
  else
    rc = stable ? spmvtk_k_crs_to_ccs_stable(n, nnz, a.ptr.get(), seg_idx, a.val.get(), col_ptr,
                                             row_out, val_out, scratch, st)
                : spmvtk_k_crs_to_ccs(n, nnz, a.ptr.get(), seg_idx, a.val.get(), col_ptr,
                                      row_out, val_out, scratch, st);
  rt::check_launch(rc, col_out ? "CRS->COO-col" : "CRS->CCS");
}
}  // namespace

Matrix* crs_from_arrays(std::int64_t n, std::int64_t nnz, const void* row_ptr,
                        const void* col_idx, const double* values, int index_width,
                        int index_base, bool on_device) {
  return crs_block_from_arrays(n, n, 0, nnz, row_ptr, col_idx, values, index_width, index_base,
                               on_device);
}

Matrix* crs_block_from_arrays(std::int64_t n, std::int64_t ncols, std::int64_t row_offset,
                              std::int64_t nnz, const void* row_ptr, const void* col_idx,
                              const double* values, int index_width, int index_base,
                              bool on_device) {
  rt::init();
  require_int32_range(n, nnz);
  require_int32_range(ncols, 0);
  if (row_offset < 0 || row_offset > INT32_MAX)
    throw Error(ErrorCode::InvalidArgument, "row offset out of range");
  if (nnz < 0) throw Error(ErrorCode::InvalidArgument, "negative nnz");
  if (index_width != 4 && index_width != 8)
    throw Error(ErrorCode::InvalidArgument, "index_width must be 4 or 8");
  if (index_base != 0 && index_base != 1)
    throw Error(ErrorCode::InvalidArgument, "index_base must be 0 or 1");
  if (!row_ptr || ((!col_idx || !values) && nnz > 0))
    throw Error(ErrorCode::InvalidArgument, "null array");
  std::unique_ptr<Matrix> m(new_matrix(SPMVTK_FORMAT_CRS, n, nnz));
  m->ncols = ncols;
  m->row_offset = row_offset;
  upload_index(m->ptr, row_ptr, n + 1, index_width, index_base, on_device, "row_ptr upload");
  upload_index(m->col, col_idx, nnz, index_width, index_base, on_device, "col_idx upload");
  m->val.reset(static_cast<std::size_t>(nnz), "values upload");
  if (nnz) {
    rt::check(cudaMemcpyAsync(m->val.get(), values, nnz * sizeof(double),
                              on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                              rt::stream()),
              "values upload");
  }
  // validation on the GPU (formats.cpp:19-41 pointer rules, :43-52 ranges)
  std::int32_t ends[2] = {0, 0};
  rt::copy_to_host(&ends[0], m->ptr.get(), sizeof(std::int32_t));
  rt::copy_to_host(&ends[1], m->ptr.get() + n, sizeof(std::int32_t));
  if (ends[0] != 0) throw Error(ErrorCode::Validation, "row_ptr[1] != 1");
  if (ends[1] != nnz)
    throw Error(ErrorCode::Validation, "pointer array end " + std::to_string(ends[1] + 1) +
                                           ", expected nnz+1 = " + std::to_string(nnz + 1));
  rt::Moments mo = rt::row_moments(m->ptr.get(), n);
  if (!mo.monotone) throw Error(ErrorCode::Validation, "row_ptr not nondecreasing");
  m->moments = mo;
  if (nnz && count_bad_indices(m->col.get(), nnz, ncols))
    throw Error(ErrorCode::Validation, "column index out of range");
  pairs_ascending(*m);  // ordering of every row, cached (a CCS precondition)
  return m.release();
}

Matrix* coo_from_arrays(std::int64_t n, std::int64_t nnz, const void* rows, const void* cols,
                        const double* values, int index_width, int index_base, int ordering) {
  rt::init();
  require_int32_range(n, nnz);
  if (ordering != 0 && ordering != 1)
    throw Error(ErrorCode::InvalidArgument, "COO ordering must be row- or column-major");
  std::unique_ptr<Matrix> m(new_matrix(ordering == 0 ? SPMVTK_FORMAT_COO_ROW
                                                     : SPMVTK_FORMAT_COO_COL,
                                       n, nnz));
  m->ordering = ordering;
  upload_index(m->row, rows, nnz, index_width, index_base, false, "COO row upload");
  upload_index(m->col, cols, nnz, index_width, index_base, false, "COO col upload");
  m->val.reset(static_cast<std::size_t>(nnz), "COO values upload");
  if (nnz) rt::copy_to_device(m->val.get(), values, nnz * sizeof(double));
  if (nnz && (count_bad_indices(m->row.get(), nnz, n) || count_bad_indices(m->col.get(), nnz, n)))
    throw Error(ErrorCode::Validation, "COO index out of range");
  if (ordering == 0 && nnz > 1) {
    DevArray<unsigned long long> bad(1, "validation");
    rt::check_launch(spmvtk_k_count_descents(m->row.get(), nnz, bad.get(), s()), "validation");
    unsigned long long h = 0;
    rt::copy_to_host(&h, bad.get(), sizeof(h));
    m->rows_sorted = h == 0;
  }
  return m.release();
}

Matrix* ell_from_arrays(std::int64_t n, std::int64_t band_count, const std::int64_t* col_1based,
                        const double* values, const std::int64_t* row_entry_count,
                        std::int64_t stored_nnz) {
  rt::init();
  require_int32_range(n, stored_nnz);
  if (band_count < 0 || band_count > INT32_MAX)
    throw Error(ErrorCode::InvalidArgument, "band count out of range");
  std::unique_ptr<Matrix> m(new_matrix(SPMVTK_FORMAT_ELL, n, stored_nnz));
  m->band_count = static_cast<std::int32_t>(band_count);
  m->ld = round_up(n, 32);
  const std::size_t slots = static_cast<std::size_t>(m->ld) * static_cast<std::size_t>(band_count);
  m->val.reset(slots, "ELL values");
  m->col.reset(slots, "ELL col_idx");
  m->count.reset(n, "ELL row_entry_count");
  cudaStream_t st = rt::stream();
  if (slots) {
    rt::check(cudaMemsetAsync(m->val.get(), 0, slots * sizeof(double), st), "ELL upload");
    rt::check(cudaMemsetAsync(m->col.get(), 0, slots * sizeof(std::int32_t), st), "ELL upload");
    DevArray<std::int32_t> compact;
    upload_index(compact, col_1based, n * band_count, 8, 1, false, "ELL col upload");
    DevArray<double> vcompact(static_cast<std::size_t>(n * band_count), "ELL value upload");
    rt::copy_to_device(vcompact.get(), values, static_cast<std::size_t>(n * band_count) * 8);
    rt::check(cudaMemcpy2DAsync(m->val.get(), m->ld * 8, vcompact.get(), n * 8, n * 8,
                                band_count, cudaMemcpyDeviceToDevice, st),
              "ELL upload");
    rt::check(cudaMemcpy2DAsync(m->col.get(), m->ld * 4, compact.get(), n * 4, n * 4, band_count,
                                cudaMemcpyDeviceToDevice, st),
              "ELL upload");
    if (count_bad_indices(m->col.get(), static_cast<std::int64_t>(slots), n))
      throw Error(ErrorCode::Validation, "ELL column index out of range");
  }
  upload_index(m->count, row_entry_count, n, 8, 0, false, "ELL counts upload");
  rt::sync();
  return m.release();
}

std::uint64_t reference_ell_estimate(const Matrix& crs) {
  rt::Moments mo = crs_moments(crs);
  return static_cast<std::uint64_t>(crs.n) * mo.max * 16ull;
}

std::uint64_t device_bytes_for(const Matrix& crs, spmvtk_format to) {
  const std::uint64_t n = static_cast<std::uint64_t>(crs.n);
  const std::uint64_t nnz = static_cast<std::uint64_t>(crs.nnz);
  switch (to) {
    case SPMVTK_FORMAT_CRS:
    case SPMVTK_FORMAT_CCS: return 12 * nnz + 4 * (n + 1);
    case SPMVTK_FORMAT_COO_ROW:
    case SPMVTK_FORMAT_COO_COL: return 16 * nnz;
    case SPMVTK_FORMAT_ELL: {
      rt::Moments mo = crs_moments(crs);
      return 12ull * static_cast<std::uint64_t>(round_up(crs.n, 32)) * mo.max + 4 * n;
    }
    case SPMVTK_FORMAT_ELL_ROWMAJOR: {
      rt::Moments mo = crs_moments(crs);
      return 12ull * n * mo.max + 4 * n;
    }
  }
  return 0;
}

Matrix* convert(const Matrix& a, spmvtk_format to, std::uint64_t max_bytes) {
  rt::init();
  if (a.format != SPMVTK_FORMAT_CRS)
    throw Error(ErrorCode::InvalidArgument, "operation requires a CRS handle");
  const std::int64_t n = a.n, nnz = a.nnz;
  switch (to) {
    case SPMVTK_FORMAT_CRS: {
      std::unique_ptr<Matrix> m(derived(a, SPMVTK_FORMAT_CRS, nnz));
      m->ptr.reset(n + 1, "CRS copy");
      m->col.reset(nnz, "CRS copy");
      m->val.reset(nnz, "CRS copy");
      cudaStream_t st = rt::stream();
      rt::check(cudaMemcpyAsync(m->ptr.get(), a.ptr.get(), a.ptr.bytes(), cudaMemcpyDeviceToDevice, st), "CRS copy");
      rt::check(cudaMemcpyAsync(m->col.get(), a.col.get(), a.col.bytes(), cudaMemcpyDeviceToDevice, st), "CRS copy");
      rt::check(cudaMemcpyAsync(m->val.get(), a.val.get(), a.val.bytes(), cudaMemcpyDeviceToDevice, st), "CRS copy");
      std::lock_guard<std::mutex> lk(a.mu);
      m->moments = a.moments;
      return m.release();
    }
    case SPMVTK_FORMAT_COO_ROW: {
      // convert.cpp:11-22: copy values / col_idx, expand row_ptr
      std::unique_ptr<Matrix> m(derived(a, SPMVTK_FORMAT_COO_ROW, nnz));
      m->ordering = 0;
      m->row.reset(nnz, "COO row_idx");
      m->col.reset(nnz, "COO col_idx");
      m->val.reset(nnz, "COO values");
      cudaStream_t st = rt::stream();
      if (nnz)
        rt::check_launch(spmvtk_k_crs_to_coo_row(n, nnz, a.ptr.get(), a.col.get(), a.val.get(),
                                                 m->row.get(), m->col.get(), m->val.get(), st),
                         "CRS->COO-row");
      return m.release();
    }
    case SPMVTK_FORMAT_CCS:
    case SPMVTK_FORMAT_COO_COL: {
      // Phase I (convert.cpp:24-53) into the output arrays directly; for
      // COO-col Phase II (convert.cpp:55-66) expands col_ptr into col_idx
      // and the CCS arrays become the COO arrays without a copy.
      const bool coo = to == SPMVTK_FORMAT_COO_COL;
      if (a.ncols != a.n)
        throw Error(ErrorCode::InvalidArgument,
                    "column-ordered formats need a square matrix (row-block shards convert to "
                    "CRS, COO-row and ELL only)");
      std::unique_ptr<Matrix> m(derived(a, to, nnz));
      m->row.reset(nnz, "CCS row_idx");
      m->val.reset(nnz, "CCS values");
      DevArray<std::int32_t> colptr(n + 1, "CCS col_ptr");
      DevArray<unsigned char> scratch(spmvtk_k_ccs_scratch_bytes(n, nnz), "CCS scratch");
      cudaStream_t st = rt::stream();
      if (coo) {
        // Phase II folded into Phase I: the sort writes each entry's column
        m->ordering = 1;
        m->col.reset(nnz, "COO col_idx");
        launch_ccs(a, a.col.get(), colptr.get(), m->row.get(), m->col.get(), m->val.get(),
                   scratch.get(), st);
      } else {
        launch_ccs(a, a.col.get(), colptr.get(), m->row.get(), nullptr, m->val.get(),
                   scratch.get(), st);
        m->ptr = std::move(colptr);
      }
      return m.release();
    }
    case SPMVTK_FORMAT_ELL:
    case SPMVTK_FORMAT_ELL_ROWMAJOR: {
      // convert.cpp:81-115: guard, band_count = max row, padded scatter.
      // The max row comes from a fresh GPU reduction (as the reference
      // recomputes it), never from a cache.
      // band_count = the max row, from the handle's exact row moments
      // (reduced on the GPU when the handle was built; the handle is
      // immutable, so no reduction or host round trip on this path)
      rt::Moments mo = crs_moments(a);
      if (max_bytes != 0) {
        std::uint64_t est = static_cast<std::uint64_t>(n) * mo.max * 16ull;
        if (est > max_bytes)
          throw Error(ErrorCode::MemoryLimit, "ELL footprint estimate " + std::to_string(est) +
                                                  " bytes exceeds limit " +
                                                  std::to_string(max_bytes));
      }
      if (mo.max > static_cast<std::uint64_t>(INT32_MAX))
        throw Error(ErrorCode::InvalidArgument, "band count exceeds int32");
      const std::int32_t nz = static_cast<std::int32_t>(mo.max);
      const bool cm = to == SPMVTK_FORMAT_ELL;
      std::unique_ptr<Matrix> m(derived(a, to, nnz));
      m->band_count = nz;
      m->ld = cm ? round_up(n, 32) : n;
      {
        std::lock_guard<std::mutex> lk(a.mu);
        m->band = a.band;  // measured at upload (pairs_ascending): no work here
      }
      const std::size_t slots =
          static_cast<std::size_t>(cm ? m->ld : n) * static_cast<std::size_t>(nz);
      // values | col_idx | row_entry_count in one allocation
      const std::size_t vbytes = (slots * 8 + 255) & ~std::size_t(255);
      const std::size_t cbytes = (slots * 4 + 255) & ~std::size_t(255);
      m->block.reset(vbytes + cbytes + static_cast<std::size_t>(n) * 4, "ELL arrays");
      unsigned char* base = m->block.get();
      m->val.view(reinterpret_cast<double*>(base), slots);
      m->col.view(reinterpret_cast<std::int32_t*>(base + vbytes), slots);
      m->count.view(reinterpret_cast<std::int32_t*>(base + vbytes + cbytes),
                    static_cast<std::size_t>(n));
      cudaStream_t st = rt::stream();
      if (cm)
        rt::check_launch(spmvtk_k_crs_to_ell_cm(n, nz, m->ld, a.ptr.get(), a.col.get(),
                                                a.val.get(), m->val.get(), m->col.get(),
                                                m->count.get(), a.row_offset, st),
                         "CRS->ELL");
      else
        rt::check_launch(spmvtk_k_crs_to_ell_rm(n, nz, a.ptr.get(), a.col.get(), a.val.get(),
                                                m->val.get(), m->col.get(), m->count.get(),
                                                a.row_offset, st),
                         "CRS->ELL row-major");
      return m.release();
    }
  }
  throw Error(ErrorCode::InvalidArgument, "unknown target format");
}

Matrix* to_crs(const Matrix& a) {
  rt::init();
  const std::int64_t n = a.n, nnz = a.nnz;
  std::unique_ptr<Matrix> m(derived(a, SPMVTK_FORMAT_CRS, nnz));
  m->ptr.reset(n + 1, "CRS row_ptr");
  m->col.reset(nnz, "CRS col_idx");
  m->val.reset(nnz, "CRS values");
  cudaStream_t st = rt::stream();
  DevArray<unsigned long long> dup(1, "duplicate flag");
  DevArray<unsigned char> scratch(spmvtk_k_canon_scratch_bytes(n) +
                                      spmvtk_k_ccs_scratch_bytes(a.ncols, nnz),
                                  "canonical CRS scratch");
  bool check_dup = true;
  switch (a.format) {
    case SPMVTK_FORMAT_CRS:
      rt::check(cudaMemcpyAsync(m->ptr.get(), a.ptr.get(), a.ptr.bytes(), cudaMemcpyDeviceToDevice, st), "copy");
      rt::check(cudaMemcpyAsync(m->col.get(), a.col.get(), a.col.bytes(), cudaMemcpyDeviceToDevice, st), "copy");
      rt::check(cudaMemcpyAsync(m->val.get(), a.val.get(), a.val.bytes(), cudaMemcpyDeviceToDevice, st), "copy");
      rt::check_launch(spmvtk_k_sort_segments(m->ptr.get(), n, a.ncols, m->col.get(), m->val.get(),
                                              dup.get(), scratch.get(), st),
                       "canonicalize");
      check_dup = false;  // canonicalize() does not refuse (formats.cpp:228-244)
      break;
    case SPMVTK_FORMAT_CCS:
      // the CCS of A is the CRS of A^T: transposing it back yields the CRS of
      // A with rows visited in order, i.e. columns ascending in every row
      launch_ccs(a, a.row.get(), m->ptr.get(), m->col.get(), nullptr, m->val.get(),
                 scratch.get(), st);
      check_dup = false;
      break;
    case SPMVTK_FORMAT_COO_ROW:
    case SPMVTK_FORMAT_COO_COL:
      rt::check_launch(spmvtk_k_coo_to_crs(n, a.ncols, nnz, a.row.get(), a.col.get(),
                                           a.val.get(), m->ptr.get(), m->col.get(),
                                           m->val.get(), dup.get(), scratch.get(), st),
                       "COO->CRS");
      break;
    case SPMVTK_FORMAT_ELL:
    case SPMVTK_FORMAT_ELL_ROWMAJOR: {
      const bool cm = a.format == SPMVTK_FORMAT_ELL;
      rt::check_launch(spmvtk_k_ell_to_crs(n, a.ncols, cm ? a.ld : 1, cm ? 1 : a.band_count,
                                           a.val.get(), a.col.get(), a.count.get(),
                                           m->ptr.get(), m->col.get(), m->val.get(), dup.get(),
                                           scratch.get(), st),
                       "ELL->CRS");
      break;
    }
  }
  if (check_dup) {
    unsigned long long d = 0;
    rt::copy_to_host(&d, dup.get(), sizeof(d));
    if (d != ~0ull)
      throw Error(ErrorCode::Validation,
                  "duplicate (row, col) pair (" + std::to_string((d >> 32) + 1 + a.row_offset) +
                      ", " + std::to_string((d & 0xffffffffull) + 1) + ")");
  }
  return m.release();
}

double transform_kernel_seconds(const Matrix& a, spmvtk_format to, int repeats) {
  if (a.format != SPMVTK_FORMAT_CRS)
    throw Error(ErrorCode::InvalidArgument, "operation requires a CRS handle");
  if (repeats < 1) throw Error(ErrorCode::InvalidArgument, "repeats must be at least 1");
  // outputs and scratch allocated once, outside the timed launches
  std::unique_ptr<Matrix> out(convert(a, to, 0));
  const std::int64_t n = a.n, nnz = a.nnz;
  cudaStream_t st = rt::stream();
  DevArray<std::int32_t> colptr;
  DevArray<unsigned char> scratch;
  if (to == SPMVTK_FORMAT_CCS || to == SPMVTK_FORMAT_COO_COL) {
    colptr.reset(n + 1, "CCS col_ptr");
    scratch.reset(spmvtk_k_ccs_scratch_bytes(n, nnz), "CCS scratch");
  }
  auto once = [&] {
    switch (to) {
      case SPMVTK_FORMAT_CRS:
        cudaMemcpyAsync(out->ptr.get(), a.ptr.get(), a.ptr.bytes(), cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(out->col.get(), a.col.get(), a.col.bytes(), cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(out->val.get(), a.val.get(), a.val.bytes(), cudaMemcpyDeviceToDevice, st);
        break;
      case SPMVTK_FORMAT_COO_ROW:
        rt::check_launch(spmvtk_k_crs_to_coo_row(n, nnz, a.ptr.get(), a.col.get(), a.val.get(),
                                                 out->row.get(), out->col.get(), out->val.get(),
                                                 st),
                         "CRS->COO-row");
        break;
      case SPMVTK_FORMAT_CCS:
      case SPMVTK_FORMAT_COO_COL:
        launch_ccs(a, a.col.get(), colptr.get(), out->row.get(),
                   to == SPMVTK_FORMAT_COO_COL ? out->col.get() : nullptr, out->val.get(),
                   scratch.get(), st);
        break;
      case SPMVTK_FORMAT_ELL:
        rt::check_launch(spmvtk_k_crs_to_ell_cm(n, out->band_count, out->ld, a.ptr.get(),
                                                a.col.get(), a.val.get(), out->val.get(),
                                                out->col.get(), out->count.get(), a.row_offset,
                                                st),
                         "CRS->ELL");
        break;
      case SPMVTK_FORMAT_ELL_ROWMAJOR:
        rt::check_launch(spmvtk_k_crs_to_ell_rm(n, out->band_count, a.ptr.get(), a.col.get(),
                                                a.val.get(), out->val.get(), out->col.get(),
                                                out->count.get(), a.row_offset, st),
                         "CRS->ELL row-major");
        break;
    }
  };
  once();
  rt::sync();
  std::vector<double> samples;
  rt::EventTimer timer;
  for (int r = 0; r < repeats; ++r) {
    timer.start();
    once();
    samples.push_back(timer.stop_seconds());
  }
  std::sort(samples.begin(), samples.end());
  return samples[samples.size() / 2];
}

bool spmv_row_splittable(const Matrix& m, spmvtk_kernel kernel) {
  return (kernel == SPMVTK_KERNEL_CRS && m.format == SPMVTK_FORMAT_CRS) ||
         (kernel == SPMVTK_KERNEL_ELL_INNER && m.format == SPMVTK_FORMAT_ELL) ||
         (kernel == SPMVTK_KERNEL_ELL_ROWMAJOR && m.format == SPMVTK_FORMAT_ELL_ROWMAJOR);
}

void spmv_device_rows(const Matrix& m, spmvtk_kernel kernel, const double* x, double* y,
                      std::int64_t r0, std::int64_t r1) {
  if (!spmv_row_splittable(m, kernel) || r0 < 0 || r1 > m.n || r0 > r1 || (r0 & 63))
    throw Error(ErrorCode::InvalidArgument, "row-range SpMV not available for this kernel");
  const std::int64_t rows = r1 - r0;
  if (rows == 0) return;
  cudaStream_t st = rt::stream();
  switch (kernel) {
    case SPMVTK_KERNEL_CRS:
      spmv_crs_rows(m, x, y, r0, r1, st);
      return;
    case SPMVTK_KERNEL_ELL_INNER:
      rt::check_launch(spmvtk_k_spmv_ell_cm(rows, m.band_count, m.ld, m.val.get() + r0,
                                            m.col.get() + r0, x, y + r0, st),
                       "spmv ell-inner");
      return;
    default:
      rt::check_launch(spmvtk_k_spmv_ell_rm(rows, m.band_count,
                                            m.val.get() + r0 * static_cast<std::int64_t>(m.band_count),
                                            m.col.get() + r0 * static_cast<std::int64_t>(m.band_count),
                                            x, y + r0, st),
                       "spmv ell-row");
      return;
  }
}

void spmv_device(const Matrix& m, spmvtk_kernel kernel, const double* x, double* y) {
  cudaStream_t st = rt::stream();
  switch (kernel) {
    case SPMVTK_KERNEL_CRS: {
      if (m.format != SPMVTK_FORMAT_CRS)
        throw Error(ErrorCode::InvalidArgument, "operation requires a CRS handle");
      if (m.n > 0) spmv_crs_rows(m, x, y, 0, m.n, st);
      return;
    }
    case SPMVTK_KERNEL_COO_ROW_OUTER:
      if (m.format != SPMVTK_FORMAT_COO_ROW && m.format != SPMVTK_FORMAT_COO_COL)
        throw Error(ErrorCode::InvalidArgument, "kernel requires a row-major COO handle");
      if (m.ordering != 0)
        throw Error(ErrorCode::InvalidArgument,
                    "spmv_coo_row_outer requires the matching COO ordering");
      if (!m.rows_sorted) {
        // host-built COO tagged row-major whose rows are not sorted: the
        // segmented kernel needs sorted rows, the reduction kernel does not
        rt::check_launch(spmvtk_k_spmv_coo_col(m.n, m.nnz, m.row.get(), m.col.get(),
                                               m.val.get(), x, y, st),
                         "spmv coo-row (unsorted)");
        return;
      }
      rt::check_launch(spmvtk_k_spmv_coo_row(m.n, m.nnz, m.row.get(), m.col.get(), m.val.get(),
                                             x, y, st),
                       "spmv coo-row");
      return;
    case SPMVTK_KERNEL_COO_COL_OUTER:
      if (m.format != SPMVTK_FORMAT_COO_ROW && m.format != SPMVTK_FORMAT_COO_COL)
        throw Error(ErrorCode::InvalidArgument, "kernel requires a column-major COO handle");
      if (m.ordering != 1)
        throw Error(ErrorCode::InvalidArgument,
                    "spmv_coo_col_outer requires the matching COO ordering");
      rt::check_launch(spmvtk_k_spmv_coo_col(m.n, m.nnz, m.row.get(), m.col.get(), m.val.get(),
                                             x, y, st),
                       "spmv coo-col");
      return;
    case SPMVTK_KERNEL_ELL_INNER:
    case SPMVTK_KERNEL_ELL_OUTER: {
      if (m.format != SPMVTK_FORMAT_ELL)
        throw Error(ErrorCode::InvalidArgument, "kernel requires an ELL handle");
      if (kernel == SPMVTK_KERNEL_ELL_INNER) {
        rt::check_launch((ell_banded(m) ? spmvtk_k_spmv_ell_cm_banded : spmvtk_k_spmv_ell_cm)(
                             m.n, m.band_count, m.ld, m.val.get(), m.col.get(), x, y, st),
                         "spmv ell-inner");
      } else {
        int splits = ell_splits(m.n, m.band_count);
        DevArray<double> partial;
        if (splits > 1) partial.reset(static_cast<std::size_t>(splits) * m.n, "ELL partials");
        if (splits <= 1 && ell_banded(m)) {  // one band chunk: ell-inner's kernel, as above
          rt::check_launch(spmvtk_k_spmv_ell_cm_banded(m.n, m.band_count, m.ld, m.val.get(),
                                                       m.col.get(), x, y, st),
                           "spmv ell-outer");
          return;
        }
        rt::check_launch(spmvtk_k_spmv_ell_cm_split(m.n, m.band_count, m.ld, m.val.get(),
                                                    m.col.get(), x, y, splits, partial.get(), st),
                         "spmv ell-outer");
      }
      return;
    }
    case SPMVTK_KERNEL_ELL_ROWMAJOR:
      if (m.format != SPMVTK_FORMAT_ELL_ROWMAJOR)
        throw Error(ErrorCode::InvalidArgument, "kernel requires a row-major ELL handle");
      rt::check_launch(spmvtk_k_spmv_ell_rm(m.n, m.band_count, m.val.get(), m.col.get(), x, y, st),
                       "spmv ell-row");
      return;
  }
  throw Error(ErrorCode::InvalidArgument, "unknown kernel id");
}

void spmv_device_push(const Matrix& m, spmvtk_kernel kernel, const double* x,
                      const spmvtk_push& push, const spmvtk_push_sync* sync) {
  if (push.ndst < 1 || push.ndst > SPMVTK_MAX_PEERS)
    throw Error(ErrorCode::InvalidArgument, "push needs 1..8 destinations");
  if (push.local < 0 || push.local >= push.ndst)
    throw Error(ErrorCode::InvalidArgument, "push.local must index a destination");
  for (int w = 0; w < push.ndst; ++w)
    if (push.dst[w] == nullptr && m.n > 0)
      throw Error(ErrorCode::InvalidArgument, "null push destination");
  cudaStream_t st = rt::stream();
  if (kernel == SPMVTK_KERNEL_CRS) {
    if (m.format != SPMVTK_FORMAT_CRS)
      throw Error(ErrorCode::InvalidArgument, "operation requires a CRS handle");
    rt::Moments mo = crs_moments(m);
    const double mean = m.n > 0 ? static_cast<double>(mo.sum) / static_cast<double>(m.n) : 0;
    if (m.n > 0 && spmvtk_k_crs_use_seg(mean, static_cast<std::int64_t>(mo.max))) {
      const std::int32_t* plan = nullptr;
      const auto& hp = crs_seg_plan(m, &plan);
      rt::check_launch(spmvtk_k_spmv_crs_seg_push(m.ptr.get(), m.col.get(), m.val.get(), x, &push,
                                                  sync, plan,
                                                  static_cast<std::int32_t>(hp.size()) - 1, m.n,
                                                  m.nnz, st),
                       "spmv crs (push)");
      return;
    }
    DevArray<std::int32_t> long_rows;
    if (static_cast<std::int64_t>(mo.max) > spmvtk_k_crs_long_limit(mean))
      long_rows.reset(m.n + 1, "CRS long-row queue");
    rt::check_launch(spmvtk_k_spmv_crs_push(m.n, m.ptr.get(), m.col.get(), m.val.get(), x, &push,
                                            sync, mean,
                                            static_cast<std::int32_t>(std::min<std::uint64_t>(mo.max, INT32_MAX)),
                                            long_rows.get(), st),
                     "spmv crs (push)");
    return;
  }
  if (kernel == SPMVTK_KERNEL_ELL_INNER) {
    if (m.format != SPMVTK_FORMAT_ELL)
      throw Error(ErrorCode::InvalidArgument, "kernel requires an ELL handle");
    rt::check_launch(spmvtk_k_spmv_ell_cm_push(m.n, m.band_count, m.ld, m.val.get(), m.col.get(),
                                               x, &push, sync, st),
                     "spmv ell-inner (push)");
    return;
  }
  throw Error(ErrorCode::InvalidArgument, "pushed SpMV supports the CRS and ELL_INNER kernels");
}

std::int64_t device_array(const Matrix& m, spmvtk_array which, void** out) {
  const DevArray<std::int32_t>* ia = nullptr;
  switch (which) {
    case SPMVTK_ARRAY_VALUES:
      *out = m.val.get();
      return static_cast<std::int64_t>(m.val.size());
    case SPMVTK_ARRAY_POINTER: ia = &m.ptr; break;
    case SPMVTK_ARRAY_ROW_IDX: ia = &m.row; break;
    case SPMVTK_ARRAY_COL_IDX: ia = &m.col; break;
    case SPMVTK_ARRAY_ROW_ENTRY_COUNT: ia = &m.count; break;
  }
  if (!ia || (ia->size() == 0 && !(which == SPMVTK_ARRAY_COL_IDX || which == SPMVTK_ARRAY_ROW_IDX)))
    throw Error(ErrorCode::InvalidArgument, "array not present in this format");
  *out = ia->get();
  return static_cast<std::int64_t>(ia->size());
}

std::int64_t copy_array(const Matrix& m, spmvtk_array which, void* dst, std::int64_t capacity,
                        int index_width, int index_base) {
  if (which != SPMVTK_ARRAY_VALUES && index_width != 4 && index_width != 8)
    throw Error(ErrorCode::InvalidArgument, "index_width must be 4 or 8");
  // which arrays exist per format (formats.hpp of the reference)
  bool present = false;
  switch (m.format) {
    case SPMVTK_FORMAT_CRS:
      present = which == SPMVTK_ARRAY_VALUES || which == SPMVTK_ARRAY_POINTER ||
                which == SPMVTK_ARRAY_COL_IDX;
      break;
    case SPMVTK_FORMAT_CCS:
      present = which == SPMVTK_ARRAY_VALUES || which == SPMVTK_ARRAY_POINTER ||
                which == SPMVTK_ARRAY_ROW_IDX;
      break;
    case SPMVTK_FORMAT_COO_ROW:
    case SPMVTK_FORMAT_COO_COL:
      present = which == SPMVTK_ARRAY_VALUES || which == SPMVTK_ARRAY_ROW_IDX ||
                which == SPMVTK_ARRAY_COL_IDX;
      break;
    case SPMVTK_FORMAT_ELL:
    case SPMVTK_FORMAT_ELL_ROWMAJOR:
      present = which == SPMVTK_ARRAY_VALUES || which == SPMVTK_ARRAY_COL_IDX ||
                which == SPMVTK_ARRAY_ROW_ENTRY_COUNT;
      break;
  }
  if (!present) throw Error(ErrorCode::InvalidArgument, "array not present in this format");

  const bool ell = m.format == SPMVTK_FORMAT_ELL || m.format == SPMVTK_FORMAT_ELL_ROWMAJOR;
  const bool ell_cm = m.format == SPMVTK_FORMAT_ELL;
  std::int64_t len = 0;
  if (which == SPMVTK_ARRAY_VALUES || which == SPMVTK_ARRAY_COL_IDX)
    len = ell ? m.n * static_cast<std::int64_t>(m.band_count) : m.nnz;
  else if (which == SPMVTK_ARRAY_POINTER)
    len = m.n + 1;
  else if (which == SPMVTK_ARRAY_ROW_IDX)
    len = m.nnz;
  else
    len = m.n;
  if (!dst) return len;
  if (capacity < len) throw Error(ErrorCode::InvalidArgument, "destination too small");
  if (len == 0) return 0;

  cudaStream_t st = rt::stream();
  // gather the logical array into a contiguous device buffer (compacting
  // the ELL leading-dimension padding), then convert width/base
  const std::size_t esz = which == SPMVTK_ARRAY_VALUES ? 8 : 4;
  if (which == SPMVTK_ARRAY_ROW_ENTRY_COUNT) index_base = 0;  // a count, not an index
  void* src = nullptr;
  device_array(m, which, &src);
  DevArray<unsigned char> compact;
  const void* contiguous = src;
  if (ell_cm && (which == SPMVTK_ARRAY_VALUES || which == SPMVTK_ARRAY_COL_IDX) && m.ld != m.n) {
    compact.reset(static_cast<std::size_t>(len) * esz, "ELL export");
    rt::check(cudaMemcpy2DAsync(compact.get(), m.n * esz, src, m.ld * esz, m.n * esz,
                                m.band_count, cudaMemcpyDeviceToDevice, st),
              "ELL export");
    contiguous = compact.get();
  }
  if (which == SPMVTK_ARRAY_VALUES || (index_width == 4 && index_base == 0)) {
    rt::copy_to_host(dst, contiguous, static_cast<std::size_t>(len) * esz);
    return len;
  }
  DevArray<std::int64_t> wide(static_cast<std::size_t>(len), "index export");
  rt::check_launch(spmvtk_k_widen_index(static_cast<const std::int32_t*>(contiguous), wide.get(),
                                        len, index_base, st),
                   "index export");
  if (index_width == 8) {
    rt::copy_to_host(dst, wide.get(), static_cast<std::size_t>(len) * 8);
  } else {
    DevArray<std::int32_t> narrow(static_cast<std::size_t>(len), "index export");
    rt::check_launch(spmvtk_k_narrow_index(wide.get(), narrow.get(), len, 0, st), "index export");
    rt::copy_to_host(dst, narrow.get(), static_cast<std::size_t>(len) * 4);
  }
  return len;
}

void copy_ell_bands(const Matrix& m, std::int64_t k0, std::int64_t k1, double* values,
                    std::int64_t* col_idx, int index_base) {
  if (m.format != SPMVTK_FORMAT_ELL)
    throw Error(ErrorCode::InvalidArgument, "kernel requires an ELL handle");
  if (k0 < 0 || k1 > m.band_count || k0 > k1)
    throw Error(ErrorCode::InvalidArgument, "band range out of bounds");
  const std::int64_t bands = k1 - k0, len = bands * m.n;
  if (len == 0) return;
  cudaStream_t st = rt::stream();
  if (values)
    rt::check(cudaMemcpy2DAsync(values, m.n * 8, m.val.get() + k0 * m.ld, m.ld * 8, m.n * 8, bands,
                                cudaMemcpyDeviceToHost, st),
              "ELL band export");
  if (col_idx) {
    DevArray<std::int32_t> compact(static_cast<std::size_t>(len), "ELL band export");
    rt::check(cudaMemcpy2DAsync(compact.get(), m.n * 4, m.col.get() + k0 * m.ld, m.ld * 4, m.n * 4,
                                bands, cudaMemcpyDeviceToDevice, st),
              "ELL band export");
    DevArray<std::int64_t> wide(static_cast<std::size_t>(len), "ELL band export");
    rt::check_launch(spmvtk_k_widen_index(compact.get(), wide.get(), len, index_base, st),
                     "ELL band export");
    rt::copy_to_host(col_idx, wide.get(), static_cast<std::size_t>(len) * 8);
  }
  rt::sync();
}

}  // namespace spmvtk::dev
