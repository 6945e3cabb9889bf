// ref_shim.cpp -- array-level C entry points into the REFERENCE library.
//
// TEST INFRASTRUCTURE ONLY (oracle).  Compiled by oracle/Makefile together
// with the unmodified reference sources from /root/reference/proj/src into
// oracle/_ref/libspmvtk_ref.so, with -Dspmvtk=spmvtk_ref so the reference's
// C++ symbols live in namespace spmvtk_ref.  The reference's own C ABI
// (capi.cpp, spmvtk.h:50-160) is linked in unchanged; it cannot build a
// matrix from raw arrays nor read arrays back, so this shim
// adds exactly that: ref_matrix_from_crs() and ref_matrix_get_array().
// It also exposes the reference timing protocol (autotune.cpp:95-128) for
// bench.py's cpu_baseline / --impl reference legs.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <variant>
#include <vector>

#include "spmvtk/autotune.hpp"
#include "spmvtk/convert.hpp"
#include "spmvtk/error.hpp"
#include "spmvtk/formats.hpp"
#include "spmvtk/spmv.hpp"
#include "spmvtk/spmvtk.h"
#include "spmvtk/stats.hpp"
#include "../paper_2407_00019_b200/csrc/generators.hpp"

using namespace spmvtk;  // -> spmvtk_ref

// Same definition as the reference capi.cpp:23-25 so handles made here are
// released by the reference's own spmvtk_matrix_free().
struct spmvtk_matrix {
  std::variant<CrsMatrix, CcsMatrix, CooMatrix, EllMatrix> data;
};

namespace {
thread_local std::string g_err;

template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    g_err.clear();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    switch (e.code()) {
      case ErrorCode::InvalidArgument: return 1;
      case ErrorCode::MemoryLimit: return 4;
      default: return 2;
    }
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// row_ptr / col_idx are int64, 1-based (the reference layout).
int ref_matrix_from_crs(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                        const double* values, spmvtk_matrix** out) {
  return guard([&] {
    CrsMatrix m;
    m.n = n;
    int64_t nnz = row_ptr[n] - 1;
    m.row_ptr.assign(row_ptr, row_ptr + n + 1);
    m.col_idx.assign(col_idx, col_idx + nnz);
    m.values.assign(values, values + nnz);
    *out = new spmvtk_matrix{std::move(m)};
  });
}

// which: 0 values, 1 pointer (row_ptr/col_ptr), 2 row_idx, 3 col_idx,
//        4 row_entry_count (ELL).  Returns the element count in *len; when
// dst is non-null copies the array (int64 for index arrays).
// meta: [n, nnz, band_count, stored_nnz, ordering(0 row,1 col,2 unordered)]
int ref_matrix_meta(const spmvtk_matrix* m, int64_t* meta) {
  return guard([&] {
    std::visit(
        [&](const auto& a) {
          using T = std::decay_t<decltype(a)>;
          meta[0] = a.n;
          meta[2] = 0;
          meta[3] = 0;
          meta[4] = -1;
          if constexpr (std::is_same_v<T, EllMatrix>) {
            meta[1] = a.stored_nnz;
            meta[2] = a.band_count;
            meta[3] = a.stored_nnz;
          } else {
            meta[1] = static_cast<int64_t>(a.values.size());
          }
          if constexpr (std::is_same_v<T, CooMatrix>)
            meta[4] = a.ordering == CooOrdering::RowMajor   ? 0
                      : a.ordering == CooOrdering::ColMajor ? 1
                                                            : 2;
        },
        m->data);
  });
}

int ref_matrix_get_array(const spmvtk_matrix* m, int which, void* dst,
                         int64_t* len) {
  return guard([&] {
    const std::vector<double>* dv = nullptr;
    const std::vector<index_t>* iv = nullptr;
    std::visit(
        [&](const auto& a) {
          using T = std::decay_t<decltype(a)>;
          if (which == 0) dv = &a.values;
          if constexpr (std::is_same_v<T, CrsMatrix>) {
            if (which == 1) iv = &a.row_ptr;
            if (which == 3) iv = &a.col_idx;
          } else if constexpr (std::is_same_v<T, CcsMatrix>) {
            if (which == 1) iv = &a.col_ptr;
            if (which == 2) iv = &a.row_idx;
          } else if constexpr (std::is_same_v<T, CooMatrix>) {
            if (which == 2) iv = &a.row_idx;
            if (which == 3) iv = &a.col_idx;
          } else {
            if (which == 3) iv = &a.col_idx;
            if (which == 4) iv = &a.row_entry_count;
          }
        },
        m->data);
    if (dv) {
      *len = static_cast<int64_t>(dv->size());
      if (dst) std::memcpy(dst, dv->data(), dv->size() * sizeof(double));
    } else if (iv) {
      *len = static_cast<int64_t>(iv->size());
      if (dst) std::memcpy(dst, iv->data(), iv->size() * sizeof(int64_t));
    } else {
      throw Error(ErrorCode::InvalidArgument, "array not present in this format");
    }
  });
}

// Reference timing protocol on a CRS handle (autotune.cpp:95-120): one
// untimed warm-up then the median of `repeats` wall-clock calls.  x = ones
// as in autotune.cpp:183.  kernel uses the spmvtk_kernel numbering; the
// handle must already be in the kernel's format.
int ref_measure_spmv(const spmvtk_matrix* m, int kernel, int lanes,
                     int repeats, double* seconds) {
  return guard([&] {
    std::vector<double> x;
    MatrixRef ref = static_cast<const CrsMatrix*>(nullptr);
    std::visit(
        [&](const auto& a) {
          using T = std::decay_t<decltype(a)>;
          x.assign(static_cast<std::size_t>(a.n), 1.0);
          if constexpr (std::is_same_v<T, CrsMatrix>) ref = &a;
          else if constexpr (std::is_same_v<T, CooMatrix>) ref = &a;
          else if constexpr (std::is_same_v<T, EllMatrix>) ref = &a;
          else throw Error(ErrorCode::InvalidArgument, "no kernel for CCS");
        },
        m->data);
    *seconds = measure_spmv(static_cast<Kernel>(kernel), ref, x, lanes, repeats);
  });
}

// One cold conversion timed with the wall clock as the reference does
// (autotune.cpp:122-128 for ELL, :197-214 for the COO variants).
int ref_measure_transformation(const spmvtk_matrix* m, int format,
                               uint64_t max_bytes, double* seconds,
                               spmvtk_matrix** out) {
  return guard([&] {
    const auto* crs = std::get_if<CrsMatrix>(&m->data);
    if (!crs) throw Error(ErrorCode::InvalidArgument, "needs CRS");
    auto t0 = std::chrono::steady_clock::now();
    std::variant<CrsMatrix, CcsMatrix, CooMatrix, EllMatrix> res;
    switch (format) {
      case SPMVTK_FORMAT_CCS: res = crs_to_ccs(*crs); break;
      case SPMVTK_FORMAT_COO_ROW: res = crs_to_coo_row(*crs); break;
      case SPMVTK_FORMAT_COO_COL: res = crs_to_coo_col(*crs); break;
      case SPMVTK_FORMAT_ELL: res = crs_to_ell(*crs, max_bytes); break;
      default: throw Error(ErrorCode::InvalidArgument, "bad format");
    }
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (out) *out = new spmvtk_matrix{std::move(res)};
  });
}

int ref_row_stats(const spmvtk_matrix* m, double* mu, double* sigma,
                  double* d_mat) {
  return guard([&] {
    const auto* crs = std::get_if<CrsMatrix>(&m->data);
    if (!crs) throw Error(ErrorCode::InvalidArgument, "needs CRS");
    RowStats s = row_stats(*crs);
    *mu = s.mu;
    *sigma = s.sigma;
    *d_mat = s.d_mat;
  });
}

int ref_stats_from_counts(int64_t n, const int64_t* counts, double* mu,
                          double* sigma, double* d_mat) {
  return guard([&] {
    RowHistogram h;
    h.counts.assign(counts, counts + n);
    RowStats s = stats_from_histogram(h);
    *mu = s.mu;
    *sigma = s.sigma;
    *d_mat = s.d_mat;
  });
}

uint64_t ref_estimate_ell_bytes(const spmvtk_matrix* m, int vb, int ib) {
  const auto* crs = std::get_if<CrsMatrix>(&m->data);
  return crs ? estimate_ell_bytes(*crs, vb, ib) : 0;
}

double ref_find_d_star(size_t count, const double* d_mat, const double* r,
                       double c) {
  std::vector<std::pair<double, double>> v;
  for (size_t i = 0; i < count; ++i) v.emplace_back(d_mat[i], r[i]);
  return find_d_star(std::span<const std::pair<double, double>>(v), c);
}

int64_t ref_amortization(double t_crs, double t_ell, double t_trans) {
  int64_t out = -2;
  guard([&] {
    auto k = amortization_iterations(Timings{t_crs, t_ell, t_trans});
    out = k ? *k : -1;
  });
  return out;
}

// A BASELINE workload (gen::baseline, int32 0-based) as a reference CRS
// handle (int64 1-based), for bench.py's reference arm.
int ref_gen_baseline(int config, int64_t param, double dparam, uint64_t seed,
                     spmvtk_matrix** out) {
  return guard([&] {
    gen::HostCrs h = gen::baseline(config, param, dparam, seed);
    CrsMatrix m;
    m.n = h.n;
    m.row_ptr.resize(static_cast<std::size_t>(h.n) + 1);
    m.col_idx.resize(h.values.size());
    if (h.wide()) {
      for (std::size_t i = 0; i < m.row_ptr.size(); ++i) m.row_ptr[i] = h.row_ptr[i] - h.base + 1;
      for (std::size_t p = 0; p < m.col_idx.size(); ++p) m.col_idx[p] = h.col_idx[p] - h.base + 1;
    } else {
      for (std::size_t i = 0; i < m.row_ptr.size(); ++i) m.row_ptr[i] = h.row_ptr32[i] - h.base + 1;
      for (std::size_t p = 0; p < m.col_idx.size(); ++p) m.col_idx[p] = h.col32[p] - h.base + 1;
    }
    m.values = std::move(h.values);
    *out = new spmvtk_matrix{std::move(m)};
  });
}

int ref_gen_vector(int64_t n, uint64_t seed, double* out) {
  return guard([&] { gen::vector_u11(n, seed, out); });
}

int ref_partition_range(int64_t len, int lanes, int64_t* istart, int64_t* iend) {
  return guard([&] {
    ThreadPartition p = partition_range(len, lanes);
    for (int k = 0; k < lanes; ++k) {
      istart[k] = p.istart[k];
      iend[k] = p.iend[k];
    }
  });
}

}  // extern "C"
