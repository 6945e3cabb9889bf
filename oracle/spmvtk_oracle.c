/*
 * spmvtk_oracle.c -- CPU restatement of the reference transform / SpMV /
 * auto-tuning arithmetic (arXiv 2407.00019, "spmvtk").
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2407_00019_b200/ links, loads
 * or calls this file; only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py do, and only as the checker.
 *
 * Conventions follow the reference exactly so its outputs can be compared
 * array-for-array: indices and pointers are 1-based int64
 * (/root/reference/proj/include/spmvtk/formats.hpp:10-14), ELL is band-major
 * with slot(k,i) = n*(k-1) + (i-1) (formats.hpp:46-61).  Each function names
 * the reference file:line it restates.  Lanes are emulated sequentially:
 * every lane writes its own partial column and the reduction order is the
 * reference's, so results are identical to the threaded reference.
 *
 * Pinned by tests/test_oracle.py against the reference's own known-answer
 * tests (tests/golden/kat.json) and against the reference compiled from
 * /root/reference (oracle/_ref, see oracle/Makefile).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t idx_t;

/* ---- stats: proj/src/stats.cpp:9-29 (Welford, population sigma) -------- */
/* returns 0 on success, 1 when mu == 0 (reference throws InvalidArgument,
 * stats.cpp:10-11,21-23) */
int or_row_stats(idx_t n, const idx_t* row_ptr, double* mu, double* sigma,
                 double* d_mat) {
  if (n <= 0) return 1;
  double mean = 0.0, m2 = 0.0;
  for (idx_t i = 0; i < n; ++i) {
    double c = (double)(row_ptr[i + 1] - row_ptr[i]);
    double k = (double)(i + 1);
    double delta = c - mean;
    mean += delta / k;
    m2 += delta * (c - mean);
  }
  if (mean == 0.0) return 1;
  *mu = mean;
  *sigma = sqrt(m2 / (double)n);
  *d_mat = *sigma / *mu;
  return 0;
}

/* max row length: convert.cpp:74-76 / :91-96 */
idx_t or_max_row(idx_t n, const idx_t* row_ptr) {
  idx_t m = 0;
  for (idx_t i = 0; i < n; ++i) {
    idx_t r = row_ptr[i + 1] - row_ptr[i];
    if (r > m) m = r;
  }
  return m;
}

/* estimate_ell_bytes: convert.cpp:72-79 */
uint64_t or_estimate_ell_bytes(idx_t n, const idx_t* row_ptr, int value_bytes,
                               int index_bytes) {
  return (uint64_t)n * (uint64_t)or_max_row(n, row_ptr) *
         (uint64_t)(value_bytes + index_bytes);
}

/* ---- crs_to_coo_row: convert.cpp:11-22 -------------------------------- */
void or_crs_to_coo_row(idx_t n, const idx_t* row_ptr, const idx_t* col_idx,
                       const double* val, idx_t* out_row, idx_t* out_col,
                       double* out_val) {
  idx_t nnz = row_ptr[n] - 1;
  memcpy(out_val, val, (size_t)nnz * sizeof(double));
  memcpy(out_col, col_idx, (size_t)nnz * sizeof(idx_t));
  for (idx_t i = 1; i <= n; ++i)
    for (idx_t p = row_ptr[i - 1]; p < row_ptr[i]; ++p) out_row[p - 1] = i;
}

/* ---- crs_to_ccs (Phase I): convert.cpp:24-53 ----------------------------
 * count, exclusive prefix, scatter with per-column cursors scanning CRS rows
 * in order (so row indices ascend inside every column). */
void or_crs_to_ccs(idx_t n, const idx_t* row_ptr, const idx_t* col_idx,
                   const double* val, idx_t* out_col_ptr, idx_t* out_row,
                   double* out_val) {
  idx_t nnz = row_ptr[n] - 1;
  idx_t* next = (idx_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(idx_t));
  for (idx_t p = 0; p < nnz; ++p) next[col_idx[p] - 1]++;
  out_col_ptr[0] = 1;
  for (idx_t j = 1; j <= n; ++j) out_col_ptr[j] = out_col_ptr[j - 1] + next[j - 1];
  for (idx_t j = 0; j < n; ++j) next[j] = out_col_ptr[j];
  for (idx_t i = 1; i <= n; ++i)
    for (idx_t p = row_ptr[i - 1]; p < row_ptr[i]; ++p) {
      idx_t slot = next[col_idx[p - 1] - 1]++;
      out_val[slot - 1] = val[p - 1];
      out_row[slot - 1] = i;
    }
  free(next);
}

/* ---- ccs_to_coo_col (Phase II): convert.cpp:55-66 ---------------------- */
void or_ccs_to_coo_col(idx_t n, const idx_t* col_ptr, const idx_t* row_idx,
                       const double* val, idx_t* out_row, idx_t* out_col,
                       double* out_val) {
  idx_t nnz = col_ptr[n] - 1;
  memcpy(out_val, val, (size_t)nnz * sizeof(double));
  memcpy(out_row, row_idx, (size_t)nnz * sizeof(idx_t));
  for (idx_t j = 1; j <= n; ++j)
    for (idx_t p = col_ptr[j - 1]; p < col_ptr[j]; ++p) out_col[p - 1] = j;
}

/* ---- crs_to_ell: convert.cpp:81-115 -------------------------------------
 * Returns 0, or 4 (MemoryLimit) when max_bytes != 0 and the 8+8 byte
 * estimate exceeds it (convert.cpp:82-88).  Outputs are band-major with
 * n*band_count slots; padding is value +0.0 and column = own row. */
int or_crs_to_ell(idx_t n, const idx_t* row_ptr, const idx_t* col_idx,
                  const double* val, uint64_t max_bytes, idx_t band_count,
                  double* out_val, idx_t* out_col, idx_t* out_count) {
  if (max_bytes != 0 && or_estimate_ell_bytes(n, row_ptr, 8, 8) > max_bytes)
    return 4;
  for (idx_t i = 1; i <= n; ++i) {
    idx_t r = row_ptr[i] - row_ptr[i - 1];
    out_count[i - 1] = r;
    for (idx_t k = 1; k <= band_count; ++k) {
      size_t s = (size_t)(n * (k - 1) + (i - 1));
      if (k <= r) {
        size_t p = (size_t)(row_ptr[i - 1] - 1 + k - 1);
        out_val[s] = val[p];
        out_col[s] = col_idx[p];
      } else {
        out_val[s] = 0.0;
        out_col[s] = i;
      }
    }
  }
  return 0;
}

/* Bands [k0, k1) (1-based k) of crs_to_ell's band-major arrays, the same
 * fill as convert.cpp:101-113 restricted to those bands: out has
 * (k1 - k0) * n slots, band k at offset (k - k0) * n.  Lets a test compare
 * an ELL too large for host memory band by band. */
void or_crs_to_ell_bands(idx_t n, const idx_t* row_ptr, const idx_t* col_idx,
                         const double* val, idx_t k0, idx_t k1, double* out_val,
                         idx_t* out_col) {
  for (idx_t i = 1; i <= n; ++i) {
    idx_t r = row_ptr[i] - row_ptr[i - 1];
    for (idx_t k = k0; k < k1; ++k) {
      size_t s = (size_t)(n * (k - k0) + (i - 1));
      if (k <= r) {
        size_t p = (size_t)(row_ptr[i - 1] - 1 + k - 1);
        out_val[s] = val[p];
        out_col[s] = col_idx[p];
      } else {
        out_val[s] = 0.0;
        out_col[s] = i;
      }
    }
  }
}

/* Row-major ELL has no reference counterpart: its oracle is
 * the transpose of the band-major arrays, same padding rules. */
void or_ell_to_rowmajor(idx_t n, idx_t band_count, const double* bm_val,
                        const idx_t* bm_col, double* rm_val, idx_t* rm_col) {
  for (idx_t i = 0; i < n; ++i)
    for (idx_t k = 0; k < band_count; ++k) {
      rm_val[(size_t)(i * band_count + k)] = bm_val[(size_t)(k * n + i)];
      rm_col[(size_t)(i * band_count + k)] = bm_col[(size_t)(k * n + i)];
    }
}

/* ---- partition_range: spmv.cpp:36-54 ----------------------------------- */
int or_partition_range(idx_t len, int lanes, idx_t* istart, idx_t* iend) {
  if (lanes < 1) return 1;
  idx_t base = len / lanes, rem = len % lanes, pos = 1;
  for (int k = 0; k < lanes; ++k) {
    idx_t size = base + (k < rem ? 1 : 0);
    istart[k] = pos;
    iend[k] = pos + size - 1;
    pos += size;
  }
  return 0;
}

/* ---- reduce_partials: spmv.cpp:56-62 (ascending lanes) ----------------- */
void or_reduce_partials(idx_t n, int lanes, const double* yy, double* y) {
  for (idx_t i = 0; i < n; ++i) y[i] = 0.0;
  for (int k = 0; k < lanes; ++k)
    for (idx_t i = 0; i < n; ++i) y[i] += yy[(size_t)k * (size_t)n + (size_t)i];
}

/* ---- spmv_crs: spmv.cpp:64-75 (left-to-right, no FMA contraction) ----- */
void or_spmv_crs(idx_t n, const idx_t* row_ptr, const idx_t* col_idx,
                 const double* val, const double* x, double* y) {
  for (idx_t i = 1; i <= n; ++i) {
    double acc = 0.0;
    for (idx_t p = row_ptr[i - 1]; p < row_ptr[i]; ++p) {
      double prod = val[p - 1] * x[col_idx[p - 1] - 1];
      acc += prod;
    }
    y[i - 1] = acc;
  }
}

/* ---- spmv_coo_outer: spmv.cpp:79-101 -----------------------------------
 * Ordering is checked by the caller (spmv.cpp:82-84). */
void or_spmv_coo_outer(idx_t n, idx_t nnz, const idx_t* row, const idx_t* col,
                       const double* val, const double* x, int lanes,
                       double* y) {
  idx_t* is = (idx_t*)malloc(sizeof(idx_t) * (size_t)lanes);
  idx_t* ie = (idx_t*)malloc(sizeof(idx_t) * (size_t)lanes);
  double* yy = (double*)calloc((size_t)lanes * (size_t)(n > 0 ? n : 1), sizeof(double));
  or_partition_range(nnz, lanes, is, ie);
  for (int k = 0; k < lanes; ++k)
    for (idx_t p = is[k]; p <= ie[k]; ++p) {
      double prod = val[p - 1] * x[col[p - 1] - 1];
      yy[(size_t)k * (size_t)n + (size_t)(row[p - 1] - 1)] += prod;
    }
  or_reduce_partials(n, lanes, yy, y);
  free(is);
  free(ie);
  free(yy);
}

/* ---- spmv_ell_inner: spmv.cpp:117-136 (bands serial, rows split) ------- */
void or_spmv_ell_inner(idx_t n, idx_t band_count, const double* val,
                       const idx_t* col, const double* x, double* y) {
  for (idx_t i = 0; i < n; ++i) y[i] = 0.0;
  for (idx_t b = 1; b <= band_count; ++b) {
    idx_t base = n * (b - 1);
    for (idx_t i = 1; i <= n; ++i) {
      size_t s = (size_t)(base + i - 1);
      double prod = val[s] * x[col[s] - 1];
      y[i - 1] += prod;
    }
  }
}

/* ---- spmv_ell_outer: spmv.cpp:138-158 (bands split, serial reduce) ----- */
void or_spmv_ell_outer(idx_t n, idx_t band_count, const double* val,
                       const idx_t* col, const double* x, int lanes,
                       double* y) {
  idx_t* is = (idx_t*)malloc(sizeof(idx_t) * (size_t)lanes);
  idx_t* ie = (idx_t*)malloc(sizeof(idx_t) * (size_t)lanes);
  double* yy = (double*)calloc((size_t)lanes * (size_t)(n > 0 ? n : 1), sizeof(double));
  or_partition_range(band_count, lanes, is, ie);
  for (int k = 0; k < lanes; ++k)
    for (idx_t b = is[k]; b <= ie[k]; ++b) {
      idx_t base = n * (b - 1);
      for (idx_t i = 1; i <= n; ++i) {
        size_t s = (size_t)(base + i - 1);
        double prod = val[s] * x[col[s] - 1];
        yy[(size_t)k * (size_t)n + (size_t)(i - 1)] += prod;
      }
    }
  or_reduce_partials(n, lanes, yy, y);
  free(is);
  free(ie);
  free(yy);
}

/* ---- compute_metrics: autotune.cpp:36-44 (tt = t_trans / t_crs) -------- */
int or_compute_metrics(double t_crs, double t_ell, double t_trans, double* sp,
                       double* tt, double* r) {
  if (t_crs <= 0.0 || t_ell <= 0.0 || t_trans <= 0.0) return 1;
  *sp = t_crs / t_ell;
  *tt = t_trans / t_crs;
  *r = *sp / *tt;
  return 0;
}

/* ---- amortization_iterations: autotune.cpp:46-60 ------------------------
 * returns -1 for "none" (t_ell >= t_crs), -2 for invalid timings. */
int64_t or_amortization(double t_crs, double t_ell, double t_trans) {
  if (t_crs <= 0.0 || t_ell <= 0.0 || t_trans <= 0.0) return -2;
  if (t_ell >= t_crs) return -1;
  int64_t k = (int64_t)ceil(t_trans / (t_crs - t_ell));
  while (k > 1 && t_trans + (double)(k - 1) * t_ell <= (double)(k - 1) * t_crs)
    --k;
  while (t_trans + (double)k * t_ell > (double)k * t_crs) ++k;
  return k;
}

/* ---- find_d_star: autotune.cpp:130-150 ----------------------------------
 * conservative prefix rule: walk records by ascending d_mat; a tie group
 * qualifies only if every member has r >= c; stop at the first failure. */
static int cmp_first(const void* a, const void* b) {
  double x = ((const double*)a)[0], y = ((const double*)b)[0];
  return (x > y) - (x < y);
}

double or_find_d_star(size_t count, const double* d_mat, const double* r,
                      double c) {
  double* pts = (double*)malloc(sizeof(double) * 2 * (count ? count : 1));
  for (size_t i = 0; i < count; ++i) {
    pts[2 * i] = d_mat[i];
    pts[2 * i + 1] = r[i];
  }
  qsort(pts, count, 2 * sizeof(double), cmp_first);
  double d_star = 0.0;
  size_t i = 0;
  while (i < count) {
    size_t j = i;
    int all_pass = 1;
    while (j < count && pts[2 * j] == pts[2 * i]) {
      if (pts[2 * j + 1] < c) all_pass = 0;
      ++j;
    }
    if (!all_pass) break;
    d_star = pts[2 * i];
    i = j;
  }
  free(pts);
  return d_star;
}
