/* spmv_capi.c -- the C ABI from plain C (C11), as a reference user would
 * call it after swapping libspmvtk.so: generate, convert, multiply, profile,
 * select.  Prints "ok" and exits 0 when every product matches CRS.
 *
 *   cc -std=c11 -I include examples/spmv_capi.c \
 *      -L paper_2407_00019_b200 -lspmvtk -Wl,-rpath,paper_2407_00019_b200 -lm
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "spmvtk/spmvtk.h"

#define CHECK(call)                                                            \
  do {                                                                         \
    spmvtk_status st_ = (call);                                                \
    if (st_ != SPMVTK_OK) {                                                    \
      fprintf(stderr, "%s failed (%d): %s\n", #call, (int)st_, spmvtk_last_error()); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

int main(void) {
  const int64_t n = 20000;
  spmvtk_matrix* crs = NULL;
  CHECK(spmvtk_gen_cv_target(n, 12.0, 0.3, 7, &crs));
  spmvtk_matrix_info info;
  CHECK(spmvtk_matrix_get_info(crs, &info));
  printf("n=%lld nnz=%lld max_row=%lld d_mat=%.4f\n", (long long)info.n, (long long)info.nnz,
         (long long)info.max_row_entries, info.d_mat);

  double* x = malloc(sizeof(double) * n);
  double* y0 = malloc(sizeof(double) * n);
  double* y1 = malloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; ++i) x[i] = sin((double)i);
  double secs = 0.0;
  CHECK(spmvtk_spmv(crs, SPMVTK_KERNEL_CRS, x, n, 1, y0, &secs));

  const struct { spmvtk_format f; spmvtk_kernel k; const char* name; } forms[] = {
      {SPMVTK_FORMAT_COO_ROW, SPMVTK_KERNEL_COO_ROW_OUTER, "coo-row"},
      {SPMVTK_FORMAT_COO_COL, SPMVTK_KERNEL_COO_COL_OUTER, "coo-col"},
      {SPMVTK_FORMAT_ELL, SPMVTK_KERNEL_ELL_INNER, "ell-inner"},
      {SPMVTK_FORMAT_ELL, SPMVTK_KERNEL_ELL_OUTER, "ell-outer"},
  };
  for (size_t j = 0; j < sizeof(forms) / sizeof(forms[0]); ++j) {
    spmvtk_matrix* h = NULL;
    CHECK(spmvtk_matrix_convert(crs, forms[j].f, 0, &h));
    CHECK(spmvtk_spmv(h, forms[j].k, x, n, 4, y1, &secs));
    double num = 0.0, den = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      num = fmax(num, fabs(y1[i] - y0[i]));
      den = fmax(den, fabs(y0[i]));
    }
    printf("%-10s rel.err %.2e  %.1f us\n", forms[j].name, num / den, secs * 1e6);
    if (num > 1e-12 * den) return 2;
    spmvtk_matrix_free(h);
  }

  /* off-line AT over the one matrix, then the on-line decision */
  const spmvtk_matrix* set[1] = {crs};
  const char* ids[1] = {"cv"};
  spmvtk_profile* prof = NULL;
  CHECK(spmvtk_profile_build(set, ids, 1, SPMVTK_KERNEL_ELL_INNER, 1, 1.0, 5, 0, "example", &prof));
  spmvtk_decision d;
  double dm = 0.0;
  CHECK(spmvtk_select(crs, prof, &d, &dm));
  printf("d_star=%.4f decision=%s\n", spmvtk_profile_d_star(prof),
         d == SPMVTK_USE_ELL ? "UseEll" : "UseCrs");
  spmvtk_profile_free(prof);
  spmvtk_matrix_free(crs);
  free(x);
  free(y0);
  free(y1);
  printf("ok\n");
  return 0;
}
