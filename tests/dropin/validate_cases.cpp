// validate() on a battery of malformed matrices, every message printed: the
// same source is built against the reference library (-Dspmvtk=spmvtk_ref)
// and against this repository's (GPU validation, kernels_validate.cu), and
// tests/test_dropin.py compares the two outputs line for line.
#include <cstdio>
#include <string>
#include <vector>

#include "spmvtk/formats.hpp"

using namespace spmvtk;

static void show(const char* name, const std::vector<std::string>& v) {
  std::printf("== %s (%zu)\n", name, v.size());
  for (const auto& s : v) std::printf("%s\n", s.c_str());
}

static CrsMatrix crs(index_t n, std::vector<double> v, std::vector<index_t> c,
                     std::vector<index_t> p) {
  CrsMatrix m;
  m.n = n;
  m.values = std::move(v);
  m.col_idx = std::move(c);
  m.row_ptr = std::move(p);
  return m;
}

int main() {
  show("crs ok", validate(crs(2, {1, 1}, {1, 2}, {1, 2, 3})));
  show("crs descent", validate(crs(3, {1, 1}, {1, 2}, {1, 3, 2, 3})));
  show("crs range", validate(crs(3, {1, 1, 1, 1}, {0, 5, 2, -7}, {1, 3, 4, 5})));
  show("crs dup", validate(crs(3, {1, 1, 1, 1, 1, 1}, {2, 2, 1, 3, 3, 3}, {1, 3, 4, 7})));
  show("crs lengths", validate(crs(2, {1, 1, 1}, {1, 2}, {1, 2, 3})));
  show("crs ptr len", validate(crs(3, {1, 1}, {1, 2}, {1, 3})));
  show("crs ptr ends", validate(crs(2, {1, 1}, {1, 2}, {2, 2, 4})));
  show("crs negative", validate(crs(-1, {}, {}, {1})));
  {
    std::vector<double> v(3000, 1.0);
    std::vector<index_t> c, p = {1};
    for (int r = 0; r < 30; ++r) {
      for (int k = 0; k < 100; ++k) c.push_back(1 + (k * 7 + r) % (r < 5 ? 13 : 97));
      p.push_back(static_cast<index_t>(c.size()) + 1);
    }
    while (p.size() < 101) p.push_back(p.back());  // rows 31..100 empty
    show("crs many dups", validate(crs(100, v, c, p)));
  }
  CcsMatrix s;
  s.n = 3;
  s.values = {1, 1, 1, 1};
  s.row_idx = {1, 1, 4, 2};
  s.col_ptr = {1, 3, 4, 5};
  show("ccs dup+range", validate(s));
  s.row_idx = {1, 1, 3, 2};
  show("ccs dup", validate(s));
  CooMatrix t;
  t.n = 3;
  t.values = {1, 1, 1, 1, 1};
  t.row_idx = {1, 2, 1, 3, 1};
  t.col_idx = {2, 1, 2, 3, 2};
  t.ordering = CooOrdering::RowMajor;
  show("coo dups+order", validate(t));
  t.ordering = CooOrdering::ColMajor;
  show("coo col order", validate(t));
  t.ordering = CooOrdering::Unordered;
  t.row_idx = {1, 2, 5, 3, 0};
  show("coo range", validate(t));
  t.values.pop_back();
  show("coo lengths", validate(t));
  EllMatrix e;
  e.n = 3;
  e.band_count = 2;
  e.values = {1, 2, 3, 0, 5, 0};
  e.col_idx = {1, 2, 3, 1, 2, 3};
  e.row_entry_count = {1, 2, 1};
  e.stored_nnz = 4;
  show("ell ok", validate(e));
  e.values = {1, 2, 3, 9, 5, 8};
  e.col_idx = {1, 2, 3, 3, 2, 1};
  e.row_entry_count = {1, 7, 1};
  e.stored_nnz = 3;
  show("ell padding", validate(e));
  e.col_idx = {1, 2, 4, 3, 2, 1};
  e.row_entry_count = {0, 0, 0};
  show("ell counts", validate(e));
  e.values.pop_back();
  show("ell lengths", validate(e));
  return 0;
}
