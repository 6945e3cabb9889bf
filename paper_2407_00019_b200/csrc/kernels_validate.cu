// kernels_validate.cu -- the reference's structural validation
// (formats.cpp:75-182, the messages its tests grep for) done on the GPU.
//
// The arrays of a CrsMatrix / CcsMatrix / CooMatrix / EllMatrix (1-based
// int64, host) are uploaded once; every O(nnz) check is a device pass that
// reports offending positions, and the host turns them into the reference's
// messages in the reference's order (ascending position):
//   * pointer arrays: first descent (one atomicMin);
//   * index ranges: every out-of-range position (device append, host sort);
//   * duplicates inside a segment / matrix: a device hash table keyed by
//     (segment, index) keeps each key's first position (atomicMin); every
//     later occurrence is reported -- the same set the reference's per-row
//     unordered_set walk reports;
//   * ELL: entry counts, padding values and padding columns per slot.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "common.cuh"
#include "runtime.hpp"
#include "spmvtk/error.hpp"
#include "validate.hpp"

using namespace spmvtk_dev;

namespace {

constexpr unsigned long long kEmpty = ~0ull;

__device__ __forceinline__ void append(unsigned long long* count, int64_t* list, int64_t cap,
                                       int64_t v) {
  const unsigned long long k = atomicAdd(count, 1ull);
  if (static_cast<int64_t>(k) < cap) list[k] = v;
}

// first i in [1, len) with a[i] < a[i-1] (len if none)
__global__ void k_first_descent(const int64_t* __restrict__ a, int64_t len,
                                unsigned long long* first) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x + 1; i < len;
       i += stride)
    if (a[i] < a[i - 1]) atomicMin(first, static_cast<unsigned long long>(i));
}

// positions p with a[p] outside [lo, hi]
__global__ void k_out_of_range(const int64_t* __restrict__ a, int64_t len, int64_t lo, int64_t hi,
                               int64_t* list, int64_t cap, unsigned long long* count) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < len;
       p += stride)
    if (a[p] < lo || a[p] > hi) append(count, list, cap, p);
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// key of entry p: (segment, index) or (row, col), as one 64-bit value
struct SegKey {
  const int64_t* ptr;  // 1-based segment pointers, nseg + 1 (NULL: COO pairs)
  int64_t nseg;
  const int64_t* a;    // index (segments) / row (pairs)
  const int64_t* b;    // column (pairs)
  int64_t n;
  __device__ uint64_t operator()(int64_t p) const {
    if (ptr) {  // segment of p: the last s with ptr[s] - 1 <= p
      int64_t lo = 0, hi = nseg - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (ptr[mid] - 1 <= p) lo = mid;
        else hi = mid - 1;
      }
      return static_cast<uint64_t>(lo) * static_cast<uint64_t>(n + 1) + static_cast<uint64_t>(a[p]);
    }
    return static_cast<uint64_t>(a[p]) * static_cast<uint64_t>(n + 1) + static_cast<uint64_t>(b[p]);
  }
};

// pass 1: insert every key, keeping its smallest position
__global__ void k_dup_insert(SegKey key, int64_t len, unsigned long long* keys,
                             unsigned long long* first, uint64_t mask) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < len;
       p += stride) {
    const unsigned long long k = key(p);
    uint64_t h = mix64(k) & mask;
    while (true) {
      const unsigned long long prev = atomicCAS(keys + h, kEmpty, k);
      if (prev == kEmpty || prev == k) {
        atomicMin(first + h, static_cast<unsigned long long>(p));
        break;
      }
      h = (h + 1) & mask;
    }
  }
}

// pass 2: every position that is not its key's first is a duplicate
__global__ void k_dup_report(SegKey key, int64_t len, const unsigned long long* keys,
                             const unsigned long long* first, uint64_t mask, int64_t* list,
                             int64_t cap, unsigned long long* count) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < len;
       p += stride) {
    const unsigned long long k = key(p);
    uint64_t h = mix64(k) & mask;
    while (keys[h] != k) h = (h + 1) & mask;
    if (first[h] != static_cast<unsigned long long>(p)) append(count, list, cap, p);
  }
}

// ELL: rows with an out-of-range count (list 0), padding slots with a
// nonzero value (list 1) or a column other than the row (list 2); slots are
// reported as (i - 1) * band_count + (k - 1), i.e. in the reference's
// row-then-band order
__global__ void k_ell_padding(int64_t n, int64_t bc, const int64_t* __restrict__ cnt,
                              const double* __restrict__ val, const int64_t* __restrict__ col,
                              int64_t* l0, int64_t* l1, int64_t* l2, int64_t cap,
                              unsigned long long* counts) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const int64_t r = cnt[i];
    if (r < 0 || r > bc) {
      append(counts + 0, l0, cap, i);
      continue;
    }
    for (int64_t k = r; k < bc; ++k) {  // 0-based bands past the row's entries
      const int64_t s = k * n + i;
      if (val[s] != 0.0) append(counts + 1, l1, cap, i * bc + k);
      if (col[s] != i + 1) append(counts + 2, l2, cap, i * bc + k);
    }
  }
}

int blocks_for(int64_t len) { return grid_for(std::max<int64_t>(len, 1), 256, 8); }

using spmvtk::rt::DevArray;

template <typename T>
DevArray<T> upload(const std::vector<T>& v) {
  DevArray<T> d(std::max<std::size_t>(v.size(), 1), "validation upload");
  if (!v.empty()) spmvtk::rt::copy_to_device(d.get(), v.data(), v.size() * sizeof(T));
  return d;
}

std::vector<int64_t> fetch_list(const DevArray<int64_t>& list, const DevArray<unsigned long long>& count,
                                int which = 0) {
  unsigned long long c = 0;
  spmvtk::rt::copy_to_host(&c, count.get() + which, sizeof(c));
  std::vector<int64_t> out(static_cast<std::size_t>(std::min<unsigned long long>(c, list.size())));
  if (!out.empty()) spmvtk::rt::copy_to_host(out.data(), list.get(), out.size() * 8);
  std::sort(out.begin(), out.end());
  return out;
}

std::string fmt(const char* f, long long a, long long b = 0) {
  char buf[192];
  std::snprintf(buf, sizeof(buf), f, a, b);
  return buf;
}

// positions of out-of-range indices (ascending)
std::vector<int64_t> out_of_range(const DevArray<int64_t>& a, int64_t len, int64_t n) {
  DevArray<int64_t> list(std::max<int64_t>(len, 1), "validation");
  DevArray<unsigned long long> count(1, "validation");
  cudaStream_t s = spmvtk::rt::stream();
  cudaMemsetAsync(count.get(), 0, 8, s);
  if (len) k_out_of_range<<<blocks_for(len), 256, 0, s>>>(a.get(), len, 1, n, list.get(), len, count.get());
  spmvtk::rt::check(cudaGetLastError(), "validation");
  return fetch_list(list, count);
}

std::vector<int64_t> duplicates(const SegKey& key, int64_t len) {
  if (len <= 1) return {};
  uint64_t cap = 1;
  while (cap < static_cast<uint64_t>(len) * 2) cap <<= 1;
  DevArray<unsigned long long> keys(cap, "validation"), first(cap, "validation");
  DevArray<int64_t> list(len, "validation");
  DevArray<unsigned long long> count(1, "validation");
  cudaStream_t s = spmvtk::rt::stream();
  cudaMemsetAsync(keys.get(), 0xff, cap * 8, s);
  cudaMemsetAsync(first.get(), 0xff, cap * 8, s);
  cudaMemsetAsync(count.get(), 0, 8, s);
  k_dup_insert<<<blocks_for(len), 256, 0, s>>>(key, len, keys.get(), first.get(), cap - 1);
  k_dup_report<<<blocks_for(len), 256, 0, s>>>(key, len, keys.get(), first.get(), cap - 1,
                                               list.get(), len, count.get());
  spmvtk::rt::check(cudaGetLastError(), "validation");
  return fetch_list(list, count);
}

}  // namespace

namespace spmvtk::dev {

// pointer array + index range + distinct indices per segment: the rules of
// validate(CrsMatrix) with seg = "row" (ptr = row_ptr, idx = col_idx) and of
// validate(CcsMatrix) with seg = "column"
std::vector<std::string> validate_segments(std::int64_t n, const std::vector<std::int64_t>& ptr,
                                           const std::vector<std::int64_t>& idx,
                                           std::size_t nvalues, const char* ptr_name,
                                           const char* idx_name, const char* idx_kind,
                                           const char* seg_kind) {
  std::vector<std::string> out;
  if (n < 0) out.push_back("negative dimension");
  if (nvalues != idx.size())
    out.push_back(std::string("values / ") + idx_name + " length mismatch");
  const int64_t nnz = static_cast<int64_t>(nvalues);
  cudaStream_t s = rt::stream();
  const bool ptr_ok_len = static_cast<int64_t>(ptr.size()) == n + 1;
  if (!ptr_ok_len) {
    out.push_back(fmt("pointer array length %lld, expected %lld",
                      static_cast<long long>(ptr.size()), static_cast<long long>(n + 1)));
  } else {
    if (ptr.front() != 1) out.push_back(std::string(ptr_name) + "[1] != 1");
    if (ptr.back() != nnz + 1)
      out.push_back(fmt("pointer array end %lld, expected nnz+1 = %lld",
                        static_cast<long long>(ptr.back()), static_cast<long long>(nnz + 1)));
    DevArray<int64_t> dptr = upload(ptr);
    DevArray<unsigned long long> first(1, "validation");
    const unsigned long long none = static_cast<unsigned long long>(ptr.size());
    rt::copy_to_device(first.get(), &none, 8);
    k_first_descent<<<blocks_for(static_cast<int64_t>(ptr.size())), 256, 0, s>>>(
        dptr.get(), static_cast<int64_t>(ptr.size()), first.get());
    rt::check(cudaGetLastError(), "validation");
    unsigned long long f = none;
    rt::copy_to_host(&f, first.get(), 8);
    if (f != none)
      out.push_back(std::string(ptr_name) +
                    fmt(" not nondecreasing at position %lld", static_cast<long long>(f + 1)));
  }
  DevArray<int64_t> didx = upload(idx);
  for (int64_t p : out_of_range(didx, static_cast<int64_t>(idx.size()), n))
    out.push_back(std::string(idx_kind) +
                  fmt(" index %lld out of range at entry %lld", static_cast<long long>(idx[p]),
                      static_cast<long long>(p + 1)));
  if (!out.empty()) return out;
  // distinct indices inside every segment (pointers and ranges are valid)
  DevArray<int64_t> dptr = upload(ptr);
  for (int64_t p : duplicates(SegKey{dptr.get(), n, didx.get(), nullptr, n},
                              static_cast<int64_t>(idx.size()))) {
    const auto seg = std::upper_bound(ptr.begin(), ptr.end(), p + 1) - ptr.begin();  // 1-based
    out.push_back(std::string("duplicate index in ") + seg_kind +
                  fmt(" %lld (index %lld)", static_cast<long long>(seg),
                      static_cast<long long>(idx[p])));
  }
  return out;
}

std::vector<std::string> validate_triplets(std::int64_t n, const std::vector<std::int64_t>& row,
                                           const std::vector<std::int64_t>& col,
                                           std::size_t nvalues, int ordering) {
  std::vector<std::string> out;
  if (n < 0) out.push_back("negative dimension");
  if (nvalues != row.size() || nvalues != col.size()) {
    out.push_back("triplet sequences have differing lengths");
    return out;
  }
  const int64_t len = static_cast<int64_t>(nvalues);
  DevArray<int64_t> drow = upload(row), dcol = upload(col);
  for (int64_t p : out_of_range(drow, len, n))
    out.push_back(fmt("row index %lld out of range at entry %lld", static_cast<long long>(row[p]),
                      static_cast<long long>(p + 1)));
  for (int64_t p : out_of_range(dcol, len, n))
    out.push_back(fmt("column index %lld out of range at entry %lld",
                      static_cast<long long>(col[p]), static_cast<long long>(p + 1)));
  if (!out.empty()) return out;
  for (int64_t p : duplicates(SegKey{nullptr, 0, drow.get(), dcol.get(), n}, len))
    out.push_back(fmt("duplicate (row, col) pair (%lld, %lld)", static_cast<long long>(row[p]),
                      static_cast<long long>(col[p])));
  if (ordering == 0 || ordering == 1) {  // row-major / column-major tag
    const DevArray<int64_t>& key = ordering == 0 ? drow : dcol;
    DevArray<unsigned long long> first(1, "validation");
    const unsigned long long none = static_cast<unsigned long long>(len);
    rt::copy_to_device(first.get(), &none, 8);
    cudaStream_t s = rt::stream();
    k_first_descent<<<blocks_for(len), 256, 0, s>>>(key.get(), len, first.get());
    rt::check(cudaGetLastError(), "validation");
    unsigned long long f = none;
    rt::copy_to_host(&f, first.get(), 8);
    if (f != none)
      out.push_back(fmt(ordering == 0 ? "row_idx not nondecreasing at entry %lld"
                                      : "col_idx not nondecreasing at entry %lld",
                        static_cast<long long>(f + 1)));
  }
  return out;
}

std::vector<std::string> validate_ell(std::int64_t n, std::int64_t bc,
                                      const std::vector<double>& values,
                                      const std::vector<std::int64_t>& col,
                                      const std::vector<std::int64_t>& count,
                                      std::int64_t stored_nnz) {
  std::vector<std::string> out;
  if (n < 0) out.push_back("negative dimension");
  if (bc < 0) out.push_back("negative band count");
  const std::size_t slots = static_cast<std::size_t>(n * bc);
  if (values.size() != slots || col.size() != slots) {
    out.push_back("data sequences are not n * band_count long");
    return out;
  }
  if (static_cast<int64_t>(count.size()) != n) {
    out.push_back("row_entry_count length mismatch");
    return out;
  }
  DevArray<int64_t> dcol = upload(col);
  for (int64_t p : out_of_range(dcol, static_cast<int64_t>(slots), n))
    out.push_back(fmt("column index %lld out of range at entry %lld",
                      static_cast<long long>(col[p]), static_cast<long long>(p + 1)));
  DevArray<double> dval = upload(values);
  DevArray<int64_t> dcnt = upload(count);
  const int64_t cap = static_cast<int64_t>(std::max<std::size_t>(slots, static_cast<std::size_t>(n))) + 1;
  DevArray<int64_t> l0(cap, "validation"), l1(cap, "validation"), l2(cap, "validation");
  DevArray<unsigned long long> counts(3, "validation");
  cudaStream_t s = rt::stream();
  cudaMemsetAsync(counts.get(), 0, 24, s);
  if (n > 0)
    k_ell_padding<<<blocks_for(n), 256, 0, s>>>(n, bc, dcnt.get(), dval.get(), dcol.get(),
                                                l0.get(), l1.get(), l2.get(), cap, counts.get());
  rt::check(cudaGetLastError(), "validation");
  const std::vector<int64_t> bad_rows = fetch_list(l0, counts, 0);
  const std::vector<int64_t> bad_vals = fetch_list(l1, counts, 1);
  const std::vector<int64_t> bad_cols = fetch_list(l2, counts, 2);
  // the reference walks rows in order; inside a row, bands in order, the
  // value message before the column message of the same slot
  std::size_t ia = 0, ib = 0, ic = 0;
  for (int64_t i = 0; i < n && (ia < bad_rows.size() || ib < bad_vals.size() || ic < bad_cols.size());
       ++i) {
    if (ia < bad_rows.size() && bad_rows[ia] == i) {
      out.push_back(fmt("row %lld entry count %lld out of range", static_cast<long long>(i + 1),
                        static_cast<long long>(count[static_cast<std::size_t>(i)])));
      ++ia;
      continue;
    }
    for (int64_t k = 0; k < bc; ++k) {
      const int64_t slot = i * bc + k;
      if (ib < bad_vals.size() && bad_vals[ib] == slot) {
        out.push_back(fmt("nonzero padding value in row %lld band %lld",
                          static_cast<long long>(i + 1), static_cast<long long>(k + 1)));
        ++ib;
      }
      if (ic < bad_cols.size() && bad_cols[ic] == slot) {
        out.push_back(fmt("padding column in row %lld band %lld is not the row index",
                          static_cast<long long>(i + 1), static_cast<long long>(k + 1)));
        ++ic;
      }
      if ((ib >= bad_vals.size() || bad_vals[ib] >= (i + 1) * bc) &&
          (ic >= bad_cols.size() || bad_cols[ic] >= (i + 1) * bc))
        break;
    }
  }
  int64_t total = 0, max_r = 0;
  for (int64_t r : count) {
    if (r >= 0 && r <= bc) total += r;
    max_r = std::max(max_r, r);
  }
  if (total != stored_nnz)
    out.push_back(fmt("stored_nnz %lld inconsistent with row counts (sum %lld)",
                      static_cast<long long>(stored_nnz), static_cast<long long>(total)));
  if (n > 0 && max_r != bc)
    out.push_back(fmt("band count %lld is not the max row entry count %lld",
                      static_cast<long long>(bc), static_cast<long long>(max_r)));
  return out;
}

}  // namespace spmvtk::dev
