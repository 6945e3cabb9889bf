// matrix.hpp -- the device-resident matrix handle behind spmvtk_matrix*.
//
// One handle type for every format (the reference keeps a
// variant<Crs,Ccs,Coo,Ell> of host vectors, capi.cpp:23-25).  Arrays live in
// HBM in the GPU layout: fp64 values, int32 0-based indices, ELL band-major
// with a 32-aligned leading dimension.  Handles are immutable after
// construction except for the cached row moments (guarded by a mutex), so
// concurrent reads from several threads are safe, as in the reference
// (SPEC.md:100-101).
#pragma once

#include <cstdint>
#include <mutex>
#include <optional>
#include <vector>

#include "runtime.hpp"
#include "spmvtk/spmvtk.h"

struct spmvtk_matrix {
  spmvtk_format format = SPMVTK_FORMAT_CRS;
  int ordering = -1;  // COO: 0 row-major, 1 column-major
  bool rows_sorted = true;  // COO row-major tag verified (host-built COO may not be)
  int device = 0;
  std::int64_t n = 0;     // rows
  std::int64_t nnz = 0;   // stored entries; ELL: stored_nnz (real entries)
  std::int64_t ncols = 0; // columns (== n except for row-block shards)
  std::int64_t row_offset = 0;  // global index of row 0 (row-block shards)

  spmvtk::rt::DevArray<double> val;
  spmvtk::rt::DevArray<std::int32_t> ptr;    // CRS row_ptr / CCS col_ptr
  spmvtk::rt::DevArray<std::int32_t> row;    // COO / CCS row indices
  spmvtk::rt::DevArray<std::int32_t> col;    // CRS / COO / ELL column indices
  spmvtk::rt::DevArray<std::int32_t> count;  // ELL row_entry_count
  // one allocation holding several of the arrays above (they are views into
  // it); declared after them so it is released last
  spmvtk::rt::DevArray<unsigned char> block;
  std::int32_t band_count = 0;               // ELL
  std::int64_t ld = 0;                       // ELL band-major leading dim

  mutable std::mutex mu;
  mutable std::optional<spmvtk::rt::Moments> moments;  // CRS row moments
  // CRS: entry-balanced SpMV plan (warp -> first row), built at the first
  // segmented SpMV; host copy for row-range launches
  mutable spmvtk::rt::DevArray<std::int32_t> seg_plan;
  mutable std::vector<std::int32_t> seg_plan_host;
  mutable std::int32_t seg_plan_chunk = 0;
  // CRS / CCS: columns (rows) strictly ascending inside every row (column),
  // hence no duplicate pairs -- the fast CCS pipeline's precondition
  mutable std::optional<bool> pairs_ascending;
  // CRS (and the ELL built from it): band shape from the same pass --
  // max(last column - row), max(row - first column), entries that continue
  // a run of consecutive columns; picks the SM-local ELL kernel
  struct BandShape {
    std::int64_t right = 0, left = 0;
    std::uint64_t adjacent = 0;
  };
  mutable std::optional<BandShape> band;

  std::uint64_t device_bytes() const {
    return val.bytes() + ptr.bytes() + row.bytes() + col.bytes() + count.bytes();
  }
};

namespace spmvtk::dev {

using Matrix = spmvtk_matrix;

// Exact row moments of a CRS handle (cached after the first GPU reduction).
rt::Moments crs_moments(const Matrix& m);
// Whether the pointer-structured handle (CRS; CCS = CRS of the transpose)
// has strictly ascending indices inside every segment (cached).
bool pairs_ascending(const Matrix& m);
// The segmented-SpMV plan of a CRS handle (cached; nwarps + 1 entries).
const std::vector<std::int32_t>& crs_seg_plan(const Matrix& m, const std::int32_t** dev);

// CRS from caller arrays; see spmvtk_matrix_from_crs.
Matrix* crs_from_arrays(std::int64_t n, std::int64_t nnz, const void* row_ptr,
                        const void* col_idx, const double* values, int index_width,
                        int index_base, bool on_device);
// Row-block shard: nrows local rows holding global columns in [0, ncols);
// row_offset = global index of local row 0 (multi-GPU row partitioning).
Matrix* crs_block_from_arrays(std::int64_t nrows, std::int64_t ncols, std::int64_t row_offset,
                              std::int64_t nnz, const void* row_ptr, const void* col_idx,
                              const double* values, int index_width, int index_base,
                              bool on_device);

// COO from caller arrays (ordering: 0 row-major, 1 column-major).  A
// row-major tag is checked on the GPU; unsorted rows keep the tag but the
// SpMV then uses the order-independent kernel.
Matrix* coo_from_arrays(std::int64_t n, std::int64_t nnz, const void* rows, const void* cols,
                        const double* values, int index_width, int index_base, int ordering);
// Band-major ELL from reference-layout arrays (n*band_count values and
// columns, row_entry_count[n]); re-pitched to the device leading dimension.
Matrix* ell_from_arrays(std::int64_t n, std::int64_t band_count, const std::int64_t* col_1based,
                        const double* values, const std::int64_t* row_entry_count,
                        std::int64_t stored_nnz);

// Reference ELL estimate (8+8 bytes per slot, convert.cpp:72-79).
std::uint64_t reference_ell_estimate(const Matrix& crs);
std::uint64_t device_bytes_for(const Matrix& crs, spmvtk_format to);

// Conversions of a CRS handle (the guard applies to the ELL formats).
Matrix* convert(const Matrix& crs, spmvtk_format to, std::uint64_t max_bytes);

// Any handle -> canonical CRS on the device (columns ascending inside rows);
// duplicate positions refused with the reference's message
// (convert.cpp:119-154).  For a CRS handle this is canonicalize().
Matrix* to_crs(const Matrix& m);

// Median device time of the transform's kernels alone (outputs and scratch
// preallocated; the ELL variants include the band-count reduction).
double transform_kernel_seconds(const Matrix& crs, spmvtk_format to, int repeats);

// y = A x on device vectors, async on the current stream.  Throws
// InvalidArgument when the kernel does not match the handle's format (or
// COO ordering), with the reference's messages (capi.cpp:230-252).
void spmv_device(const Matrix& m, spmvtk_kernel kernel, const double* x, double* y);
// SpMV whose result rows are pushed to peer buffers (spmvtk_spmv_device_push):
// CRS (kernel CRS) and band-major ELL (kernel ELL_INNER)
void spmv_device_push(const Matrix& m, spmvtk_kernel kernel, const double* x,
                      const spmvtk_push& push, const spmvtk_push_sync* sync);

// True when `kernel` on `m` can be launched on row sub-ranges (CRS, ELL
// band-major inner, row-major ELL): rows are independent and y is written
// once per row, so a host pipeline can copy finished row blocks back while
// later ones compute.
bool spmv_row_splittable(const Matrix& m, spmvtk_kernel kernel);
// y[r0:r1) = A[r0:r1, :] x (r0 a multiple of 64).
void spmv_device_rows(const Matrix& m, spmvtk_kernel kernel, const double* x, double* y,
                      std::int64_t r0, std::int64_t r1);

// One array to host memory in the requested index width / base.
std::int64_t copy_array(const Matrix& m, spmvtk_array which, void* dst, std::int64_t capacity,
                        int index_width, int index_base);
std::int64_t device_array(const Matrix& m, spmvtk_array which, void** ptr);
// Bands [k0, k1) of a band-major ELL handle in the reference layout
// ((k1-k0) * n slots; columns widened to int64 in index_base).
void copy_ell_bands(const Matrix& m, std::int64_t k0, std::int64_t k1, double* values,
                    std::int64_t* col_idx, int index_base);

const char* kernel_label(spmvtk_kernel k);

}  // namespace spmvtk::dev

struct spmvtk_dist;
namespace spmvtk::dist {
spmvtk_dist* init(int rank, int world, const unsigned char* id);
void destroy(spmvtk_dist* d);
int rank_of(const spmvtk_dist& d);
int world_of(const spmvtk_dist& d);
void unique_id(unsigned char* out);
double iterate(const spmvtk_dist& d, const dev::Matrix& shard, spmvtk_kernel kernel, double* x,
               std::int64_t steps);
struct Push;
Push* push_create(const spmvtk_dist& d, const dev::Matrix& shard, spmvtk_kernel kernel,
                  bool sparse);
void push_free(Push* p);
double push_iterate(Push& p, double* x, std::int64_t steps);
}  // namespace spmvtk::dist
