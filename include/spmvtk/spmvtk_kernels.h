/* spmvtk_kernels.h -- the thin lower C ABI into the sm_100a kernels.
 *
 * Device pointers + sizes + a CUDA stream in, a status out (0 = launched;
 * otherwise a cudaError_t value).  No allocation happens behind these calls
 * except where a function says so.  All launches are asynchronous on
 * `stream` (a cudaStream_t passed as void*; NULL = legacy default stream).
 *
 * Device layout ("GPU layout"): values fp64, every index and
 * pointer int32 and 0-based; ELL slot offsets are int64.  The reference keeps
 * 1-based int64 (/root/reference/proj/include/spmvtk/formats.hpp:10-14);
 * spmvtk_k_narrow_index / spmvtk_k_widen_index convert at the boundary.
 */
#ifndef SPMVTK_KERNELS_H
#define SPMVTK_KERNELS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- row statistics (formats.cpp:184-192 + stats.cpp:9-29 + the max of
 * convert.cpp:74-76) ------------------------------------------------------
 * acc (device, 3 x uint64) receives {max row length, sum, sum of squares};
 * it is zeroed by the call.  rows with ptr[i+1] < ptr[i] set bit 63 of
 * acc[0] (validation). */
int spmvtk_k_row_stats(const int32_t* ptr, int64_t n, unsigned long long* acc,
                       void* stream);
/* The same reduction published without a copy or a stream synchronisation:
 * acc = 4 device u64 that start zeroed (the kernel leaves them zeroed), host
 * = 4 u64 of mapped pinned memory; when the last CTA finishes it writes
 * {max | bad<<63, sum, sumsq} to host[0..2] and then seq to host[3], so the
 * caller spins on host[3] == seq.  n must be > 0. */
int spmvtk_k_row_stats_mapped(const int32_t* ptr, int64_t n, unsigned long long* acc,
                              unsigned long long* host, unsigned long long seq,
                              void* stream);

/* dst[i] = (int32)(src[i] - base) ; src int64 (reference layout). */
int spmvtk_k_narrow_index(const int64_t* src, int32_t* dst, int64_t len,
                          int64_t base, void* stream);
/* dst[i] = (int64)src[i] + base */
int spmvtk_k_widen_index(const int32_t* src, int64_t* dst, int64_t len,
                         int64_t base, void* stream);

/* Counts indices outside [0, n) into *bad (device uint64, zeroed first). */
int spmvtk_k_count_out_of_range(const int32_t* idx, int64_t len, int64_t n,
                                unsigned long long* bad, void* stream);
/* Counts positions p with key[p] < key[p-1] (ordering check). */
int spmvtk_k_count_descents(const int32_t* key, int64_t len,
                            unsigned long long* bad, void* stream);

/* ---- transforms ---------------------------------------------------------*/

/* Phase-II style pointer expansion (convert.cpp:15-20, :62-64):
 * out_idx[p] = r for ptr[r] <= p < ptr[r+1]. */
int spmvtk_k_expand_ptr(const int32_t* ptr, int64_t n, int64_t nnz,
                        int32_t* out_idx, void* stream);

/* CRS -> COO-row in one pass (convert.cpp:11-22): col / values copied,
 * row ids expanded from the row pointers. */
int spmvtk_k_crs_to_coo_row(int64_t n, int64_t nnz, const int32_t* irp,
                            const int32_t* icol, const double* val,
                            int32_t* out_row, int32_t* out_col, double* out_val,
                            void* stream);

/* Entries of a CRS whose column is not above the previous column of the same
 * row (0 = columns strictly ascending in every row: no duplicate pairs). */
int spmvtk_k_count_row_descents(const int32_t* irp, int64_t n, const int32_t* col,
                                unsigned long long* bad, void* stream);

/* The same pass plus the band shape that picks the SM-local ELL kernel:
 * out[0] descents, out[1] entries equal to the previous column + 1 of their
 * row, out[2] max(last column - row) + 2^32, out[3] max(row - first column)
 * + 2^32 over non-empty rows (row = row_offset + local row; out: device, 4
 * values, zeroed here). */
int spmvtk_k_row_order_stats(const int32_t* irp, int64_t n, int64_t row_offset,
                             const int32_t* col, unsigned long long* out, void* stream);

/* CRS -> CCS Phase I (convert.cpp:24-53).  scratch: device buffer of
 * spmvtk_k_ccs_scratch_bytes(n, nnz) bytes.  Row indices come out ascending
 * inside every column, exactly as the reference's cursor scatter.
 * spmvtk_k_crs_to_ccs / _coo_col place each entry by its rank by row inside
 * its column, so they need distinct (row, col) pairs;
 * spmvtk_k_crs_to_ccs_stable / _coo_col_stable are stable partitions that
 * keep the CRS order of every pair, duplicates included (same scratch). */
size_t spmvtk_k_ccs_scratch_bytes(int64_t n, int64_t nnz);
int spmvtk_k_crs_to_ccs(int64_t n, int64_t nnz, const int32_t* irp,
                        const int32_t* icol, const double* val,
                        int32_t* col_ptr, int32_t* row_idx, double* out_val,
                        void* scratch, void* stream);
/* CRS -> COO-col (convert.cpp:68-70 = Phase I then Phase II, ccs_to_coo_col
 * :55-66) in one pass: as spmvtk_k_crs_to_ccs, and the sort that places each
 * entry also writes its column into col_idx (no separate col_ptr expansion).
 * Same scratch as spmvtk_k_crs_to_ccs. */
/* 1 when the "ccs_stable" tuning knob routes every conversion to the stable
 * pipeline (testing). */
int spmvtk_k_ccs_force_stable(void);
int spmvtk_k_crs_to_ccs_stable(int64_t n, int64_t nnz, const int32_t* irp,
                               const int32_t* icol, const double* val, int32_t* col_ptr,
                               int32_t* row_idx, double* out_val, void* scratch,
                               void* stream);
int spmvtk_k_crs_to_coo_col_stable(int64_t n, int64_t nnz, const int32_t* irp,
                                   const int32_t* icol, const double* val,
                                   int32_t* col_ptr, int32_t* row_idx, int32_t* col_idx,
                                   double* out_val, void* scratch, void* stream);
int spmvtk_k_crs_to_coo_col(int64_t n, int64_t nnz, const int32_t* irp,
                            const int32_t* icol, const double* val,
                            int32_t* col_ptr, int32_t* row_idx, int32_t* col_idx,
                            double* out_val, void* scratch, void* stream);
/* Exclusive scan of n int32 counts into out[0..n] (out[n] = total). */
size_t spmvtk_k_scan_scratch_bytes(int64_t n);
int spmvtk_k_exclusive_scan(const int32_t* in, int32_t* out, int64_t n,
                            void* scratch, void* stream);

/* CRS -> ELL (convert.cpp:81-115), band-major: slot(k,i) = k*ld + i, with
 * ld >= n a multiple of 32 (the rows [n, ld) are layout padding: value 0,
 * column pad_base; exporting the first n rows of each band reproduces the
 * reference array).  Padding slots get value +0.0 and column = own row
 * (pad_base + i: pad_base is the global index of row 0 for a row-block
 * shard, 0 otherwise).  out_count[i] = row length. */
int spmvtk_k_crs_to_ell_cm(int64_t n, int32_t nz, int64_t ld, const int32_t* irp,
                           const int32_t* icol, const double* val,
                           double* out_val, int32_t* out_col,
                           int32_t* out_count, int64_t pad_base, void* stream);
/* Row-major ELL (no reference counterpart): slot(i,k) = i*nz + k. */
int spmvtk_k_crs_to_ell_rm(int64_t n, int32_t nz, const int32_t* irp,
                           const int32_t* icol, const double* val,
                           double* out_val, int32_t* out_col,
                           int32_t* out_count, int64_t pad_base, void* stream);

/* ---- inverse conversions -> canonical CRS (convert.cpp:117-183,
 * formats.cpp:228-244).  dup (device uint64) receives the smallest
 * duplicate position as (row << 32 | col), all-ones when there is none.
 * scratch: spmvtk_k_canon_scratch_bytes(n) bytes. ------------------------*/
size_t spmvtk_k_canon_scratch_bytes(int64_t nseg);
/* Sorts key[ptr[s]..ptr[s+1]) (payload val) for every segment s; keys must
 * be < key_bound. */
int spmvtk_k_sort_segments(const int32_t* ptr, int64_t nseg, int64_t key_bound,
                           int32_t* key, double* val, unsigned long long* dup,
                           void* scratch, void* stream);
/* ELL (slot(k,i) = k*stride_k + i*stride_i: band-major stride_k = ld,
 * stride_i = 1; row-major stride_k = 1, stride_i = nz) -> canonical CRS;
 * padding dropped by row_entry_count. */
int spmvtk_k_ell_to_crs(int64_t n, int64_t ncols, int64_t stride_k, int64_t stride_i,
                        const double* eval, const int32_t* ecol, const int32_t* cnt,
                        int32_t* irp, int32_t* icol, double* val,
                        unsigned long long* dup, void* scratch, void* stream);
/* COO triplets in any order -> canonical CRS. */
int spmvtk_k_coo_to_crs(int64_t n, int64_t ncols, int64_t nnz, const int32_t* row,
                        const int32_t* col, const double* v, int32_t* irp,
                        int32_t* icol, double* val, unsigned long long* dup,
                        void* scratch, void* stream);

/* ---- SpMV (y is overwritten; every row of y is written) ----------------*/

/* spmv_crs (spmv.cpp:64-75).  max_row = longest row (from row stats); rows
 * longer than the vector kernel's limit go to a block-per-row pass, which
 * needs `long_rows` (device int32 scratch of n+1 entries, may be NULL when
 * max_row is small). */
int spmvtk_k_spmv_crs(int64_t n, const int32_t* irp, const int32_t* icol,
                      const double* val, const double* x, double* y,
                      double mean_row, int32_t max_row, int32_t* long_rows,
                      void* stream);
/* ---- entry-balanced ("segmented") CRS SpMV (kernels_spmv_seg.cu)
 * A plan assigns warp w the rows whose first entry lies in [w*chunk,
 * (w+1)*chunk): plan[w] = first row r with irp[r] >= w*chunk, plan[nwarps]
 * = n (nwarps + 1 int32 entries; chunk <= 0 = SPMVTK_SEG_CHUNK). */
#define SPMVTK_SEG_CHUNK 2048
int32_t spmvtk_k_seg_plan_warps(int64_t nnz, int32_t chunk);
/* The chunk the library's plans use (SPMVTK_SEG_CHUNK unless tuned). */
int32_t spmvtk_k_seg_chunk(void);
int spmvtk_k_seg_plan(int64_t n, int64_t nnz, const int32_t* irp, int32_t chunk,
                      int32_t* plan, void* stream);
/* y[r] for the rows of warps [w_base, w_end) clipped to [row_lo, row_hi);
 * every row of that range is written. */
int spmvtk_k_spmv_crs_seg(const int32_t* irp, const int32_t* icol, const double* val,
                          const double* x, double* y, const int32_t* plan,
                          int32_t w_base, int32_t w_end, int64_t row_lo, int64_t row_hi,
                          int64_t nnz, void* stream);
/* The CRS kernel choice: 1 = segmented (plan needed), 0 = sub-warp per row. */
int spmvtk_k_crs_use_seg(double mean_row, int64_t max_row);
/* ell-outer's band chunks when forced through spmvtk_k_tune("ell_splits", k)
 * (0 = chosen by occupancy: split only when row pairs cannot fill the GPU). */
int spmvtk_k_ell_splits_forced(void);
/* The SM-local ELL choice forced by spmvtk_k_tune("ell_banded", v): -1 =
 * automatic (from the handle's band shape), 0 = never, 1 = always. */
int spmvtk_k_ell_banded_forced(void);
/* Row length above which spmvtk_k_spmv_crs hands a row to the block-per-row
 * pass (long_rows must then be non-NULL when max_row exceeds it). */
int64_t spmvtk_k_crs_long_limit(double mean_row);
/* spmv_coo_row_outer (spmv.cpp:79-101,111-115): row-sorted triplets,
 * deterministic segmented reduction, no atomics. */
int spmvtk_k_spmv_coo_row(int64_t n, int64_t nnz, const int32_t* row,
                          const int32_t* col, const double* val,
                          const double* x, double* y, void* stream);
/* spmv_coo_col_outer (spmv.cpp:105-109): column-sorted triplets; y is
 * zeroed, then fp64 reductions into y (order of additions not fixed). */
int spmvtk_k_spmv_coo_col(int64_t n, int64_t nnz, const int32_t* row,
                          const int32_t* col, const double* val,
                          const double* x, double* y, void* stream);
/* spmv_ell_inner (spmv.cpp:117-136): thread per row pair, bands in order,
 * 128-bit loads; every slot (padding included) is multiplied. */
int spmvtk_k_spmv_ell_cm(int64_t n, int32_t nz, int64_t ld, const double* val,
                         const int32_t* col, const double* x, double* y,
                         void* stream);
/* The same product for banded matrices whose columns scatter inside a band
 * window of x (one 1024-thread CTA per SM, each sweeping one contiguous row
 * region, so an SM's gathers stay inside one window that L1 holds).  Picked
 * by the library from the handle's band shape; same results as
 * spmvtk_k_spmv_ell_cm (each row summed band by band in the same order). */
int spmvtk_k_spmv_ell_cm_banded(int64_t n, int32_t nz, int64_t ld, const double* val,
                                const int32_t* col, const double* x, double* y,
                                void* stream);
/* spmv_ell_outer (spmv.cpp:138-158): bands split in `splits` contiguous
 * chunks (partition_range rule), per-chunk partial vectors in `partial`
 * (device, splits*n doubles), then an ascending-chunk reduction. */
int spmvtk_k_spmv_ell_cm_split(int64_t n, int32_t nz, int64_t ld,
                               const double* val, const int32_t* col,
                               const double* x, double* y, int32_t splits,
                               double* partial, void* stream);
/* Row-major ELL SpMV (no reference counterpart). */
int spmvtk_k_spmv_ell_rm(int64_t n, int32_t nz, const double* val,
                         const int32_t* col, const double* x, double* y,
                         void* stream);

/* ---- pushed results (multi-GPU, spmvtk.h "exchange folded into the SpMV")
 * Same products as spmvtk_k_spmv_crs / spmvtk_k_spmv_ell_cm; row r of the
 * result goes to dst[w][r] for every w with bit w of mask[r] (mask NULL =
 * all), then each thread fences at system scope; sync (may be NULL): the
 * step's flag wait (kernel prologue) and signal (last CTA) in the same launch. */
struct spmvtk_push;
struct spmvtk_push_sync;
int spmvtk_k_spmv_crs_push(int64_t n, const int32_t* irp, const int32_t* icol,
                           const double* val, const double* x,
                           const struct spmvtk_push* push,
                           const struct spmvtk_push_sync* sync, double mean_row,
                           int32_t max_row, int32_t* long_rows, void* stream);
int spmvtk_k_spmv_crs_seg_push(const int32_t* irp, const int32_t* icol, const double* val,
                               const double* x, const struct spmvtk_push* push,
                               const struct spmvtk_push_sync* sync, const int32_t* plan,
                               int32_t nwarps, int64_t n, int64_t nnz, void* stream);
int spmvtk_k_spmv_ell_cm_push(int64_t n, int32_t nz, int64_t ld, const double* val,
                              const int32_t* col, const double* x,
                              const struct spmvtk_push* push,
                              const struct spmvtk_push_sync* sync, void* stream);
/* Step flags (system scope): signal stores value to every target; wait
 * spins (one thread per source) until flags[s] >= value or timeout_ns. */
struct spmvtk_flag_targets;
int spmvtk_k_flags_signal(const struct spmvtk_flag_targets* targets, uint64_t value,
                          void* stream);
int spmvtk_k_flags_wait(const uint64_t* flags, int32_t n, uint64_t value,
                        uint64_t timeout_ns, uint32_t* status, void* stream);

/* Push-exchange setup: need[c] = 1 for every column in col[0..len); the
 * per-row reader mask from every rank's need array (need_all: world * n
 * bytes): bit w of mask[r] = rank w reads global row row_offset + r. */
int spmvtk_k_mark_columns(const int32_t* col, int64_t len, uint8_t* need, void* stream);
int spmvtk_k_push_mask(const uint8_t* need_all, int32_t world, int64_t n, int64_t row_offset,
                       int64_t rows, int32_t rank, uint8_t* mask, void* stream);

/* Random 8-byte gathers from x[0..n_pow2) (L2-resident), 2 CTAs x 512
 * threads per SM, `iters` per thread: the gather-rate roofline of the SpMV
 * kernels (gathers = 1024 * SMs * iters). */
int spmvtk_k_gather_probe(const double* x, int64_t n_pow2, int iters, double* out,
                          void* stream);

/* Tuning override for experiments ("crs_variant": -1 = heuristic, 0..9 pick
 * a (lanes per row, rows per sub-warp) instance of the CRS kernel). */
int spmvtk_k_tune(const char* key, int value);
/* Transform tuning knobs ("ccs_slices", "ccs_threads"); spmvtk_k_tune
 * forwards keys it does not know here. */
int spmvtk_k_tune_convert(const char* key, int value);

/* SpMV kernel launches this process has made through the library (every
 * SpMV entry point counts the kernels it launches): bench.py's gpu_launches. */
unsigned long long spmvtk_k_launch_count(void);

/* Forces every kernel of the library to be loaded (lazy module loading
 * would otherwise charge the first timed call). */
int spmvtk_k_preload(void);

#ifdef __cplusplus
}
#endif

#endif /* SPMVTK_KERNELS_H */
