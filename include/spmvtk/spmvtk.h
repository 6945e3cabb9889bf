/* spmvtk.h -- C ABI of the B200-native spmvtk (arXiv 2407.00019 path).
 *
 * Part 1 is a drop-in for the reference C ABI
 * (/root/reference/proj/include/spmvtk/spmvtk.h:17-160): same 23 entry
 * points, same enum values, same status mapping (capi.cpp:35-62).  Handles
 * own DEVICE buffers on the current CUDA device; host arrays passed to the
 * legacy calls are copied in and out.  Part 2 are extensions the reference
 * lacks: building a handle from raw arrays, reading arrays
 * back, device-pointer SpMV on a caller stream, row-major ELL, the synthetic
 * BASELINE generators.  Every call returns a status; spmvtk_last_error()
 * holds the calling thread's message (thread-local, cleared on success).
 */
#ifndef SPMVTK_H
#define SPMVTK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ======================= part 1: reference ABI ========================== */

typedef enum spmvtk_status {      /* spmvtk.h:17-23 */
  SPMVTK_OK = 0,
  SPMVTK_ERR_USAGE = 1,           /* InvalidArgument */
  SPMVTK_ERR_DATA = 2,            /* Validation / Io / Parse / CUDA failure */
  SPMVTK_ERR_CHECK = 3,           /* never returned by the library */
  SPMVTK_ERR_MEMORY_LIMIT = 4,    /* ELL guard or device allocation */
} spmvtk_status;

typedef enum spmvtk_format {      /* spmvtk.h:28-34 */
  SPMVTK_FORMAT_CRS = 0,
  SPMVTK_FORMAT_CCS = 1,
  SPMVTK_FORMAT_COO_ROW = 2,
  SPMVTK_FORMAT_COO_COL = 3,
  SPMVTK_FORMAT_ELL = 4,          /* band-major ("column-major") */
  SPMVTK_FORMAT_ELL_ROWMAJOR = 5, /* extension: row-major ELL */
} spmvtk_format;

typedef enum spmvtk_kernel {      /* spmvtk.h:36-42 */
  SPMVTK_KERNEL_CRS = 0,
  SPMVTK_KERNEL_COO_ROW_OUTER = 1,
  SPMVTK_KERNEL_COO_COL_OUTER = 2,
  SPMVTK_KERNEL_ELL_INNER = 3,
  SPMVTK_KERNEL_ELL_OUTER = 4,
  SPMVTK_KERNEL_ELL_ROWMAJOR = 5, /* extension: SpMV on a row-major ELL */
} spmvtk_kernel;

typedef enum spmvtk_decision {    /* spmvtk.h:44-47 */
  SPMVTK_USE_ELL = 0,
  SPMVTK_USE_CRS = 1,
} spmvtk_decision;

typedef struct spmvtk_matrix spmvtk_matrix;
typedef struct spmvtk_profile spmvtk_profile;

const char* spmvtk_last_error(void);
void spmvtk_matrix_free(spmvtk_matrix* m);
void spmvtk_profile_free(spmvtk_profile* p);

/* Matrix Market coordinate real general|symmetric -> CRS handle
 * (ingest.cpp:95-212); write is canonical general, %.17g (ingest.cpp:214-232). */
spmvtk_status spmvtk_read_matrix_market(const char* path, spmvtk_matrix** out);
spmvtk_status spmvtk_write_matrix_market(const spmvtk_matrix* m, const char* path);

/* Generators, byte-identical to the reference for equal seeds
 * (ingest.cpp:234-316, mt19937_64 raw-bit convention). */
spmvtk_status spmvtk_gen_banded(int64_t n, int64_t half_width, spmvtk_matrix** out);
spmvtk_status spmvtk_gen_skewed(int64_t n, int64_t base_deg, int64_t heavy_rows,
                                int64_t heavy_deg, uint64_t seed, spmvtk_matrix** out);
spmvtk_status spmvtk_gen_cv_target(int64_t n, double mean_deg, double target_dmat,
                                   uint64_t seed, spmvtk_matrix** out);

typedef struct spmvtk_matrix_info {  /* spmvtk.h:76-84 */
  int64_t n;
  int64_t nnz;
  int64_t max_row_entries;
  double mu;
  double sigma;
  double d_mat;
  uint64_t ell_bytes;  /* reference estimate: n * max_row * (8 + 8) */
} spmvtk_matrix_info;

spmvtk_format spmvtk_matrix_get_format(const spmvtk_matrix* m);
/* CRS handle only; statistics need nnz >= 1 (stats.cpp:31-35). */
spmvtk_status spmvtk_matrix_get_info(const spmvtk_matrix* m, spmvtk_matrix_info* out);

/* CRS handle -> new handle in `to`.  max_bytes != 0 arms the ELL guard on
 * the reference's 16-byte-per-slot estimate (convert.cpp:82-88). */
spmvtk_status spmvtk_matrix_convert(const spmvtk_matrix* m, spmvtk_format to,
                                    uint64_t max_bytes, spmvtk_matrix** out);

/* Host x (len n) in, host y (len n) out.  `lanes` is validated (>= 1) and
 * otherwise ignored on the GPU.  elapsed_seconds (may be NULL) is the device
 * time of the SpMV kernels, copies excluded (the reference times the kernel
 * call without the copy-out, capi.cpp:222-256). */
spmvtk_status spmvtk_spmv(const spmvtk_matrix* m, spmvtk_kernel kernel, const double* x,
                          int64_t len, int lanes, double* y, double* elapsed_seconds);

typedef struct spmvtk_bench_result {  /* spmvtk.h:104-111 */
  double t_crs;
  double t_ell;
  double t_trans;
  double sp;
  double tt;
  double r;
} spmvtk_bench_result;

/* (t_crs, t_trans, t_ell) on a CRS handle, x = ones (capi.cpp:260-306).
 * SpMV times: one untimed warm-up, median of `repeats` CUDA-event timings.
 * t_trans: one cold conversion (allocation included), wall clock. */
spmvtk_status spmvtk_bench(const spmvtk_matrix* m, spmvtk_kernel variant, int lanes,
                           int repeats, uint64_t max_bytes, spmvtk_bench_result* out);

spmvtk_status spmvtk_profile_build(const spmvtk_matrix* const* matrices,
                                   const char* const* ids, size_t count,
                                   spmvtk_kernel variant, int lanes, double c, int repeats,
                                   uint64_t max_bytes, const char* machine_label,
                                   spmvtk_profile** out);
/* JSON schema version 1, unknown keys rejected (autotune.cpp:264-377). */
spmvtk_status spmvtk_profile_write(const spmvtk_profile* p, const char* path);
spmvtk_status spmvtk_profile_read(const char* path, spmvtk_profile** out);

double spmvtk_profile_d_star(const spmvtk_profile* p);
double spmvtk_profile_c(const spmvtk_profile* p);
int spmvtk_profile_lanes(const spmvtk_profile* p);
spmvtk_kernel spmvtk_profile_kernel(const spmvtk_profile* p);
size_t spmvtk_profile_record_count(const spmvtk_profile* p);

typedef struct spmvtk_record_view {  /* spmvtk.h:123-140 */
  const char* matrix_id;        /* borrowed from the profile */
  int64_t n;
  int64_t nnz;
  double mu;
  double sigma;
  double d_mat;
  int excluded;
  const char* exclusion_reason; /* NULL unless excluded */
  double t_crs;                 /* NaN when excluded */
  double t_ell;
  double t_trans;
  double sp;
  double tt;
  double r;
} spmvtk_record_view;

spmvtk_status spmvtk_profile_record(const spmvtk_profile* p, size_t index,
                                    spmvtk_record_view* out);

/* UseEll iff d_mat < d_star, strict (autotune.cpp:231-236); d_mat is
 * computed on the GPU. */
spmvtk_status spmvtk_select(const spmvtk_matrix* m, const spmvtk_profile* p,
                            spmvtk_decision* decision, double* d_mat);

/* ========================= part 2: extensions =========================== */

/* All GPU work of the calling thread is issued on this stream (a
 * cudaStream_t; NULL = legacy default stream).  Thread-local. */
void spmvtk_set_stream(void* stream);
void* spmvtk_get_stream(void);
/* Synchronises the current stream; maps a pending CUDA error to a status. */
spmvtk_status spmvtk_synchronize(void);

/* Build a CRS handle from arrays.  index_width 4 or 8 bytes, index_base 0 or
 * 1 (the reference layout is width 8, base 1).  on_device != 0: the three
 * pointers are device pointers.  Validated on the GPU: pointer array
 * monotone, starts at base, ends at nnz+base; column indices in range.
 * (Duplicate positions are not checked, as in the reference converters.) */
spmvtk_status spmvtk_matrix_from_crs(int64_t n, int64_t nnz, const void* row_ptr,
                                     const void* col_idx, const double* values,
                                     int index_width, int index_base, int on_device,
                                     spmvtk_matrix** out);

/* Row-block shard for multi-GPU row partitioning: nrows local rows of a
 * matrix with ncols columns; row_offset is the global index of local row 0
 * (used for ELL padding columns).  Shards convert to CRS, COO-row and ELL
 * (both layouts); SpMV takes x of length ncols and writes nrows entries. */
spmvtk_status spmvtk_matrix_from_crs_block(int64_t nrows, int64_t ncols, int64_t row_offset,
                                           int64_t nnz, const void* row_ptr, const void* col_idx,
                                           const double* values, int index_width, int index_base,
                                           int on_device, spmvtk_matrix** out);

/* Any handle -> new canonical CRS handle (columns ascending in each row),
 * on the device: the inverse conversions coo_to_crs / ell_to_crs
 * (convert.cpp:117-183), CCS -> CRS, and canonicalize for a CRS handle.
 * Duplicate positions in COO / ELL input -> SPMVTK_ERR_DATA
 * "duplicate (row, col) pair (r, c)". */
spmvtk_status spmvtk_matrix_to_crs(const spmvtk_matrix* m, spmvtk_matrix** out);

typedef struct spmvtk_matrix_desc {
  int32_t format;       /* spmvtk_format */
  int32_t ordering;     /* COO: 0 row-major, 1 column-major; else -1 */
  int64_t n;            /* rows */
  int64_t nnz;          /* stored entries (ELL: stored_nnz) */
  int64_t band_count;   /* ELL only */
  int64_t ld;           /* ELL band-major leading dimension on the device */
  uint64_t device_bytes;
  int64_t ncols;        /* columns (== n unless a row-block shard) */
  int64_t row_offset;   /* global index of row 0 (row-block shards) */
} spmvtk_matrix_desc;

spmvtk_status spmvtk_matrix_describe(const spmvtk_matrix* m, spmvtk_matrix_desc* out);

typedef enum spmvtk_array {
  SPMVTK_ARRAY_VALUES = 0,
  SPMVTK_ARRAY_POINTER = 1,         /* CRS row_ptr / CCS col_ptr (n+1) */
  SPMVTK_ARRAY_ROW_IDX = 2,         /* COO, CCS */
  SPMVTK_ARRAY_COL_IDX = 3,         /* CRS, COO, ELL */
  SPMVTK_ARRAY_ROW_ENTRY_COUNT = 4, /* ELL */
} spmvtk_array;

/* Copies one array to host memory `dst` (capacity in elements) in the
 * requested index width/base; *len receives the element count (call with
 * dst = NULL to query).  ELL arrays come out in the reference layout:
 * band-major n*band_count (row-major for SPMVTK_FORMAT_ELL_ROWMAJOR).
 * Values are copied bit for bit; row_entry_count ignores index_base. */
spmvtk_status spmvtk_matrix_copy_array(const spmvtk_matrix* m, spmvtk_array which,
                                       void* dst, int64_t capacity, int index_width,
                                       int index_base, int64_t* len);

/* Device view of an array in the GPU layout (int32 0-based indices; ELL
 * band-major with leading dimension desc.ld).  Borrowed from the handle. */
spmvtk_status spmvtk_matrix_device_array(const spmvtk_matrix* m, spmvtk_array which,
                                         void** ptr, int64_t* len);

/* SpMV on device vectors (x, y: n doubles each, device pointers), async on
 * the current stream.  No host synchronisation, no allocation unless the
 * kernel needs scratch (CRS rows > 4096 entries, ELL_OUTER splits). */
spmvtk_status spmvtk_spmv_device(const spmvtk_matrix* m, spmvtk_kernel kernel,
                                 const double* x, double* y);

typedef struct spmvtk_row_stats {
  int64_t n;
  int64_t nnz;
  int64_t max_row;
  double mu;
  double sigma;
  double d_mat;
} spmvtk_row_stats;

/* D_mat statistics of a CRS handle computed by the on-GPU reduction. */
spmvtk_status spmvtk_matrix_row_stats(const spmvtk_matrix* m, spmvtk_row_stats* out);

/* Synthetic BASELINE.json workloads.  config:
 *   1  2-D 5-point Laplacian, param = grid edge (256)
 *   2  random rows, lengths U{8..24}, columns uniform, param = n (2^20)
 *   3  3-D 27-point stencil, param = grid edge (128)
 *   4  power-law rows, log-normal lengths (mean 16, sigma_log 1.2, cap 4096),
 *      param = n (2^22)
 *   5  D_mat sweep, Gamma lengths (mean 32) with target D = dparam, columns
 *      within +-n/64 of the diagonal, param = n (2^21)
 * Values N(0,1) (config 1: 4 / -1; config 3: diagonal 27). */
spmvtk_status spmvtk_gen_baseline(int config, int64_t param, double dparam, uint64_t seed,
                                  spmvtk_matrix** out);
/* The same workloads generated into host memory only (no device touched),
 * e.g. to feed a CPU implementation; export as 1-based or 0-based int64. */
typedef struct spmvtk_host_crs spmvtk_host_crs;
spmvtk_status spmvtk_gen_baseline_host(int config, int64_t param, double dparam, uint64_t seed,
                                       spmvtk_host_crs** out, int64_t* n, int64_t* nnz);
spmvtk_status spmvtk_host_crs_export(const spmvtk_host_crs* h, int64_t* row_ptr,
                                     int64_t* col_idx, double* values, int index_base);
void spmvtk_host_crs_free(spmvtk_host_crs* h);
/* Matrix Market file -> host CRS (no device work; same parser and refusals
 * as spmvtk_read_matrix_market, multi-threaded). */
spmvtk_status spmvtk_read_matrix_market_host(const char* path, spmvtk_host_crs** out,
                                             int64_t* n, int64_t* nnz);
/* Uploads a host CRS (from spmvtk_gen_baseline_host) into a device handle. */
spmvtk_status spmvtk_matrix_from_host_crs(const spmvtk_host_crs* h, spmvtk_matrix** out);

/* Bands [k0, k1) (0-based) of a band-major ELL handle, in the reference
 * layout: (k1-k0)*n values and int64 column indices in index_base (either
 * output may be NULL) -- to stream an ELL too large for one host copy. */
spmvtk_status spmvtk_matrix_copy_ell_bands(const spmvtk_matrix* m, int64_t k0, int64_t k1,
                                           double* values, int64_t* col_idx, int index_base);

/* ---- multi-GPU: row-block shards, one process per GPU, NCCL -------------
 * The rows are cut into `world` contiguous entry-balanced blocks
 * (spmvtk_partition_rows: rank k starts at the first row whose start reaches
 * k*nnz/world -- the reference's partition_range, spmv.cpp:36-54, applied to
 * entries instead of rows).  A shard holds its rows with global column
 * indices, so every transform of it is local; SpMV iterations exchange x
 * between ranks over NCCL (spmvtk_dist_spmv_iterate). */
#define SPMVTK_DIST_ID_BYTES 128
typedef struct spmvtk_dist spmvtk_dist;
/* Rank 0 makes the id and sends it to the others (any channel). */
spmvtk_status spmvtk_dist_unique_id(unsigned char id[SPMVTK_DIST_ID_BYTES]);
/* Joins the communicator on the calling thread's current CUDA device. */
spmvtk_status spmvtk_dist_init(int rank, int world, const unsigned char id[SPMVTK_DIST_ID_BYTES],
                               spmvtk_dist** out);
void spmvtk_dist_free(spmvtk_dist* d);
/* begin[world + 1] for a CRS given by its n + 1 row pointers (host; any
 * index base). */
spmvtk_status spmvtk_partition_rows(const int64_t* row_ptr, int64_t n, int world, int64_t* begin);
/* This rank's shard of a global CRS in host arrays: only the rank's rows are
 * read and uploaded (index_width 4 or 8, index_base 0 or 1). */
spmvtk_status spmvtk_matrix_distribute(const spmvtk_dist* d, int64_t n, const void* row_ptr,
                                       const void* col_idx, const double* values, int index_width,
                                       int index_base, spmvtk_matrix** shard);
/* A BASELINE workload's shard for (rank, world), generated alone on the host
 * (every row length is drawn for the partition, only the rank's rows are
 * filled): identical to the rows of spmvtk_gen_baseline_host's matrix.  The
 * host variant needs no device; the other uploads it. */
spmvtk_status spmvtk_gen_baseline_shard_host(int config, int64_t param, double dparam,
                                             uint64_t seed, int rank, int world,
                                             spmvtk_host_crs** out, int64_t* rows,
                                             int64_t* row_offset, int64_t* ncols);
spmvtk_status spmvtk_gen_baseline_shard(const spmvtk_dist* d, int config, int64_t param,
                                        double dparam, uint64_t seed, spmvtk_matrix** shard);
/* x_{t+1} = A x_t, `steps` times.  x: device vector of ncols doubles on the
 * current stream, x_0 on entry (the same on every rank), x_steps on exit on
 * every rank.  Each step: the shard's SpMV writes its rows of x_{t+1}
 * straight into its block, then every block is broadcast to the other ranks
 * (grouped ncclBroadcast, in place).  seconds (may be NULL): this rank's
 * device time per step (CUDA events); take the max over ranks. */
spmvtk_status spmvtk_dist_spmv_iterate(const spmvtk_dist* d, const spmvtk_matrix* shard,
                                       spmvtk_kernel kernel, double* x, int64_t steps,
                                       double* seconds);

/* The same iteration with the exchange folded into the SpMV: every rank's
 * x buffers and step flags are shared through CUDA IPC (handles exchanged
 * over the communicator), and each step is ONE kernel launch that waits for
 * the step's flags, computes the shard's rows and stores each of them
 * straight into the next-x buffer of every rank that reads it (sparse != 0:
 * only the ranks whose shard references the row; else all), then raises the
 * next flag on every rank.  CRS or band-major ELL_INNER shards, up to 8
 * ranks.  iterate: x as for spmvtk_dist_spmv_iterate; a flag wait that times
 * out returns SPMVTK_ERR_DATA. */
typedef struct spmvtk_dist_push spmvtk_dist_push;
spmvtk_status spmvtk_dist_push_create(const spmvtk_dist* d, const spmvtk_matrix* shard,
                                      spmvtk_kernel kernel, int sparse, spmvtk_dist_push** out);
spmvtk_status spmvtk_dist_push_iterate(spmvtk_dist_push* p, double* x, int64_t steps,
                                       double* seconds);
void spmvtk_dist_push_free(spmvtk_dist_push* p);

/* x ~ U(-1,1) from seed with the reference's raw-bit mapping. */
spmvtk_status spmvtk_gen_vector(int64_t n, uint64_t seed, double* out);

/* Reference-layout ELL footprint estimate and the device (GPU-layout) bytes
 * a conversion to `to` would allocate. */
spmvtk_status spmvtk_conversion_bytes(const spmvtk_matrix* m, spmvtk_format to,
                                      uint64_t* reference_estimate, uint64_t* device_bytes);

/* One CRS -> `to` conversion timed as the reference's measure_transformation
 * (autotune.cpp:122-128): wall clock in the library around the conversion,
 * the device synchronised before and after, allocation and the max-row
 * reduction included -- the t_trans of spmvtk_bench for any target format. */
spmvtk_status spmvtk_matrix_convert_timed(const spmvtk_matrix* m, spmvtk_format to,
                                          uint64_t max_bytes, spmvtk_matrix** out,
                                          double* seconds);

/* Median device time (seconds) of the kernels of one CRS -> `to` conversion
 * with outputs preallocated (allocation and host synchronisation excluded;
 * spmvtk_bench's t_trans includes them, as the reference's does). */
spmvtk_status spmvtk_transform_kernel_seconds(const spmvtk_matrix* m, spmvtk_format to,
                                              int repeats, double* seconds);

/* Grows the device memory pool by `bytes` once (allocate + free) and keeps
 * up to that many bytes cached after frees (the pool's release threshold;
 * default 2 GiB), so later stream-ordered allocations of handles are
 * sub-allocations. */
spmvtk_status spmvtk_reserve_device_memory(uint64_t bytes);

/* Compute metrics / amortization / D* helpers (autotune.cpp:36-60, :130-158). */
spmvtk_status spmvtk_compute_metrics(double t_crs, double t_ell, double t_trans,
                                     double* sp, double* tt, double* r);
/* returns -1 when the transformed kernel is not faster (never amortizes) */
spmvtk_status spmvtk_amortization_iterations(double t_crs, double t_ell, double t_trans,
                                             int64_t* k);
double spmvtk_find_d_star(const double* d_mat, const double* r, size_t count, double c);

/* Library build / device description (for reports). */
const char* spmvtk_version(void);

/* ---- streaming host SpMV -------------------------------------------------
 * A pipeline for many products with one handle and host vectors: submit
 * enqueues H2D(x) -> SpMV -> D2H(y) on separate streams with three device
 * staging slots and returns at once, so the copy-in of one product, the
 * SpMV of another and the copy-out of a third overlap (PCIe is full duplex).
 * x and y must stay untouched until spmvtk_pipeline_wait returns; pinned
 * host memory is needed for the copies to be asynchronous.  Every product
 * is exactly the one spmvtk_spmv computes. */
typedef struct spmvtk_pipeline spmvtk_pipeline;
spmvtk_status spmvtk_pipeline_create(const spmvtk_matrix* m, spmvtk_kernel kernel,
                                     spmvtk_pipeline** out);
spmvtk_status spmvtk_pipeline_submit(spmvtk_pipeline* p, const double* x, double* y);
spmvtk_status spmvtk_pipeline_wait(spmvtk_pipeline* p);
void spmvtk_pipeline_free(spmvtk_pipeline* p);

/* ---- multi-GPU exchange folded into the SpMV (SURVEY.md §8e stretch) ----
 * Row-block SpMV x_{t+1} = A x_t with one process per GPU: instead of an
 * all-gather after the product, the SpMV epilogue stores every result row
 * straight into the next-x buffers of the ranks that need it (peer memory
 * over NVLink / NVSwitch), and a flag per (source, step) orders the steps.
 *
 * Buffers live in cudaMalloc'ed memory shared through CUDA IPC handles.
 * dst[w] must point at THIS shard's first row inside rank w's buffer (so
 * row r of the shard lands at dst[w][r]); mask (device, one byte per local
 * row, may be NULL = all ranks) selects the ranks that read row r (bit w).
 * dst[local] is in this GPU's own memory: kernels that stage (the
 * entry-balanced CRS SpMV) write every row there first and copy each
 * finished tile of rows to the other destinations with coalesced stores. */
#define SPMVTK_MAX_PEERS 8
#define SPMVTK_IPC_HANDLE_BYTES 64
typedef struct spmvtk_push {
  double* dst[SPMVTK_MAX_PEERS];
  const uint8_t* mask;
  int32_t ndst;
  int32_t local; /* 0 <= local < ndst */
} spmvtk_push;
/* flag targets: ptr[w] = address of this rank's flag slot inside rank w's
 * flag array (system-scope release stores). */
typedef struct spmvtk_flag_targets {
  uint64_t* ptr[SPMVTK_MAX_PEERS];
  int32_t n;
} spmvtk_flag_targets;
/* Step synchronisation done INSIDE the pushed SpMV kernel: every CTA first
 * waits until wait_flags[s] >= wait_value (s < nwait; bounded by timeout_ns,
 * bit 0 of *status set on timeout), and the last CTA to finish (counter:
 * device word, zero, reset by the kernel) stores signal_value to every
 * signal target after all CTAs' pushes are fenced.  One launch per step. */
typedef struct spmvtk_push_sync {
  const uint64_t* wait_flags;
  int32_t nwait;
  uint64_t wait_value;
  uint64_t timeout_ns;
  uint32_t* status;
  spmvtk_flag_targets signal;
  uint64_t signal_value;
  uint32_t* counter;
} spmvtk_push_sync;

/* cudaMalloc + zero + IPC handle (handle: SPMVTK_IPC_HANDLE_BYTES bytes). */
spmvtk_status spmvtk_ipc_alloc(uint64_t bytes, void** dev_ptr, void* handle);
spmvtk_status spmvtk_ipc_free(void* dev_ptr);
/* Maps a peer's allocation (cudaIpcOpenMemHandle, lazy peer access). */
spmvtk_status spmvtk_ipc_open(const void* handle, void** dev_ptr);
spmvtk_status spmvtk_ipc_close(void* dev_ptr);
/* SpMV of a CRS (kernel CRS) or ELL (kernel ELL_INNER) handle whose result
 * rows are pushed to push->dst instead of a local y; sync (may be NULL)
 * folds the step's flag wait and signal into the same kernel. */
spmvtk_status spmvtk_spmv_device_push(const spmvtk_matrix* m, spmvtk_kernel kernel,
                                      const double* x, const spmvtk_push* push,
                                      const spmvtk_push_sync* sync);
/* After the preceding work on the stream: *targets->ptr[w] = value for all w
 * (system-scope release).  wait: until flags[s] >= value for s < n, or the
 * timeout (ns) passes, in which case bit 0 of *status (device) is set. */
spmvtk_status spmvtk_flags_signal(const spmvtk_flag_targets* targets, uint64_t value);
spmvtk_status spmvtk_flags_wait(const uint64_t* flags, int32_t n, uint64_t value,
                                uint64_t timeout_ns, uint32_t* status);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* SPMVTK_H */
