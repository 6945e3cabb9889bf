// kernels_convert.cu -- the run-time data transformations on sm_100a.
//
//   expand_ptr     CRS->COO-row row ids / CCS->COO-col column ids
//                  (convert.cpp:11-22, :55-66)
//   crs_to_ccs     Phase I: column histogram, device exclusive scan, cursor
//                  scatter, per-column fix-up that restores the reference's
//                  ascending-row order (convert.cpp:24-53)
//   crs_to_ell_*   zero-padded scatter into band-major (coalesced) or
//                  row-major ELL (convert.cpp:81-115)
//
// All pure data movement: HBM-bound, no arithmetic on values (fp64 bit
// patterns are moved, never computed), so results are bit-exact by
// construction.  Pointer expansion is warp-cooperative over a window of 32
// row starts held one per lane, so every lane does useful work regardless of
// the row-length distribution.
#include <algorithm>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "spmvtk/spmvtk_kernels.h"

using namespace spmvtk_dev;

namespace {

// ---- pointer expansion ---------------------------------------------------
__global__ void __launch_bounds__(256) k_expand_ptr(const int32_t* __restrict__ ptr,
                                                    int64_t n, int rows_per_warp,
                                                    int32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t rb = warp * rows_per_warp;
  if (rb >= n) return;
  const int64_t re = min(rb + rows_per_warp, n);
  const int32_t e0 = __ldg(ptr + rb), e1 = __ldg(ptr + re);
  SegWindow w;
  w.r0 = rb;
  w.load(ptr, re, lane);
  for (int32_t base = e0; base < e1; base += 32) {
    int32_t p = base + lane;
    int32_t seg = resolve_segment(w, ptr, re, lane, p, p < e1);
    if (p < e1) out[p] = seg;
  }
}

int g_warp_entries = 512;  // tuning: entries per warp chunk of the row-expanding kernels

int rows_per_warp_for(int64_t n, int64_t nnz) {
  // aim at ~g_warp_entries entries per warp chunk: small chunks, many
  // warps -- the last wave's tail shrinks (profiles/r01_tune_warp_entries.txt)
  double mean = n > 0 ? static_cast<double>(nnz) / static_cast<double>(n) : 1.0;
  int64_t r = 8;
  while (r < 8192 && static_cast<double>(r) * mean < static_cast<double>(g_warp_entries)) r <<= 1;
  return static_cast<int>(r);
}

// ---- CRS -> COO-row in one pass (convert.cpp:11-22) --------------------------
// Warp per chunk of rows: the chunk's entries are copied in 32-entry batches
// (coalesced loads / streaming stores of col and value) and the row id of
// each entry is resolved from the row pointers in the same pass.
__global__ void __launch_bounds__(256) k_crs_to_coo_row(const int32_t* __restrict__ ptr,
                                                        int64_t n, int rows_per_warp,
                                                        const int32_t* __restrict__ icol,
                                                        const double* __restrict__ val,
                                                        int32_t* __restrict__ out_row,
                                                        int32_t* __restrict__ out_col,
                                                        double* __restrict__ out_val) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t rb = warp * rows_per_warp;
  if (rb >= n) return;
  const int64_t re = min(rb + rows_per_warp, n);
  const int32_t e0 = __ldg(ptr + rb), e1 = __ldg(ptr + re);
  SegWindow w;
  w.r0 = rb;
  w.load(ptr, re, lane);
  constexpr int U = 8;
  for (int32_t base = e0; base < e1; base += 32 * U) {
    int32_t p[U], c[U], r[U];
    double v[U];
    uint32_t need = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      p[u] = base + u * 32 + lane;
      r[u] = 0;
      const bool ok = p[u] < e1;
      c[u] = ok ? ld_stream(icol + p[u]) : 0;
      v[u] = ok ? ld_stream(val + p[u]) : 0.0;
      if (ok) need |= 1u << u;
    }
    resolve_segments<U>(w, ptr, re, lane, p, r, need);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (p[u] < e1) {
        out_row[p[u]] = r[u];
        out_col[p[u]] = c[u];
        st_stream(out_val + p[u], v[u]);
      }
  }
}

// ---- CRS -> CCS ------------------------------------------------------------
// 16-byte (col, row, value) records of the partition passes
__device__ __forceinline__ double rec_val(const int4& r) { return __hiloint2double(r.w, r.z); }

// Bitonic sort (all comparators ascending, "flip" first stage) of the
// segment key[0..len) with payload; elements past len act as +inf and are
// never touched, so any len works and the sort is in place.
template <typename KeyPtr, typename ValPtr>
__device__ void block_bitonic(KeyPtr key, ValPtr val, int32_t len) {
  int32_t P = 1;
  while (P < len) P <<= 1;
  const int32_t half_work = P >> 1;
  for (int32_t size = 2; size <= P; size <<= 1) {
    const int32_t h = size >> 1;
    for (int32_t t = threadIdx.x; t < half_work; t += blockDim.x) {
      int32_t blk = t / h, off = t - blk * h;
      int32_t i = blk * size + off, jx = blk * size + size - 1 - off;
      if (jx < len && key[i] > key[jx]) {
        auto k = key[i]; key[i] = key[jx]; key[jx] = k;
        auto v = val[i]; val[i] = val[jx]; val[jx] = v;
      }
    }
    __syncthreads();
    for (int32_t d = h >> 1; d > 0; d >>= 1) {
      for (int32_t t = threadIdx.x; t < half_work; t += blockDim.x) {
        int32_t blk = t / d, off = t - blk * d;
        int32_t i = blk * 2 * d + off, jx = i + d;
        if (jx < len && key[i] > key[jx]) {
          auto k = key[i]; key[i] = key[jx]; key[jx] = k;
          auto v = val[i]; val[i] = val[jx]; val[jx] = v;
        }
      }
      __syncthreads();
    }
  }
}

// ---- CRS -> CCS, bucketed (no global atomics) -------------------------------
// Columns are grouped into NB buckets of CB = 2^shift consecutive columns
// (~4k entries per bucket).  The CRS is split into kSlices row ranges of
// equal entry counts (one per SM).
//   1. k_bkt_count   slice-local bucket histograms in shared memory ->
//                    T[b * kSlices + slice]; also the number of non-empty
//                    runs (two-pass choice) and each slice's bucket window
//   2. exclusive scan of T (bucket-major) -> each (bucket, slice) owns a run
//   3. k_bkt_scatter each slice re-reads its rows and appends 16-byte
//                    records (col, row, value) to its runs with shared-memory
//                    cursors: writes are kSlices x NB sequential streams that
//                    fill whole sectors in L2 (variants: staged through shared
//                    memory for coalesced run writes -- a coarse pass + refine
//                    when columns scatter over many runs, or per slice over a
//                    banded matrix's bucket window, k_bkt_scatter_single)
//   4. k_bkt_sort    one CTA per bucket: counting sort by column in shared
//                    memory, then each entry goes to its rank by row inside
//                    its column (rows are distinct within a column, so this
//                    restores the reference's order, convert.cpp:43-51);
//                    col_ptr, row_idx, values (and for COO-col the column,
//                    Phase II fused) written from there.
// Buckets too large for shared memory take a global-memory path.
constexpr int kSlices = 3 * 148;  // max slices (3 CTAs per SM, 64 KB histograms)
int g_ccs_slices = 148;           // tuning: slices actually used (one per SM)
int g_ccs_threads = 1024;         // tuning: threads of the count/scatter CTAs
constexpr int kBktItems = 12;  // records per sort thread (bucket capacity = threads * 12)
int g_ccs_sort_threads = 512;  // tuning: 256 or 512 (bucket target = 2/3 of the capacity)
int g_ccs_sort_items = 0;      // tuning: records per sort thread (0 = from the column window, 8, 12)
int g_ccs_window = 1;          // tuning: single pass stages slices with <= 1024-bucket windows

// Two-pass or single-pass partition is decided on the device from the
// number of non-empty (fine bucket, slice) runs counted by k_bkt_count: few
// runs (banded matrices) keep their write streams L2-resident in one pass;
// many runs (scattered columns) go through the coarse pass + refine.
__device__ int32_t d_two_pass_runs = 1 << 17;  // tuning: ccs_two_pass_runs
constexpr int kStageU = 4;        // 32-entry batches per lane per staged step
constexpr int kStageMaxB = 1024;  // buckets (or bucket window) of the staged scatter
__device__ __forceinline__ bool two_pass(const int32_t* runs) {
  return runs != nullptr && *runs > d_two_pass_runs;
}

__global__ void k_slice_rows(const int32_t* __restrict__ irp, int64_t n, int ns,
                             int32_t* slice_row) {
  // slice s starts at the first row whose start >= s * nnz / ns: one warp
  // per slice, 32-way search (a handful of dependent loads, not log2(n))
  const int s = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (s > ns) return;
  const int64_t nnz = irp[n];
  const int64_t target = nnz * s / ns;
  int64_t lo = -1, hi = n;  // irp[lo] < target <= irp[hi] (irp[-1] = -inf)
  while (hi - lo > 1) {
    const int64_t probe = lo + 1 + ((hi - lo - 1) * lane) / 32;
    const unsigned m = __ballot_sync(kFull, __ldg(irp + probe) < target);
    const int64_t nlo = m ? __shfl_sync(kFull, probe, 31 - __clz(m)) : lo;
    const int64_t nhi = ~m ? __shfl_sync(kFull, probe, __ffs(~m) - 1) : hi;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) slice_row[s] = static_cast<int32_t>(s == ns ? n : hi);
}

__global__ void __launch_bounds__(1024) k_bkt_count(const int32_t* __restrict__ irp,
                                                           const int32_t* __restrict__ icol,
                                                           const int32_t* __restrict__ slice_row,
                                                           int shift, int nb, int32_t* T,
                                                           int fshift, int32_t* Tc,
                                                           int32_t* runs, int32_t* win) {
  extern __shared__ int32_t s_hist[];
  __shared__ int32_t s_lo, s_hi, s_chg, s_smp;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) s_hist[b] = 0;
  if (threadIdx.x == 0) {
    s_lo = nb;
    s_hi = -1;
    s_chg = 0;
    s_smp = 0;
  }
  __syncthreads();
  const int32_t e0 = irp[slice_row[blockIdx.x]], e1 = irp[slice_row[blockIdx.x + 1]];
  const int32_t step = static_cast<int32_t>(blockDim.x);
  const int lane = threadIdx.x & 31;
  int32_t chg = 0, smp = 0;
  // 16-byte loads over the 4-aligned body, two per thread in flight (8
  // columns); the unaligned head and the tail one column per thread
  // (aligned by address: the lower ABI accepts any 4-byte aligned icol)
  const int32_t mis = static_cast<int32_t>((reinterpret_cast<uintptr_t>(icol) >> 2) & 3);
  const int32_t a0 = min(e1, ((e0 + mis + 3) & ~3) - mis);
  const int32_t a1 = max(a0, ((e1 + mis) & ~3) - mis);
  for (int32_t p = e0 + static_cast<int32_t>(threadIdx.x); p < a0; p += step)
    atomicAdd(&s_hist[ld_stream(icol + p) >> shift], 1);
  for (int32_t p = a1 + static_cast<int32_t>(threadIdx.x); p < e1; p += step)
    atomicAdd(&s_hist[ld_stream(icol + p) >> shift], 1);
  const int4* __restrict__ q4 = reinterpret_cast<const int4*>(icol + a0);
  const int32_t nq = (a1 - a0) >> 2;
  int32_t q = static_cast<int32_t>(threadIdx.x);
  for (int it = 0; q + step < nq; q += 2 * step, ++it) {
    const int4 u = ld_stream4(q4 + q), w = ld_stream4(q4 + q + step);
    if (win && (it & 7) == 0) {  // sample: is an entry in its CRS predecessor's bucket?
      smp += 3;
      chg += ((u.y >> shift) != (u.x >> shift)) + ((u.z >> shift) != (u.y >> shift)) +
             ((u.w >> shift) != (u.z >> shift));
    }
    atomicAdd(&s_hist[u.x >> shift], 1);
    atomicAdd(&s_hist[u.y >> shift], 1);
    atomicAdd(&s_hist[u.z >> shift], 1);
    atomicAdd(&s_hist[u.w >> shift], 1);
    atomicAdd(&s_hist[w.x >> shift], 1);
    atomicAdd(&s_hist[w.y >> shift], 1);
    atomicAdd(&s_hist[w.z >> shift], 1);
    atomicAdd(&s_hist[w.w >> shift], 1);
  }
  for (; q < nq; q += step) {
    const int4 u = ld_stream4(q4 + q);
    atomicAdd(&s_hist[u.x >> shift], 1);
    atomicAdd(&s_hist[u.y >> shift], 1);
    atomicAdd(&s_hist[u.z >> shift], 1);
    atomicAdd(&s_hist[u.w >> shift], 1);
  }
  (void)lane;
  __syncthreads();
  int32_t nz = 0, lo = nb, hi = -1;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    T[static_cast<int64_t>(b) * gridDim.x + blockIdx.x] = s_hist[b];
    if (s_hist[b]) {
      ++nz;
      lo = min(lo, b);
      hi = max(hi, b);
    }
  }
  if (runs) {
    nz = __reduce_add_sync(kFull, static_cast<unsigned>(nz));
    if ((threadIdx.x & 31) == 0 && nz) atomicAdd(runs, nz);
  }
  if (win) {  // the slice's non-empty buckets span [lo, hi]
    lo = __reduce_min_sync(kFull, lo);
    hi = __reduce_max_sync(kFull, hi);
    chg = __reduce_add_sync(kFull, static_cast<unsigned>(chg));
    smp = __reduce_add_sync(kFull, static_cast<unsigned>(smp));
    if (lane == 0) {
      atomicMin(&s_lo, lo);
      atomicMax(&s_hi, hi);
      atomicAdd(&s_chg, chg);
      atomicAdd(&s_smp, smp);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // staged only where most CRS neighbours change bucket: runs of one
      // bucket inside a row already give the cursor scatter contiguous
      // stores (27-point stencil), and it skips the staging barriers
      const bool scattered = 2 * static_cast<int64_t>(s_chg) > s_smp;
      win[2 * blockIdx.x] = s_hi < 0 ? 0 : s_lo;
      win[2 * blockIdx.x + 1] = s_hi < 0 ? 0 : scattered ? s_hi + 1 - s_lo : kStageMaxB + 1;
    }
  }
  if (Tc) {  // coarse buckets of 2^fshift fine buckets (two-pass partition)
    const int F = 1 << fshift, nc = (nb + F - 1) >> fshift;
    for (int c = threadIdx.x; c < nc; c += blockDim.x) {
      int32_t sum = 0;
      for (int f = 0; f < F; ++f) {
        const int b = c * F + ((f + c) & (F - 1));  // rotated: spreads the banks
        if (b < nb) sum += s_hist[b];
      }
      Tc[static_cast<int64_t>(c) * gridDim.x + blockIdx.x] = sum;
    }
  }
}

// cursor scatter: every lane appends its record at a shared cursor of its bucket
__device__ __forceinline__ void bkt_scatter_cursor(
    const int32_t* __restrict__ irp, const int32_t* __restrict__ icol,
    const double* __restrict__ val, const int32_t* __restrict__ slice_row, int shift, int nb,
    const int32_t* __restrict__ Toff, int4* __restrict__ rec, int32_t* s_cur) {
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    s_cur[b] = Toff[static_cast<int64_t>(b) * gridDim.x + blockIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int64_t r_begin = slice_row[blockIdx.x], r_end = slice_row[blockIdx.x + 1];
  // every warp takes an equal share of the slice's ENTRIES (skewed rows
  // would unbalance a split by rows) ...
  const int32_t E0 = __ldg(irp + r_begin), E1 = __ldg(irp + r_end);
  const int64_t tot = E1 - E0;
  const int32_t p0 = E0 + static_cast<int32_t>(tot * warp / nwarps);
  const int32_t p1 = E0 + static_cast<int32_t>(tot * (warp + 1) / nwarps);
  if (p0 >= p1) return;
  // ... and finds the row holding its first entry by a 32-way search
  int64_t lo = r_begin, hi = r_end;  // irp[lo] <= p0 < irp[hi]
  while (hi - lo > 1) {
    const int64_t probe = lo + 1 + ((hi - lo - 1) * lane) / 32;
    const unsigned m = __ballot_sync(kFull, __ldg(irp + probe) <= p0);
    const int64_t nlo = m ? __shfl_sync(kFull, probe, 31 - __clz(m)) : lo;
    const int64_t nhi = ~m ? __shfl_sync(kFull, probe, __ffs(~m) - 1) : hi;
    lo = nlo;
    hi = nhi;
  }
  SegWindow w;
  w.r0 = lo;
  w.load(irp, r_end, lane);
  constexpr int kU = 4;  // 32-entry batches per lane per step
  int32_t c[kU];
  double v[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int32_t p = p0 + u * 32 + lane;
    c[u] = p < p1 ? ld_stream(icol + p) : 0;
    v[u] = p < p1 ? ld_stream(val + p) : 0.0;
  }
  for (int32_t base = p0; base < p1; base += 32 * kU) {
    int32_t cn[kU];
    double vn[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {  // next step's loads fly during this one
      const int32_t p = base + 32 * kU + u * 32 + lane;
      cn[u] = p < p1 ? ld_stream(icol + p) : 0;
      vn[u] = p < p1 ? ld_stream(val + p) : 0.0;
    }
    int32_t pp[kU], row[kU];
    uint32_t need = 0;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      pp[u] = base + u * 32 + lane;
      row[u] = 0;
      if (pp[u] < p1) need |= 1u << u;
    }
    resolve_segments<kU>(w, irp, r_end, lane, pp, row, need);
    int32_t slot[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)  // independent shared atomics, back to back
      slot[u] = pp[u] < p1 ? atomicAdd(&s_cur[c[u] >> shift], 1) : 0;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (pp[u] < p1)
        rec[slot[u]] = make_int4(c[u], row[u], __double2loint(v[u]), __double2hiint(v[u]));
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      c[u] = cn[u];
      v[u] = vn[u];
    }
  }
}

__global__ void __launch_bounds__(1024) k_bkt_scatter(
    const int32_t* __restrict__ irp, const int32_t* __restrict__ icol,
    const double* __restrict__ val, const int32_t* __restrict__ slice_row, int shift, int nb,
    const int32_t* __restrict__ Toff, int4* __restrict__ rec, const int32_t* runs, bool as_two) {
  if (runs && two_pass(runs) != as_two) return;
  extern __shared__ int32_t s_dyn[];
  bkt_scatter_cursor(irp, icol, val, slice_row, shift, nb, Toff, rec, s_dyn);
}

// Staged variant for at most kStageMaxB buckets (the coarse pass, or a
// single pass over few buckets): the 32 warps advance in lock step, 128
// entries each per step; the step's 4096 records are counting-sorted by
// bucket in shared memory and written out run by run, so consecutive lanes
// store consecutive addresses instead of 32 scattered 16-byte records.
int g_stage_threads = 1024;  // tuning: 1024 (one CTA per slice per SM) or 512

// Buckets [blo, blo + nbw) (nbw <= kStageMaxB) are renumbered from 0: a
// window of a banded matrix's buckets, or all of them.
template <int kStageThreads>
__device__ __forceinline__ void bkt_scatter_staged(
    const int32_t* __restrict__ irp, const int32_t* __restrict__ icol,
    const double* __restrict__ val, const int32_t* __restrict__ slice_row, int shift,
    int32_t blo, int nbw, const int32_t* __restrict__ Toff, int4* __restrict__ rec,
    int4* s_rec /* kStageThreads * kStageU records */) {
  constexpr int kP = kStageMaxB / kStageThreads;  // buckets owned per thread
  // run cursors double-buffered by step parity: the owner of a bucket
  // advances next step's cursor while this step's copy-out still reads its
  // own, so no barrier separates the copy-out from the next step (5 barriers
  // per step instead of 7; each thread zeroes its counters as it reads them)
  __shared__ int32_t s_cur[2][kStageMaxB], s_cnt[kStageMaxB], s_off[kStageMaxB];
  __shared__ int32_t s_wsum[kStageThreads / 32];
  __shared__ int32_t s_total;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = kStageThreads / 32;
#pragma unroll
  for (int j = 0; j < kP; ++j) {
    const int b = tid * kP + j;
    if (b < nbw) {
      s_cur[0][b] = Toff[static_cast<int64_t>(b + blo) * gridDim.x + blockIdx.x];
      s_cnt[b] = 0;
    }
  }
  const int64_t r_begin = slice_row[blockIdx.x], r_end = slice_row[blockIdx.x + 1];
  const int32_t E0 = __ldg(irp + r_begin), E1 = __ldg(irp + r_end);
  const int64_t tot = E1 - E0;
  const int32_t p0 = E0 + static_cast<int32_t>(tot * warp / nwarps);
  const int32_t p1 = E0 + static_cast<int32_t>(tot * (warp + 1) / nwarps);
  const int steps = static_cast<int>(((tot + nwarps - 1) / nwarps + 32 * kStageU - 1) /
                                     (32 * kStageU));
  int64_t lo = r_begin, hi = r_end;  // row holding p0: irp[lo] <= p0 < irp[hi]
  if (p0 < p1) {
    while (hi - lo > 1) {
      const int64_t probe = lo + 1 + ((hi - lo - 1) * lane) / 32;
      const unsigned m = __ballot_sync(kFull, __ldg(irp + probe) <= p0);
      const int64_t nlo = m ? __shfl_sync(kFull, probe, 31 - __clz(m)) : lo;
      const int64_t nhi = ~m ? __shfl_sync(kFull, probe, __ffs(~m) - 1) : hi;
      lo = nlo;
      hi = nhi;
    }
  }
  SegWindow w;
  w.r0 = lo;
  w.load(irp, r_end, lane);
  int32_t c[kStageU];
  double v[kStageU];
#pragma unroll
  for (int u = 0; u < kStageU; ++u) {
    const int32_t p = p0 + u * 32 + lane;
    c[u] = p < p1 ? ld_stream(icol + p) : 0;
    v[u] = p < p1 ? ld_stream(val + p) : 0.0;
  }
  __syncthreads();
  for (int st = 0; st < steps; ++st) {
    const int32_t base = p0 + st * 32 * kStageU;
    int32_t pp[kStageU], row[kStageU], rk[kStageU], cn[kStageU];
    double vn[kStageU];
    uint32_t need = 0;
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {  // the next step's loads fly across the barriers
      const int32_t p = base + 32 * kStageU + u * 32 + lane;
      cn[u] = p < p1 ? ld_stream(icol + p) : 0;
      vn[u] = p < p1 ? ld_stream(val + p) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
      pp[u] = base + u * 32 + lane;
      row[u] = 0;
      if (pp[u] < p1) need |= 1u << u;
    }
    resolve_segments<kStageU>(w, irp, r_end, lane, pp, row, need);
#pragma unroll
    for (int u = 0; u < kStageU; ++u)
      rk[u] = pp[u] < p1 ? atomicAdd(&s_cnt[(c[u] >> shift) - blo], 1) : 0;
    __syncthreads();
    // exclusive scan of the step's bucket counts (thread t owns buckets
    // [t*kP, t*kP + kP))
    int32_t loc[kP];
    int32_t x = 0;
#pragma unroll
    for (int j = 0; j < kP; ++j) {
      const int b = tid * kP + j;
      loc[j] = b < nbw ? s_cnt[b] : 0;
      if (b < nbw) s_cnt[b] = 0;  // read once: free for the next step's counts
      x += loc[j];
    }
    int32_t inc = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t t = __shfl_up_sync(kFull, inc, d);
      if (lane >= d) inc += t;
    }
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const int32_t wv = lane < nwarps ? s_wsum[lane] : 0;
      int32_t wi = wv;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int32_t t = __shfl_up_sync(kFull, wi, d);
        if (lane >= d) wi += t;
      }
      if (lane < nwarps) s_wsum[lane] = wi - wv;
      if (lane == nwarps - 1) s_total = wi;
    }
    __syncthreads();
    const int par = st & 1;
    {
      int32_t e = s_wsum[warp] + inc - x;
#pragma unroll
      for (int j = 0; j < kP; ++j) {
        const int b = tid * kP + j;
        if (b < nbw) {
          s_off[b] = e;
          s_cur[par ^ 1][b] = s_cur[par][b] + loc[j];
        }
        e += loc[j];
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kStageU; ++u)
      if (pp[u] < p1)
        s_rec[s_off[(c[u] >> shift) - blo] + rk[u]] =
            make_int4(c[u], row[u], __double2loint(v[u]), __double2hiint(v[u]));
    __syncthreads();
    const int32_t count = s_total;
    for (int32_t i = tid; i < count; i += kStageThreads) {
      const int4 r = s_rec[i];
      const int b = (r.x >> shift) - blo;
      rec[s_cur[par][b] + i - s_off[b]] = r;
    }
    // no barrier: the next step's first shared writes (its counts) come after
    // this step's reads of s_cnt, and its offsets, cursors and staged records
    // only after its own first barrier, which every thread reaches after its
    // copy-out
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
      c[u] = cn[u];
      v[u] = vn[u];
    }
  }
}

template <int kStageThreads>
__global__ void __launch_bounds__(kStageThreads) k_bkt_scatter_staged(
    const int32_t* __restrict__ irp, const int32_t* __restrict__ icol,
    const double* __restrict__ val, const int32_t* __restrict__ slice_row, int shift, int nb,
    const int32_t* __restrict__ Toff, int4* __restrict__ rec, const int32_t* runs, bool as_two) {
  if (runs && two_pass(runs) != as_two) return;
  extern __shared__ int4 s_dyn4[];
  bkt_scatter_staged<kStageThreads>(irp, icol, val, slice_row, shift, 0, nb, Toff, rec, s_dyn4);
}

// Single pass over more buckets than the staged scatter holds: each slice
// (CTA) picks its scatter from the window k_bkt_count measured -- staged over
// its bucket window when that is narrow and CRS neighbours mostly change
// bucket (banded random columns), else the cursor scatter.  One launch for
// both, so the choice costs no host round trip and no idle CTAs.
__global__ void __launch_bounds__(1024) k_bkt_scatter_single(
    const int32_t* __restrict__ irp, const int32_t* __restrict__ icol,
    const double* __restrict__ val, const int32_t* __restrict__ slice_row, int shift, int nb,
    const int32_t* __restrict__ Toff, int4* __restrict__ rec, const int32_t* runs,
    const int32_t* __restrict__ win) {
  if (runs && two_pass(runs)) return;
  const int32_t blo = win[2 * blockIdx.x];
  const int nbw = win[2 * blockIdx.x + 1];
  if (nbw == 0) return;  // empty slice
  extern __shared__ int4 s_dyn4[];
  if (nbw <= kStageMaxB)
    bkt_scatter_staged<1024>(irp, icol, val, slice_row, shift, blo, nbw, Toff, rec, s_dyn4);
  else
    bkt_scatter_cursor(irp, icol, val, slice_row, shift, nb, Toff, rec,
                       reinterpret_cast<int32_t*>(s_dyn4));
}

// Two-pass partition, second pass: the coarse-partitioned records are cut
// into chunks of kRefineItems; a chunk's fine buckets form a window (its
// records lie in a contiguous range of coarse buckets); the chunk claims a
// run per fine bucket with one global atomic (fcur) and appends its records
// there with shared cursors, so every run is a contiguous write.
constexpr int kRefineThreads = 512;
constexpr int kRefinePer = 8;
constexpr int kRefineItems = kRefineThreads * kRefinePer;
constexpr int kRefineWin = 4096;

__global__ void __launch_bounds__(kRefineThreads) k_bkt_refine(
    const int4* __restrict__ rec, int64_t nnz, int shift, int fshift,
    const int32_t* __restrict__ Toff, int ns, int32_t* __restrict__ fcur,
    int4* __restrict__ rec2, const int32_t* runs) {
  // persistent CTAs walk the chunks, so in single-pass mode the launch
  // costs a few hundred CTAs that exit at once, not one per chunk
  if (!two_pass(runs)) return;
  __shared__ int32_t s_cnt[kRefineWin];
  for (int64_t q0 = static_cast<int64_t>(blockIdx.x) * kRefineItems; q0 < nnz;
       q0 += static_cast<int64_t>(gridDim.x) * kRefineItems) {
    const int32_t len = static_cast<int32_t>(min(static_cast<int64_t>(kRefineItems), nnz - q0));
    int4 r[kRefinePer];
#pragma unroll
    for (int k = 0; k < kRefinePer; ++k) {
      const int32_t q = static_cast<int32_t>(threadIdx.x) + k * kRefineThreads;
      if (q < len) r[k] = ld_stream4(rec + q0 + q);
    }
    const int32_t b_lo = ((__ldg(&rec[q0].x) >> shift) >> fshift) << fshift;
    const int32_t b_hi = (((__ldg(&rec[q0 + len - 1].x) >> shift) >> fshift) + 1) << fshift;
    const int32_t win = b_hi - b_lo;
    if (win > kRefineWin) {  // many tiny coarse buckets: global cursors
#pragma unroll
      for (int k = 0; k < kRefinePer; ++k) {
        const int32_t q = static_cast<int32_t>(threadIdx.x) + k * kRefineThreads;
        if (q < len) {
          const int32_t b = r[k].x >> shift;
          rec2[Toff[static_cast<int64_t>(b) * ns] + atomicAdd(&fcur[b], 1)] = r[k];
        }
      }
      continue;  // win is CTA-uniform: every thread takes this branch
    }
    for (int i = threadIdx.x; i < win; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRefinePer; ++k) {
      const int32_t q = static_cast<int32_t>(threadIdx.x) + k * kRefineThreads;
      if (q < len) atomicAdd(&s_cnt[(r[k].x >> shift) - b_lo], 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < win; i += blockDim.x) {
      const int32_t c = s_cnt[i];
      if (c) {
        const int64_t b = b_lo + i;
        s_cnt[i] = Toff[b * ns] + atomicAdd(&fcur[b], c);
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRefinePer; ++k) {
      const int32_t q = static_cast<int32_t>(threadIdx.x) + k * kRefineThreads;
      if (q < len) rec2[atomicAdd(&s_cnt[(r[k].x >> shift) - b_lo], 1)] = r[k];
    }
    __syncthreads();  // s_cnt is reused by the next chunk
  }
}

// one CTA per bucket; dynamic smem: cnt[cb+1] | s_val | s_row | s_col (kBktCap each)
constexpr int32_t kRankMax = 256;  // longer columns take the block network
template <int kBktThreads, int kItems = kBktItems, int kMinBlocks = 1>
__global__ void __launch_bounds__(kBktThreads, kMinBlocks) k_bkt_sort(
    const int4* rec1, const int4* rec2, const int32_t* runs,
    const int32_t* __restrict__ Toff, int64_t n, int shift,
    int nb, int ns, int32_t* __restrict__ col_ptr, int32_t* __restrict__ row_idx,
    double* __restrict__ out_val, int32_t* big_queue, int32_t* big_len,
    int32_t* __restrict__ out_col) {  // out_col: COO-col column indices (Phase II), or null
  constexpr int kBktCap = kBktThreads * kItems;
  const int4* __restrict__ rec = two_pass(runs) ? rec2 : rec1;
  extern __shared__ unsigned char s_raw[];
  const int cb = 1 << shift;
  int32_t* cnt = reinterpret_cast<int32_t*>(s_raw);  // cb + 1 entries
  double* s_val = reinterpret_cast<double*>(s_raw + ((static_cast<size_t>(cb + 1) * 4 + 15) & ~15));
  int32_t* s_row = reinterpret_cast<int32_t*>(s_val + kBktCap);
  uint16_t* s_col = reinterpret_cast<uint16_t*>(s_row + kBktCap);
  const int b = blockIdx.x;
  const int32_t bs = Toff[static_cast<int64_t>(b) * ns];
  const int32_t be = (b + 1 < nb) ? Toff[static_cast<int64_t>(b + 1) * ns]
                                  : Toff[static_cast<int64_t>(nb) * ns];
  const int64_t c0 = static_cast<int64_t>(b) << shift;
  const int ncols = static_cast<int>(min(static_cast<int64_t>(cb), n - c0));
  const int32_t len = be - bs;
  const bool fits = len <= kBktCap;
  for (int i = threadIdx.x; i <= cb; i += blockDim.x) cnt[i] = 0;
  // records stay in registers between the count and the placement
  int4 r[kItems];
  if (fits) {
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const int32_t q = static_cast<int32_t>(threadIdx.x) + k * kBktThreads;
      if (q < len) r[k] = ld_stream4(rec + bs + q);
    }
  }
  __syncthreads();
  if (fits) {
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const int32_t q = static_cast<int32_t>(threadIdx.x) + k * kBktThreads;
      if (q < len) atomicAdd(&cnt[r[k].x - c0], 1);
    }
  } else {
    for (int32_t q = threadIdx.x; q < len; q += blockDim.x)
      atomicAdd(&cnt[__ldg(&rec[bs + q].x) - c0], 1);
  }
  __syncthreads();
  // block exclusive scan of cnt[0..cb) (cb a power of two <= 4096): each
  // thread owns cb/512 consecutive counters
  {
    __shared__ int32_t s_warp[kBktThreads / 32];
    const int per = cb > kBktThreads ? cb / kBktThreads : 1;
    const int i0 = static_cast<int>(threadIdx.x) * per;
    constexpr int kPer = 4096 / kBktThreads;
    int32_t loc[kPer];
    int32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if (k < per && i0 + k < cb) {
        loc[k] = cnt[i0 + k];
        sum += loc[k];
      }
    int32_t inc = sum;
    const int ln = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t t = __shfl_up_sync(kFull, inc, d);
      if (ln >= d) inc += t;
    }
    if (ln == 31) s_warp[wp] = inc;
    __syncthreads();
    if (wp == 0) {
      const int32_t wv = ln < kBktThreads / 32 ? s_warp[ln] : 0;
      int32_t wi = wv;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int32_t t = __shfl_up_sync(kFull, wi, d);
        if (ln >= d) wi += t;
      }
      if (ln < kBktThreads / 32) s_warp[ln] = wi - wv;
      if (ln == kBktThreads / 32 - 1) cnt[cb] = wi;
    }
    __syncthreads();
    int32_t run = s_warp[wp] + inc - sum;
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if (k < per && i0 + k < cb) {
        cnt[i0 + k] = run;
        run += loc[k];
      }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ncols; i += blockDim.x) col_ptr[c0 + i] = bs + cnt[i];
  if (b == nb - 1 && threadIdx.x == 0) col_ptr[n] = be;
  __syncthreads();  // cnt becomes a cursor array below
  if (len > kBktCap) {
    // oversized bucket: place into the final arrays with shared cursors,
    // then sort every column of it in global memory (k_bkt_sort_big)
    __syncthreads();
    for (int32_t q = threadIdx.x; q < len; q += blockDim.x) {
      const int4 r = rec[bs + q];
      const int32_t slot = atomicAdd(&cnt[r.x - c0], 1);
      row_idx[bs + slot] = r.y;
      out_val[bs + slot] = rec_val(r);
      if (out_col) out_col[bs + slot] = r.x;
    }
    if (threadIdx.x == 0) big_queue[atomicAdd(big_len, 1)] = b;
    return;
  }
  // place by column (shared cursors; order inside a column arbitrary)
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int32_t q = static_cast<int32_t>(threadIdx.x) + k * kBktThreads;
    if (q < len) {
      const int32_t col = r[k].x - static_cast<int32_t>(c0);
      const int32_t slot = atomicAdd(&cnt[col], 1);
      s_row[slot] = r[k].y;
      s_val[slot] = rec_val(r[k]);
      s_col[slot] = static_cast<uint16_t>(col);
    }
  }
  __shared__ int s_long;
  if (threadIdx.x == 0) s_long = 0;
  __syncthreads();
  // cnt[i] now holds the END of column i; column i spans [end(i-1), end(i)).
  // Rows are distinct inside a column, so an entry's final position is its
  // rank by row there: one thread per slot counts the smaller rows (lanes of
  // a warp mostly share a column -> broadcast reads) and writes it out.
  // (Measured: staging the permutation for coalesced writes, or ranking 4
  // slots per thread, were both slower.)
  for (int32_t q = threadIdx.x; q < len; q += blockDim.x) {
    const int col = s_col[q];
    const int32_t a = col ? cnt[col - 1] : 0, e = cnt[col];
    if (e - a > kRankMax) {
      s_long = 1;
      continue;
    }
    const int32_t row = s_row[q];
    int32_t rank = 0;
    for (int32_t j = a; j < e; ++j) rank += s_row[j] < row;
    row_idx[bs + a + rank] = row;
    st_stream(out_val + bs + a + rank, s_val[q]);
    if (out_col) out_col[bs + a + rank] = static_cast<int32_t>(c0) + col;
  }
  __syncthreads();
  if (!s_long) return;
  // long columns: block bitonic network in shared memory, then copy out
  for (int i = 0; i < ncols; ++i) {
    const int32_t a = i ? cnt[i - 1] : 0, e = cnt[i];
    if (e - a <= kRankMax) continue;
    block_bitonic(s_row + a, s_val + a, e - a);
    for (int32_t q = a + threadIdx.x; q < e; q += blockDim.x) {
      row_idx[bs + q] = s_row[q];
      st_stream(out_val + bs + q, s_val[q]);
      if (out_col) out_col[bs + q] = static_cast<int32_t>(c0) + i;
    }
    __syncthreads();
  }
}

// columns of oversized buckets: sort each column segment in place
__global__ void __launch_bounds__(512) k_bkt_sort_big(const int32_t* __restrict__ col_ptr,
                                                      int64_t n, int shift, int32_t* row_idx,
                                                      double* vals, const int32_t* big_queue,
                                                      const int32_t* big_len) {
  const int32_t count = *big_len;
  for (int32_t q = blockIdx.x; q < count; q += gridDim.x) {
    const int64_t c0 = static_cast<int64_t>(big_queue[q]) << shift;
    const int64_t c1 = min(c0 + (int64_t(1) << shift), n);
    for (int64_t c = c0; c < c1; ++c) {
      const int32_t a = col_ptr[c], len = col_ptr[c + 1] - a;
      if (len > 1) block_bitonic(row_idx + a, vals + a, len);
      __syncthreads();
    }
  }
}

// ---- CRS -> ELL ------------------------------------------------------------
// Band-major (the reference layout, convert.cpp:101-113): a block stages
// R rows x KC bands of the CRS (row-contiguous, coalesced reads) in shared
// memory and writes them out band by band (R consecutive rows per band,
// coalesced writes).  R*KC = 2048 slots per stage.
template <int KC>
__global__ void __launch_bounds__(256) k_crs_to_ell_cm(int64_t n, int32_t nz, int64_t ld,
                                                       const int32_t* __restrict__ irp,
                                                       const int32_t* __restrict__ icol,
                                                       const double* __restrict__ val,
                                                       double* __restrict__ out_val,
                                                       int32_t* __restrict__ out_col,
                                                       int32_t* __restrict__ out_count,
                                                       int64_t pad_base) {
  constexpr int R = 2048 / KC;
  __shared__ int32_t s_ptr[R + 1];
  __shared__ double s_v[R][KC + 1];
  __shared__ int32_t s_c[R][KC + 1];
  __shared__ int32_t s_maxlen;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * R;
  if (threadIdx.x == 0) s_maxlen = 0;
  for (int t = threadIdx.x; t <= R; t += blockDim.x)
    s_ptr[t] = __ldg(irp + min(r0 + t, n));
  __syncthreads();
  for (int t = threadIdx.x; t < R; t += blockDim.x) {
    const int32_t len = s_ptr[t + 1] - s_ptr[t];
    if (r0 + t < n) out_count[r0 + t] = len;
    atomicMax(&s_maxlen, len);
  }
  __syncthreads();
  const int32_t maxlen = s_maxlen;
  for (int32_t k0 = 0; k0 < nz; k0 += KC) {
    if (k0 >= maxlen) {
      // bands past every row of the block: padding only, no staging -- a
      // thread stores a row PAIR (16-byte zero values, 8-byte own-row
      // columns; R and ld are even, so pairs never straddle ld)
      const int kc = min(KC, nz - k0);
      for (int f = threadIdx.x; f < kc * (R / 2); f += blockDim.x) {
        const int kk = f / (R / 2), row = 2 * (f % (R / 2));
        const int64_t i = r0 + row;
        if (i >= ld) continue;
        const int64_t slot = static_cast<int64_t>(k0 + kk) * ld + i;
        st_stream2(reinterpret_cast<double2*>(out_val + slot), make_double2(0.0, 0.0));
        *reinterpret_cast<int2*>(out_col + slot) =
            make_int2(static_cast<int32_t>(pad_base + (i < n ? i : 0)),
                      static_cast<int32_t>(pad_base + (i + 1 < n ? i + 1 : 0)));
      }
      continue;  // k0 >= maxlen is block-uniform
    }
    for (int f = threadIdx.x; f < R * KC; f += blockDim.x) {
      const int row = f / KC, kk = f % KC;
      const int32_t len = s_ptr[row + 1] - s_ptr[row];
      if (k0 + kk < len) {
        const int32_t p = s_ptr[row] + k0 + kk;
        s_v[row][kk] = ld_stream(val + p);
        s_c[row][kk] = ld_stream(icol + p);
      }
    }
    __syncthreads();
    for (int f = threadIdx.x; f < R * KC; f += blockDim.x) {
      const int kk = f / R, row = f % R;
      const int32_t k = k0 + kk;
      const int64_t i = r0 + row;
      if (k < nz && i < ld) {
        // rows in [n, ld) are layout padding (value 0, column 0) so that
        // the 128-bit SpMV loads of the last row pair stay in bounds
        const int32_t len = s_ptr[row + 1] - s_ptr[row];
        const int64_t slot = static_cast<int64_t>(k) * ld + i;
        const bool real = k < len;
        st_stream(out_val + slot, real ? s_v[row][kk] : 0.0);
        out_col[slot] = real ? s_c[row][kk] : static_cast<int32_t>(pad_base + (i < n ? i : 0));
      }
    }
    __syncthreads();
  }
}

// Band-major, short bands (nz <= 32): the block's ROWS rows are one
// contiguous CRS range of at most ROWS*32 entries, copied to shared memory
// with fully coalesced loads (all of a thread's loads in flight before any
// shared store), then written band by band (ROWS consecutive rows per band).
// rows per CTA of the flat band-major conversion: 0 = auto (256 rows for
// nz <= 8, else 64, measured faster than 128); 64 / 128 force one
int g_ell_flat_rows = 0;
int g_ell_wide_flat = 1;  // tuning: one-pass staging also for 33..128 bands (0 = chunked kernel)

template <int ROWS, int THREADS, int MAXNZ = 32>
__global__ void __launch_bounds__(THREADS) k_crs_to_ell_cm_flat(int64_t n, int32_t nz, int64_t ld,
                                                                const int32_t* __restrict__ irp,
                                                                const int32_t* __restrict__ icol,
                                                                const double* __restrict__ val,
                                                                double* __restrict__ out_val,
                                                                int32_t* __restrict__ out_col,
                                                                int32_t* __restrict__ out_count,
                                                                int64_t pad_base) {
  constexpr int kCap = ROWS * MAXNZ;  // rows hold at most MAXNZ >= nz entries
  // staged entry f lives at f + f/32: rows of exactly 16 or 32 entries read
  // in the write phase (one row per lane) would otherwise all hit one bank
  extern __shared__ unsigned char s_raw[];
  double* s_v = reinterpret_cast<double*>(s_raw);
  int32_t* s_c = reinterpret_cast<int32_t*>(s_v + kCap + kCap / 32);
  __shared__ int32_t s_ptr[ROWS + 1];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * ROWS;
  for (int t = threadIdx.x; t <= ROWS; t += THREADS) s_ptr[t] = __ldg(irp + min(r0 + t, n));
  __syncthreads();
  const int32_t e0 = s_ptr[0], cnt = s_ptr[ROWS] - e0;
  {
    constexpr int kPer = kCap / THREADS;
    double v[kPer];
    int32_t c[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int f = threadIdx.x + k * THREADS;
      if (f < cnt) {
        v[k] = ld_stream(val + e0 + f);
        c[k] = ld_stream(icol + e0 + f);
      }
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int f = threadIdx.x + k * THREADS;
      if (f < cnt) {
        s_v[f + (f >> 5)] = v[k];
        s_c[f + (f >> 5)] = c[k];
      }
    }
  }
  for (int t = threadIdx.x; t < ROWS; t += THREADS)
    if (r0 + t < n) out_count[r0 + t] = s_ptr[t + 1] - s_ptr[t];
  __syncthreads();
  // write phase: a thread stores a row PAIR of one band (16-byte value and
  // 8-byte column stores; r0 and ld are multiples of 32, so pairs never
  // straddle ld)
  constexpr int PAIRS = ROWS / 2;
  const int slots = nz * PAIRS;
  for (int f = threadIdx.x; f < slots; f += THREADS) {
    const int k = f / PAIRS, row = 2 * (f % PAIRS);
    const int64_t i = r0 + row;
    if (i >= ld) continue;
    double v[2];
    int32_t c[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int32_t a = s_ptr[row + h], len = s_ptr[row + h + 1] - a;
      const int fs = a - e0 + k;
      const bool real = k < len;
      v[h] = real ? s_v[fs + (fs >> 5)] : 0.0;
      c[h] = real ? s_c[fs + (fs >> 5)]
                  : static_cast<int32_t>(pad_base + (i + h < n ? i + h : 0));
    }
    const int64_t slot = static_cast<int64_t>(k) * ld + i;
    st_stream2(reinterpret_cast<double2*>(out_val + slot), make_double2(v[0], v[1]));
    *reinterpret_cast<int2*>(out_col + slot) = make_int2(c[0], c[1]);
  }
}

// Row-major ELL: the block's R rows own R*nz consecutive output slots; one
// thread per slot, writes fully coalesced, reads row-contiguous.
__global__ void __launch_bounds__(256) k_crs_to_ell_rm(int64_t n, int32_t nz, FastDiv div_nz,
                                                       int rows_per_block,
                                                       const int32_t* __restrict__ irp,
                                                       const int32_t* __restrict__ icol,
                                                       const double* __restrict__ val,
                                                       double* __restrict__ out_val,
                                                       int32_t* __restrict__ out_col,
                                                       int32_t* __restrict__ out_count,
                                                       int64_t pad_base) {
  extern __shared__ int32_t s_ptr[];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rows_per_block;
  const int rows = static_cast<int>(min(static_cast<int64_t>(rows_per_block), n - r0));
  for (int t = threadIdx.x; t <= rows; t += blockDim.x) s_ptr[t] = __ldg(irp + r0 + t);
  __syncthreads();
  for (int t = threadIdx.x; t < rows; t += blockDim.x)
    out_count[r0 + t] = s_ptr[t + 1] - s_ptr[t];
  const uint32_t slots = static_cast<uint32_t>(rows) * static_cast<uint32_t>(nz);
  const int64_t base = r0 * nz;
  constexpr int U = 4;  // slots per thread with their loads in flight together
  for (uint32_t f0 = threadIdx.x; f0 < slots; f0 += U * blockDim.x) {
    double v[U];
    int32_t c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t f = f0 + u * blockDim.x;
      v[u] = 0.0;
      c[u] = 0;
      if (f < slots) {
        const uint32_t row = div_nz.div(f);
        const int32_t k = static_cast<int32_t>(f - row * static_cast<uint32_t>(nz));
        const int32_t a = s_ptr[row], len = s_ptr[row + 1] - a;
        c[u] = static_cast<int32_t>(pad_base + r0 + row);
        if (k < len) {
          v[u] = ld_stream(val + a + k);
          c[u] = ld_stream(icol + a + k);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t f = f0 + u * blockDim.x;
      if (f < slots) {
        st_stream(out_val + base + f, v[u]);
        out_col[base + f] = c[u];
      }
    }
  }
}

}  // namespace

extern "C" {

int spmvtk_k_expand_ptr(const int32_t* ptr, int64_t n, int64_t nnz, int32_t* out_idx,
                        void* stream) {
  if (n <= 0 || nnz <= 0) SPMVTK_LAUNCH_RETURN();
  int rpw = rows_per_warp_for(n, nnz);
  int64_t warps = (n + rpw - 1) / rpw;
  int64_t blocks = (warps * 32 + 255) / 256;
  k_expand_ptr<<<static_cast<unsigned>(blocks), 256, 0, as_stream(stream)>>>(ptr, n, rpw,
                                                                            out_idx);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_crs_to_coo_row(int64_t n, int64_t nnz, const int32_t* irp, const int32_t* icol,
                            const double* val, int32_t* out_row, int32_t* out_col,
                            double* out_val, void* stream) {
  if (n <= 0 || nnz <= 0) SPMVTK_LAUNCH_RETURN();
  const int rpw = rows_per_warp_for(n, nnz);
  const int64_t warps = (n + rpw - 1) / rpw;
  const int64_t blocks = (warps * 32 + 255) / 256;
  k_crs_to_coo_row<<<static_cast<unsigned>(blocks), 256, 0, as_stream(stream)>>>(
      irp, n, rpw, icol, val, out_row, out_col, out_val);
  SPMVTK_LAUNCH_RETURN();
}

namespace {
struct BucketPlan {
  int shift;
  int nb;
  int fshift;  // coarse bucket = 2^fshift fine buckets; 0 = single pass
  int nc;      // coarse buckets
};
int g_ccs_coarse = 9;  // tuning: log2 of the coarse bucket count target (0 = one pass)
BucketPlan bucket_plan(int64_t n, int64_t nnz, int items) {
  const double per_col = n > 0 ? static_cast<double>(nnz) / static_cast<double>(n) : 1.0;
  int shift = 0;
  // buckets average 2/3 of the sort capacity: skewed column counts (config 5
  // at D = 1) overflow a tighter target into the slow global path
  const double target = (2.0 / 3.0) * items * (items == 8 ? 512 : g_ccs_sort_threads);
  while (shift < 12 && static_cast<double>(int64_t(1) << (shift + 1)) * per_col <= target) ++shift;
  while (((n + (int64_t(1) << shift) - 1) >> shift) > 32768) ++shift;
  const int nb = static_cast<int>((n + (int64_t(1) << shift) - 1) >> shift);
  int fshift = 0;
  if (g_ccs_coarse > 0)
    while ((nb >> fshift) > (1 << g_ccs_coarse)) ++fshift;
  return {shift, nb, fshift, (nb + (1 << fshift) - 1) >> fshift};
}
size_t align256(size_t v) { return (v + 255) & ~static_cast<size_t>(255); }
}  // namespace

int spmvtk_k_tune_convert(const char* key, int value) {
  if (key && std::string(key) == "ccs_slices") {
    g_ccs_slices = value;
    return 0;
  }
  if (key && std::string(key) == "ccs_window") {
    g_ccs_window = value != 0;
    return 0;
  }
  if (key && std::string(key) == "ccs_threads") {
    g_ccs_threads = value;
    return 0;
  }
  if (key && std::string(key) == "ccs_sort_threads") {
    g_ccs_sort_threads = value == 256 ? 256 : 512;
    return 0;
  }
  if (key && std::string(key) == "warp_entries") {
    g_warp_entries = value > 0 ? value : 512;
    return 0;
  }
  if (key && std::string(key) == "ell_flat_rows") {
    g_ell_flat_rows = value == 32 ? 32 : value == 64 ? 64 : value == 128 ? 128 : 0;
    return 0;
  }
  if (key && std::string(key) == "ell_wide_flat") {
    g_ell_wide_flat = value != 0;
    return 0;
  }
  if (key && std::string(key) == "ccs_stage_threads") {
    g_stage_threads = value == 512 ? 512 : 1024;
    return 0;
  }
  if (key && std::string(key) == "ccs_stable") {  // force the stable pipeline (testing)
    spmvtk_dev::g_ccs_force_stable = value;
    return 0;
  }
  if (key && std::string(key) == "ccs_two_pass_runs") {
    const int32_t v = value > 0 ? value : (1 << 17);
    return static_cast<int>(cudaMemcpyToSymbol(d_two_pass_runs, &v, sizeof(v)));
  }
  if (key && std::string(key) == "ccs_sort_items") {
    g_ccs_sort_items = value == 8 || value == 12 ? value : 0;
    return 0;
  }
  if (key && std::string(key) == "ccs_coarse") {
    g_ccs_coarse = value;
    return 0;
  }
  return static_cast<int>(cudaErrorInvalidValue);
}

// Records per sort thread: 8 (512 threads x 3 CTAs per SM, buckets of
// ~2.7 K records) when that bucket plan equals the 12-record one (config 4,
// config 5 at D >= 0.1: only the sort changes, 1-2 % faster), else 12 (512
// threads x 2 CTAs; __launch_bounds__ min 2 keeps it at 64 registers -- the
// compiler otherwise takes 89 and one CTA per SM, 20 % slower).  Smaller
// buckets elsewhere would push banded matrices into the two-pass partition.
// profiles/r02_ccs_sort_items.txt
int sort_items(int64_t n, int64_t nnz) {
  if (g_ccs_sort_items == 8 || g_ccs_sort_items == 12) return g_ccs_sort_items;
  return bucket_plan(n, nnz, 8).shift == bucket_plan(n, nnz, 12).shift ? 8 : 12;
}

size_t legacy_ccs_scratch_bytes_items(int64_t n, int64_t nnz, int items) {
  const BucketPlan bp = bucket_plan(n, nnz, items);
  const size_t t = static_cast<size_t>(bp.nb) * kSlices + 1;
  const size_t tc = static_cast<size_t>(bp.nc) * kSlices + 1;
  const size_t bucketed = 2 * align256(static_cast<size_t>(nnz) * 16) + 256 +
                          align256((kSlices + 1) * 4) + align256(kSlices * 2 * 4) +
                          2 * align256(t * 4) +
                          2 * align256(tc * 4) + 2 * align256((static_cast<size_t>(bp.nb) + 1) * 4) +
                          align256(spmvtk_k_scan_scratch_bytes(static_cast<int64_t>(t))) + 1024;
  return bucketed;
}

size_t legacy_ccs_scratch_bytes(int64_t n, int64_t nnz) {
  return std::max(legacy_ccs_scratch_bytes_items(n, nnz, 8),
                  legacy_ccs_scratch_bytes_items(n, nnz, 12));
}

namespace {
void launch_staged(int ns, cudaStream_t s, const int32_t* irp, const int32_t* icol,
                   const double* val, const int32_t* slice_row, int shift, int nb,
                   const int32_t* Toff, int4* rec, const int32_t* runs, bool as_two) {
  if (g_stage_threads == 512)
    k_bkt_scatter_staged<512><<<ns, 512, 512 * kStageU * sizeof(int4), s>>>(
        irp, icol, val, slice_row, shift, nb, Toff, rec, runs, as_two);
  else
    k_bkt_scatter_staged<1024><<<ns, 1024, 1024 * kStageU * sizeof(int4), s>>>(
        irp, icol, val, slice_row, shift, nb, Toff, rec, runs, as_two);
}
}  // namespace

namespace {
int crs_to_ccs_impl(int64_t n, int64_t nnz, const int32_t* irp, const int32_t* icol,
                    const double* val, int32_t* col_ptr, int32_t* row_idx, double* out_val,
                    int32_t* out_col, void* scratch, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) SPMVTK_LAUNCH_RETURN();
  if (nnz == 0) {
    cudaMemsetAsync(col_ptr, 0, static_cast<size_t>(n + 1) * sizeof(int32_t), s);
    SPMVTK_LAUNCH_RETURN();
  }
  const int items = sort_items(n, nnz);
  const BucketPlan bp = bucket_plan(n, nnz, items);
  const int ns = std::max(1, std::min(g_ccs_slices, kSlices));
  const int nt = g_ccs_threads == 1024 ? 1024 : 512;
  const int64_t tlen = static_cast<int64_t>(bp.nb) * ns;
  uintptr_t cur = (reinterpret_cast<uintptr_t>(scratch) + 255) & ~static_cast<uintptr_t>(255);
  auto take = [&](size_t bytes) {
    void* p = reinterpret_cast<void*>(cur);
    cur += align256(bytes);
    return p;
  };
  int4* rec = static_cast<int4*>(take(static_cast<size_t>(nnz) * 16));
  int32_t* slice_row = static_cast<int32_t*>(take((kSlices + 1) * 4));
  int32_t* win = g_ccs_window && bp.fshift > 0 ? static_cast<int32_t*>(take(kSlices * 2 * 4))
                                                : nullptr;
  int32_t* T = static_cast<int32_t*>(take(static_cast<size_t>(tlen + 1) * 4));
  int32_t* Toff = static_cast<int32_t*>(take(static_cast<size_t>(tlen + 1) * 4));
  int32_t* big = static_cast<int32_t*>(take((static_cast<size_t>(bp.nb) + 1) * 4));
  int32_t* big_len = big + bp.nb;
  void* scan_scratch = take(spmvtk_k_scan_scratch_bytes(tlen + 1));
  const bool two = bp.fshift > 0;
  const int64_t tclen = static_cast<int64_t>(bp.nc) * ns;
  int4* rec2 = two ? static_cast<int4*>(take(static_cast<size_t>(nnz) * 16)) : rec;
  int32_t* Tc = two ? static_cast<int32_t*>(take(static_cast<size_t>(tclen + 1) * 4)) : nullptr;
  int32_t* Tcoff = two ? static_cast<int32_t*>(take(static_cast<size_t>(tclen + 1) * 4)) : nullptr;
  int32_t* fcur = two ? static_cast<int32_t*>(take(static_cast<size_t>(bp.nb) * 4)) : nullptr;
  int32_t* runs = two ? static_cast<int32_t*>(take(4)) : nullptr;

  const size_t hist_smem = static_cast<size_t>(bp.nb) * 4;
  const size_t single_smem = std::max(hist_smem, size_t(1024) * kStageU * sizeof(int4));
  const int cb = 1 << bp.shift;
  const size_t sort_smem = ((static_cast<size_t>(cb + 1) * 4 + 15) & ~static_cast<size_t>(15)) +
                           static_cast<size_t>(items == 8 ? 512 : g_ccs_sort_threads) * items * 14;
  static const bool attrs = [] {  // thread-safe one-time setup
    cudaFuncSetAttribute(k_bkt_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4);
    cudaFuncSetAttribute(k_bkt_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4);
    cudaFuncSetAttribute(k_bkt_scatter_single, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         32768 * 4);
    cudaFuncSetAttribute(k_bkt_scatter_staged<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         1024 * kStageU * static_cast<int>(sizeof(int4)));
    cudaFuncSetAttribute(k_bkt_scatter_staged<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         512 * kStageU * static_cast<int>(sizeof(int4)));
    cudaFuncSetAttribute(k_bkt_sort<512, kBktItems, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(((4097 * 4 + 15) & ~15) + 512 * kBktItems * 14));
    cudaFuncSetAttribute(k_bkt_sort<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(((4097 * 4 + 15) & ~15) + 256 * kBktItems * 14));
    cudaFuncSetAttribute(k_bkt_sort<512, 8, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(((4097 * 4 + 15) & ~15) + 512 * 8 * 14));
    return true;
  }();
  (void)attrs;
  cudaMemsetAsync(big_len, 0, sizeof(int32_t), s);
  if (two) cudaMemsetAsync(runs, 0, sizeof(int32_t), s);
  k_slice_rows<<<(ns + 1 + 3) / 4, 128, 0, s>>>(irp, n, ns, slice_row);
  k_bkt_count<<<ns, nt, hist_smem, s>>>(irp, icol, slice_row, bp.shift, bp.nb, T, bp.fshift,
                                        Tc, runs, win);
  int rc = spmvtk_k_exclusive_scan(T, Toff, tlen, scan_scratch, stream);
  if (rc) return rc;
  if (two) {
    // both alternatives are launched; each returns at once unless the run
    // count (device-side, no host sync) selects it
    rc = spmvtk_k_exclusive_scan(Tc, Tcoff, tclen, scan_scratch, stream);
    if (rc) return rc;
    cudaMemsetAsync(fcur, 0, static_cast<size_t>(bp.nb) * 4, s);
    if (bp.nc <= kStageMaxB)
      launch_staged(ns, s, irp, icol, val, slice_row, bp.shift + bp.fshift, bp.nc, Tcoff, rec,
                    runs, true);
    else
      k_bkt_scatter<<<ns, nt, static_cast<size_t>(bp.nc) * 4, s>>>(
          irp, icol, val, slice_row, bp.shift + bp.fshift, bp.nc, Tcoff, rec, runs, true);
    k_bkt_refine<<<static_cast<unsigned>(std::min<int64_t>(
                       (nnz + kRefineItems - 1) / kRefineItems, int64_t(kSMs) * 2)),
                   kRefineThreads, 0, s>>>(rec, nnz, bp.shift, bp.fshift, Toff, ns, fcur, rec2,
                                           runs);
    // single pass: per slice, staged over its bucket window or cursor
    if (win && nt == 1024)
      k_bkt_scatter_single<<<ns, 1024, single_smem, s>>>(irp, icol, val, slice_row, bp.shift,
                                                         bp.nb, Toff, rec, runs, win);
    else
      k_bkt_scatter<<<ns, nt, hist_smem, s>>>(irp, icol, val, slice_row, bp.shift, bp.nb, Toff,
                                              rec, runs, false);
  } else if (bp.nb <= kStageMaxB && g_ccs_coarse > 0) {
    launch_staged(ns, s, irp, icol, val, slice_row, bp.shift, bp.nb, Toff, rec, nullptr, false);
  } else {
    k_bkt_scatter<<<ns, nt, hist_smem, s>>>(irp, icol, val, slice_row, bp.shift, bp.nb, Toff,
                                            rec, nullptr, false);
  }
  if (items == 8)
    k_bkt_sort<512, 8, 3><<<bp.nb, 512, sort_smem, s>>>(rec, rec2, runs, Toff, n, bp.shift, bp.nb,
                                                        ns, col_ptr, row_idx, out_val, big,
                                                        big_len, out_col);
  else if (g_ccs_sort_threads == 256)
    k_bkt_sort<256><<<bp.nb, 256, sort_smem, s>>>(rec, rec2, runs, Toff, n, bp.shift, bp.nb, ns,
                                                  col_ptr, row_idx, out_val, big, big_len,
                                                  out_col);
  else
    k_bkt_sort<512, kBktItems, 2><<<bp.nb, 512, sort_smem, s>>>(rec, rec2, runs, Toff, n, bp.shift, bp.nb, ns,
                                                  col_ptr, row_idx, out_val, big, big_len,
                                                  out_col);
  k_bkt_sort_big<<<kSMs, 512, 0, s>>>(col_ptr, n, bp.shift, row_idx, out_val, big, big_len);
  SPMVTK_LAUNCH_RETURN();
}
}  // namespace

int legacy_crs_to_ccs(int64_t n, int64_t nnz, const int32_t* irp, const int32_t* icol,
                      const double* val, int32_t* col_ptr, int32_t* row_idx,
                      double* out_val, void* scratch, void* stream) {
  return crs_to_ccs_impl(n, nnz, irp, icol, val, col_ptr, row_idx, out_val, nullptr, scratch,
                         stream);
}

int legacy_crs_to_coo_col(int64_t n, int64_t nnz, const int32_t* irp, const int32_t* icol,
                          const double* val, int32_t* col_ptr, int32_t* row_idx,
                          int32_t* col_idx, double* out_val, void* scratch, void* stream) {
  return crs_to_ccs_impl(n, nnz, irp, icol, val, col_ptr, row_idx, out_val, col_idx, scratch,
                         stream);
}

int spmvtk_k_crs_to_ell_cm(int64_t n, int32_t nz, int64_t ld, const int32_t* irp,
                           const int32_t* icol, const double* val, double* out_val,
                           int32_t* out_col, int32_t* out_count, int64_t pad_base,
                           void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) SPMVTK_LAUNCH_RETURN();
  if (ld < n || (ld & 31) != 0) return static_cast<int>(cudaErrorInvalidValue);
  auto launch = [&](auto kc) {
    constexpr int KC = decltype(kc)::value;
    constexpr int R = 2048 / KC;  // multiple of 32, so blocks also cover [n, ld)
    unsigned blocks = static_cast<unsigned>((ld + R - 1) / R);
    k_crs_to_ell_cm<KC><<<blocks, 256, 0, s>>>(n, nz, ld, irp, icol, val, out_val, out_col,
                                                out_count, pad_base);
  };
  if (nz <= 32) {
    static const bool attrs = [] {
      cudaFuncSetAttribute(k_crs_to_ell_cm_flat<128, 512>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (4096 + 128) * 12);
      return true;
    }();
    (void)attrs;
    if (nz <= 8 && g_ell_flat_rows == 0) {
      // short rows: 256 rows per block (the 32-entry layout would give each
      // block a few hundred entries and the grid many small waves)
      unsigned blocks = static_cast<unsigned>((ld + 255) / 256);
      k_crs_to_ell_cm_flat<256, 256, 8><<<blocks, 256, (2048 + 64) * 12, s>>>(
          n, nz, ld, irp, icol, val, out_val, out_col, out_count, pad_base);
    } else if (g_ell_flat_rows == 32) {
      unsigned blocks = static_cast<unsigned>((ld + 31) / 32);
      k_crs_to_ell_cm_flat<32, 256><<<blocks, 256, (1024 + 32) * 12, s>>>(
          n, nz, ld, irp, icol, val, out_val, out_col, out_count, pad_base);
    } else if (g_ell_flat_rows != 128) {
      unsigned blocks = static_cast<unsigned>((ld + 63) / 64);
      k_crs_to_ell_cm_flat<64, 256><<<blocks, 256, (2048 + 64) * 12, s>>>(
          n, nz, ld, irp, icol, val, out_val, out_col, out_count, pad_base);
    } else {
      unsigned blocks = static_cast<unsigned>((ld + 127) / 128);
      k_crs_to_ell_cm_flat<128, 512><<<blocks, 512, (4096 + 128) * 12, s>>>(
          n, nz, ld, irp, icol, val, out_val, out_col, out_count, pad_base);
    }
  } else if (nz <= 128 && g_ell_wide_flat) {
    // 33..128 bands (config 5 at D <= ~0.3): the same one-pass staging, 32
    // rows per CTA
    static const bool attrs = [] {
      cudaFuncSetAttribute(k_crs_to_ell_cm_flat<32, 256, 128>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (4096 + 128) * 12);

      return true;
    }();
    (void)attrs;
    // (32 rows of <= 64: 2048 staged entries, 40 registers -- measured 12 %
    // faster than 64 or 128 rows, profiles/r02_ell_wide_flat.txt)
    if (nz <= 64)
      k_crs_to_ell_cm_flat<32, 256, 64><<<static_cast<unsigned>((ld + 31) / 32), 256,
                                          (2048 + 64) * 12, s>>>(
          n, nz, ld, irp, icol, val, out_val, out_col, out_count, pad_base);
    else
      k_crs_to_ell_cm_flat<32, 256, 128><<<static_cast<unsigned>((ld + 31) / 32), 256,
                                           (4096 + 128) * 12, s>>>(
          n, nz, ld, irp, icol, val, out_val, out_col, out_count, pad_base);
  } else if (nz <= 4) launch(std::integral_constant<int, 4>{});
  else if (nz <= 8) launch(std::integral_constant<int, 8>{});
  else if (nz <= 16) launch(std::integral_constant<int, 16>{});
  else launch(std::integral_constant<int, 32>{});
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_crs_to_ell_rm(int64_t n, int32_t nz, const int32_t* irp, const int32_t* icol,
                           const double* val, double* out_val, int32_t* out_col,
                           int32_t* out_count, int64_t pad_base, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) SPMVTK_LAUNCH_RETURN();
  // ~4096 slots per block, at least one row, and at least two blocks per SM
  int rows = nz > 0 ? static_cast<int>(4096 / nz) : 4096;
  if (rows > 4096) rows = 4096;
  rows = static_cast<int>(std::min<int64_t>(rows, (n + 2 * kSMs - 1) / (2 * kSMs)));
  if (rows < 1) rows = 1;
  unsigned blocks = static_cast<unsigned>((n + rows - 1) / rows);
  size_t smem = static_cast<size_t>(rows + 1) * sizeof(int32_t);
  k_crs_to_ell_rm<<<blocks, 256, smem, s>>>(n, nz, FastDiv(static_cast<uint32_t>(nz > 0 ? nz : 1)),
                                           rows, irp, icol, val, out_val, out_col, out_count,
                                           pad_base);
  SPMVTK_LAUNCH_RETURN();
}

}  // extern "C"

namespace spmvtk_dev {
void preload_convert() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_expand_ptr);
  cudaFuncGetAttributes(&a, k_crs_to_coo_row);
  cudaFuncGetAttributes(&a, k_slice_rows);
  cudaFuncGetAttributes(&a, k_bkt_count);
  cudaFuncGetAttributes(&a, k_bkt_scatter);
  cudaFuncGetAttributes(&a, k_bkt_scatter_single);
  cudaFuncGetAttributes(&a, k_bkt_scatter_staged<1024>);
  cudaFuncGetAttributes(&a, k_bkt_scatter_staged<512>);
  cudaFuncGetAttributes(&a, k_bkt_refine);
  cudaFuncGetAttributes(&a, k_bkt_sort<256>);
  cudaFuncGetAttributes(&a, k_bkt_sort<512, kBktItems, 2>);
  cudaFuncGetAttributes(&a, k_bkt_sort<512, 8, 3>);
  cudaFuncGetAttributes(&a, k_bkt_sort_big);
  cudaFuncGetAttributes(&a, k_crs_to_ell_cm<32>);
  cudaFuncGetAttributes(&a, k_crs_to_ell_cm_flat<64, 256>);
  cudaFuncGetAttributes(&a, k_crs_to_ell_cm_flat<256, 256, 8>);
  cudaFuncGetAttributes(&a, k_crs_to_ell_cm_flat<128, 512>);
  cudaFuncGetAttributes(&a, k_crs_to_ell_cm_flat<32, 256, 64>);
  cudaFuncGetAttributes(&a, k_crs_to_ell_cm_flat<32, 256, 128>);
  cudaFuncGetAttributes(&a, k_crs_to_ell_rm);
}
}  // namespace spmvtk_dev
