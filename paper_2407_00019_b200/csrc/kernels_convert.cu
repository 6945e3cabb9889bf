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
#include <type_traits>

#include "common.cuh"
#include "spmvtk/spmvtk_kernels.h"

using namespace spmvtk_dev;

namespace {

// A window of 32 consecutive segments [r0, r0+32) of a pointer array; lane l
// holds the end of segment r0+l (ptr[r0+l+1]) or INT_MAX past the last
// segment of the chunk.  offset(p) = number of segments of the window that
// end at or before p, i.e. the segment of entry p relative to r0, valid when
// ptr[r0] <= p < end.
struct SegWindow {
  int64_t r0;
  int32_t s;
  int32_t end;

  __device__ __forceinline__ void load(const int32_t* ptr, int64_t r_end, int lane) {
    int64_t r = r0 + lane + 1;
    s = (r <= r_end) ? __ldg(ptr + r) : INT_MAX;
    end = __shfl_sync(kFull, s, 31);
  }
  __device__ __forceinline__ int offset(int32_t p) const {
    int lo = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
      int32_t v = __shfl_sync(kFull, s, lo + step - 1);
      if (v <= p) lo += step;
    }
    return lo;
  }
};

// Segment id of entry p for every lane with `need` set; warp-uniform advance
// of the window over segments (empty ones included) until all lanes resolve.
__device__ __forceinline__ int32_t resolve_segment(SegWindow& w, const int32_t* ptr,
                                                   int64_t r_end, int lane, int32_t p,
                                                   bool need) {
  int32_t seg = 0;
  for (;;) {
    bool in = need && p < w.end;
    int off = w.offset(p);
    if (in) {
      seg = static_cast<int32_t>(w.r0 + off);
      need = false;
    }
    if (!__any_sync(kFull, need)) break;
    w.r0 += 32;
    w.load(ptr, r_end, lane);
  }
  return seg;
}

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

int rows_per_warp_for(int64_t n, int64_t nnz) {
  // aim at ~1024 entries per warp chunk
  double mean = n > 0 ? static_cast<double>(nnz) / static_cast<double>(n) : 1.0;
  int64_t r = 32;
  while (r < 8192 && static_cast<double>(r) * mean < 1024.0) r <<= 1;
  return static_cast<int>(r);
}

// ---- CRS -> CCS ------------------------------------------------------------
__global__ void __launch_bounds__(256) k_col_hist(const int32_t* __restrict__ icol,
                                                  int64_t nnz, int32_t* count) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < nnz;
       p += stride)
    atomicAdd(count + ld_stream(icol + p), 1);
}

// pass 3 (convert.cpp:43-51): each entry takes the next free slot of its
// column.  Slot order inside a column is arbitrary here; k_ccs_fix_* restore
// ascending rows afterwards (rows are distinct within a column, so sorting on
// the row reproduces the reference order exactly).
__global__ void __launch_bounds__(256) k_ccs_scatter(const int32_t* __restrict__ irp,
                                                     const int32_t* __restrict__ icol,
                                                     const double* __restrict__ val,
                                                     int64_t n, int rows_per_warp,
                                                     int32_t* cursor,
                                                     int4* __restrict__ rec) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t rb = warp * rows_per_warp;
  if (rb >= n) return;
  const int64_t re = min(rb + rows_per_warp, n);
  const int32_t e0 = __ldg(irp + rb), e1 = __ldg(irp + re);
  SegWindow w;
  w.r0 = rb;
  w.load(irp, re, lane);
  for (int32_t base = e0; base < e1; base += 32) {
    int32_t p = base + lane;
    bool valid = p < e1;
    int32_t c = 0;
    double v = 0.0;
    if (valid) {
      c = ld_stream(icol + p);
      v = ld_stream(val + p);
    }
    int32_t row = resolve_segment(w, irp, re, lane, p, valid);
    if (valid) {
      // one 16-byte (row, value) record per entry: a single half-sector
      // store instead of a 4-byte and an 8-byte store into two arrays (the
      // random partial-sector writes dominated this kernel's DRAM traffic)
      const int32_t slot = atomicAdd(cursor + c, 1);
      rec[slot] = make_int4(row, 0, __double2loint(v), __double2hiint(v));
    }
  }
}

__device__ __forceinline__ double rec_val(const int4& r) { return __hiloint2double(r.w, r.z); }

// Columns of length <= 32: one warp per column, bitonic sort in registers on
// a packed key (row << 5 | source lane); values follow by shuffle.  Sorted
// columns (the common case) exit after one ballot.  Longer columns are queued
// for the block-level passes.
constexpr int kShortCol = 32;
constexpr int kMediumCol = 4096;

__global__ void __launch_bounds__(256) k_ccs_fix_short(const int32_t* __restrict__ col_ptr,
                                                       int64_t n, const int4* __restrict__ rec,
                                                       int32_t* __restrict__ row_idx,
                                                       double* __restrict__ vals, int32_t* queue,
                                                       int32_t* queue_len, bool packed_ok) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < n;
       j += warps) {
    const int32_t a = __ldg(col_ptr + j), b = __ldg(col_ptr + j + 1);
    const int32_t len = b - a;
    if (len <= 0) continue;
    if (len > kShortCol || !packed_ok) {
      if (lane == 0) queue[atomicAdd(queue_len, 1)] = static_cast<int32_t>(j);
      continue;
    }
    int4 rc = make_int4(INT_MAX, 0, 0, 0);
    if (lane < len) rc = ld_stream4(rec + a + lane);
    const int32_t r = rc.x;
    const double v = rec_val(rc);
    const int32_t rn = __shfl_down_sync(kFull, r, 1);
    const bool desc = (lane + 1 < len) && rn < r;
    if (!__any_sync(kFull, desc)) {
      if (lane < len) {
        row_idx[a + lane] = r;
        vals[a + lane] = v;
      }
      continue;
    }
    // rows < 2^26 so (row << 5 | lane) fits; padding lanes sort last
    uint32_t key = lane < len ? (static_cast<uint32_t>(r) << 5) | lane : 0xffffffffu;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int d = size >> 1; d > 0; d >>= 1) {
        uint32_t other = __shfl_xor_sync(kFull, key, d);
        bool up = ((lane & size) == 0);
        bool lower = (lane & d) == 0;
        uint32_t mn = min(key, other), mx = max(key, other);
        key = (lower == up) ? mn : mx;
      }
    }
    int src = static_cast<int>(key & 31u);
    double sv = __shfl_sync(kFull, v, src);
    if (lane < len) {
      row_idx[a + lane] = static_cast<int32_t>(key >> 5);
      vals[a + lane] = sv;
    }
  }
}

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

__global__ void __launch_bounds__(512) k_ccs_fix_long(const int32_t* __restrict__ col_ptr,
                                                      const int4* __restrict__ rec,
                                                      int32_t* row_idx, double* vals,
                                                      const int32_t* queue,
                                                      const int32_t* queue_len) {
  __shared__ int32_t s_key[kMediumCol];
  __shared__ double s_val[kMediumCol];
  const int32_t count = *queue_len;
  for (int32_t q = blockIdx.x; q < count; q += gridDim.x) {
    const int32_t j = queue[q];
    const int32_t a = col_ptr[j], len = col_ptr[j + 1] - a;
    if (len <= kMediumCol) {
      for (int32_t t = threadIdx.x; t < len; t += blockDim.x) {
        const int4 rc = rec[a + t];
        s_key[t] = rc.x;
        s_val[t] = rec_val(rc);
      }
      __syncthreads();
      block_bitonic(s_key, s_val, len);
      for (int32_t t = threadIdx.x; t < len; t += blockDim.x) {
        row_idx[a + t] = s_key[t];
        vals[a + t] = s_val[t];
      }
    } else {
      // very long column: unpack, then the same network in global memory (L2)
      for (int32_t t = threadIdx.x; t < len; t += blockDim.x) {
        const int4 rc = rec[a + t];
        row_idx[a + t] = rc.x;
        vals[a + t] = rec_val(rc);
      }
      __syncthreads();
      block_bitonic(row_idx + a, vals + a, len);
    }
    __syncthreads();
  }
}

// ---- CRS -> CCS, bucketed (no global atomics) -------------------------------
// Columns are grouped into NB buckets of CB = 2^shift consecutive columns
// (~4k entries per bucket).  The CRS is split into kSlices row ranges of
// equal entry counts (one per SM).
//   1. k_bkt_count   slice-local bucket histograms in shared memory ->
//                    T[b * kSlices + slice]
//   2. exclusive scan of T (bucket-major) -> each (bucket, slice) owns a run
//   3. k_bkt_scatter each slice re-reads its rows and appends 16-byte
//                    records (col, row, value) to its runs with shared-memory
//                    cursors: writes are kSlices x NB sequential streams that
//                    fill whole sectors in L2
//   4. k_bkt_sort    one CTA per bucket: counting sort by column in shared
//                    memory, per-column sort by row (rows are distinct within
//                    a column, so this restores the reference's order,
//                    convert.cpp:43-51), col_ptr and the final row_idx /
//                    values written fully coalesced.
// Buckets too large for shared memory take a global-memory path.
constexpr int kSlices = 3 * 148;  // 3 CTAs per SM (64 KB histograms)
constexpr int kBktThreads = 512;
constexpr int kBktItems = 12;
constexpr int kBktCap = kBktThreads * kBktItems;  // records per bucket sorted in smem

__global__ void k_slice_rows(const int32_t* __restrict__ irp, int64_t n, int32_t* slice_row) {
  // slice s starts at the first row whose start >= s * nnz / kSlices
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s > kSlices) return;
  const int64_t nnz = irp[n];
  const int64_t target = nnz * s / kSlices;
  int64_t lo = 0, hi = n;  // smallest r with irp[r] >= target
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (irp[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  slice_row[s] = static_cast<int32_t>(s == kSlices ? n : lo);
}

__global__ void __launch_bounds__(kBktThreads) k_bkt_count(const int32_t* __restrict__ irp,
                                                           const int32_t* __restrict__ icol,
                                                           const int32_t* __restrict__ slice_row,
                                                           int shift, int nb, int32_t* T) {
  extern __shared__ int32_t s_hist[];
  for (int b = threadIdx.x; b < nb; b += blockDim.x) s_hist[b] = 0;
  __syncthreads();
  const int32_t e0 = irp[slice_row[blockIdx.x]], e1 = irp[slice_row[blockIdx.x + 1]];
  const int32_t step = static_cast<int32_t>(blockDim.x);
  int32_t p = e0 + static_cast<int32_t>(threadIdx.x);
  for (; p + 3 * step < e1; p += 4 * step) {  // 4 loads in flight per thread
    const int32_t c0 = ld_stream(icol + p), c1 = ld_stream(icol + p + step);
    const int32_t c2 = ld_stream(icol + p + 2 * step), c3 = ld_stream(icol + p + 3 * step);
    atomicAdd(&s_hist[c0 >> shift], 1);
    atomicAdd(&s_hist[c1 >> shift], 1);
    atomicAdd(&s_hist[c2 >> shift], 1);
    atomicAdd(&s_hist[c3 >> shift], 1);
  }
  for (; p < e1; p += step) atomicAdd(&s_hist[ld_stream(icol + p) >> shift], 1);
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    T[static_cast<int64_t>(b) * kSlices + blockIdx.x] = s_hist[b];
}

__global__ void __launch_bounds__(kBktThreads) k_bkt_scatter(
    const int32_t* __restrict__ irp, const int32_t* __restrict__ icol,
    const double* __restrict__ val, const int32_t* __restrict__ slice_row, int shift, int nb,
    const int32_t* __restrict__ Toff, int4* __restrict__ rec) {
  extern __shared__ int32_t s_cur[];
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    s_cur[b] = Toff[static_cast<int64_t>(b) * kSlices + blockIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int64_t r_begin = slice_row[blockIdx.x], r_end = slice_row[blockIdx.x + 1];
  constexpr int kRows = 64;  // rows per warp chunk
  for (int64_t rb = r_begin + static_cast<int64_t>(warp) * kRows; rb < r_end;
       rb += static_cast<int64_t>(nwarps) * kRows) {
    const int64_t re = min(rb + kRows, r_end);
    const int32_t e0 = __ldg(irp + rb), e1 = __ldg(irp + re);
    SegWindow w;
    w.r0 = rb;
    w.load(irp, re, lane);
    for (int32_t base = e0; base < e1; base += 32) {
      const int32_t p = base + lane;
      const bool valid = p < e1;
      int32_t c = 0;
      double v = 0.0;
      if (valid) {
        c = ld_stream(icol + p);
        v = ld_stream(val + p);
      }
      const int32_t row = resolve_segment(w, irp, re, lane, p, valid);
      if (valid) {
        const int32_t slot = atomicAdd(&s_cur[c >> shift], 1);
        rec[slot] = make_int4(c, row, __double2loint(v), __double2hiint(v));
      }
    }
  }
}

// one CTA per bucket; dynamic smem: cnt[cb+1] | s_row[kBktCap] | s_val[kBktCap]
__global__ void __launch_bounds__(kBktThreads) k_bkt_sort(
    const int4* __restrict__ rec, const int32_t* __restrict__ Toff, int64_t n, int shift,
    int nb, int32_t* __restrict__ col_ptr, int32_t* __restrict__ row_idx,
    double* __restrict__ out_val, int32_t* big_queue, int32_t* big_len) {
  extern __shared__ unsigned char s_raw[];
  const int cb = 1 << shift;
  int32_t* cnt = reinterpret_cast<int32_t*>(s_raw);  // cb + 1 entries
  double* s_val = reinterpret_cast<double*>(s_raw + ((static_cast<size_t>(cb + 1) * 4 + 15) & ~15));
  int32_t* s_row = reinterpret_cast<int32_t*>(s_val + kBktCap);
  const int b = blockIdx.x;
  const int32_t bs = Toff[static_cast<int64_t>(b) * kSlices];
  const int32_t be = (b + 1 < nb) ? Toff[static_cast<int64_t>(b + 1) * kSlices]
                                  : Toff[static_cast<int64_t>(nb) * kSlices];
  const int64_t c0 = static_cast<int64_t>(b) << shift;
  const int ncols = static_cast<int>(min(static_cast<int64_t>(cb), n - c0));
  const int32_t len = be - bs;
  const bool fits = len <= kBktCap;
  for (int i = threadIdx.x; i <= cb; i += blockDim.x) cnt[i] = 0;
  // records stay in registers between the count and the placement
  int4 r[kBktItems];
  if (fits) {
#pragma unroll
    for (int k = 0; k < kBktItems; ++k) {
      const int32_t q = static_cast<int32_t>(threadIdx.x) + k * kBktThreads;
      if (q < len) r[k] = ld_stream4(rec + bs + q);
    }
  }
  __syncthreads();
  if (fits) {
#pragma unroll
    for (int k = 0; k < kBktItems; ++k) {
      const int32_t q = static_cast<int32_t>(threadIdx.x) + k * kBktThreads;
      if (q < len) atomicAdd(&cnt[r[k].x - c0], 1);
    }
  } else {
    for (int32_t q = threadIdx.x; q < len; q += blockDim.x)
      atomicAdd(&cnt[__ldg(&rec[bs + q].x) - c0], 1);
  }
  __syncthreads();
  // exclusive scan of cnt[0..cb) by warp 0 (cb <= 4096, a few passes)
  if (threadIdx.x < 32) {
    int32_t carry = 0;
    for (int base = 0; base < cb; base += 32) {
      const int i = base + threadIdx.x;
      const int32_t v = cnt[i];
      int32_t inc = v;
      for (int d = 1; d < 32; d <<= 1) {
        const int32_t t = __shfl_up_sync(kFull, inc, d);
        if (threadIdx.x >= d) inc += t;
      }
      cnt[i] = carry + inc - v;
      carry += __shfl_sync(kFull, inc, 31);
    }
    if (threadIdx.x == 0) cnt[cb] = carry;
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
    }
    if (threadIdx.x == 0) big_queue[atomicAdd(big_len, 1)] = b;
    return;
  }
  // place by column (shared cursors; order inside a column arbitrary)
#pragma unroll
  for (int k = 0; k < kBktItems; ++k) {
    const int32_t q = static_cast<int32_t>(threadIdx.x) + k * kBktThreads;
    if (q < len) {
      const int32_t slot = atomicAdd(&cnt[r[k].x - c0], 1);
      s_row[slot] = r[k].y;
      s_val[slot] = rec_val(r[k]);
    }
  }
  __syncthreads();
  // cnt[i] now holds the END of column i; column i spans [end(i-1), end(i)).
  // One warp per column: register bitonic sort on (row << 5 | lane) for
  // columns of <= 32 entries (already-sorted columns skip the network), a
  // lane-0 insertion sort beyond; results go straight to the output arrays.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = warp; i < ncols; i += blockDim.x >> 5) {
    const int32_t a = i ? cnt[i - 1] : 0, e = cnt[i], cl = e - a;
    if (cl <= 32 && n < (int64_t(1) << 27)) {  // (row << 5 | lane) must fit 32 bits
      int32_t rr = lane < cl ? s_row[a + lane] : INT_MAX;
      double v = lane < cl ? s_val[a + lane] : 0.0;
      const int32_t rn = __shfl_down_sync(kFull, rr, 1);
      if (__any_sync(kFull, lane + 1 < cl && rn < rr)) {
        uint32_t key = lane < cl ? (static_cast<uint32_t>(rr) << 5) | lane : 0xffffffffu;
#pragma unroll
        for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
          for (int d = size >> 1; d > 0; d >>= 1) {
            const uint32_t other = __shfl_xor_sync(kFull, key, d);
            const bool up = (lane & size) == 0, lower = (lane & d) == 0;
            key = (lower == up) ? min(key, other) : max(key, other);
          }
        }
        v = __shfl_sync(kFull, v, static_cast<int>(key & 31u));
        rr = static_cast<int32_t>(key >> 5);
      }
      if (lane < cl) {
        row_idx[bs + a + lane] = rr;
        st_stream(out_val + bs + a + lane, v);
      }
    } else {
      if (lane == 0)
        for (int32_t k = a + 1; k < e; ++k) {  // insertion sort on row
          const int32_t key = s_row[k];
          const double v = s_val[k];
          int32_t j = k - 1;
          while (j >= a && s_row[j] > key) {
            s_row[j + 1] = s_row[j];
            s_val[j + 1] = s_val[j];
            --j;
          }
          s_row[j + 1] = key;
          s_val[j + 1] = v;
        }
      __syncwarp();
      for (int32_t q = a + lane; q < e; q += 32) {
        row_idx[bs + q] = s_row[q];
        st_stream(out_val + bs + q, s_val[q]);
      }
    }
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
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * R;
  for (int t = threadIdx.x; t <= R; t += blockDim.x)
    s_ptr[t] = __ldg(irp + min(r0 + t, n));
  __syncthreads();
  for (int t = threadIdx.x; t < R; t += blockDim.x)
    if (r0 + t < n) out_count[r0 + t] = s_ptr[t + 1] - s_ptr[t];
  for (int32_t k0 = 0; k0 < nz; k0 += KC) {
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

// Band-major, short bands (nz <= 32): the block's 64 rows are one
// contiguous CRS range of at most 2048 entries, copied to shared memory with
// fully coalesced loads, then written band by band.
constexpr int kFlatRows = 64;
constexpr int kFlatCap = kFlatRows * 32;

__global__ void __launch_bounds__(256) k_crs_to_ell_cm_flat(int64_t n, int32_t nz, int64_t ld,
                                                            const int32_t* __restrict__ irp,
                                                            const int32_t* __restrict__ icol,
                                                            const double* __restrict__ val,
                                                            double* __restrict__ out_val,
                                                            int32_t* __restrict__ out_col,
                                                            int32_t* __restrict__ out_count,
                                                            int64_t pad_base) {
  __shared__ int32_t s_ptr[kFlatRows + 1];
  __shared__ double s_v[kFlatCap];
  __shared__ int32_t s_c[kFlatCap];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kFlatRows;
  for (int t = threadIdx.x; t <= kFlatRows; t += blockDim.x)
    s_ptr[t] = __ldg(irp + min(r0 + t, n));
  __syncthreads();
  const int32_t e0 = s_ptr[0], cnt = s_ptr[kFlatRows] - e0;
  for (int f = threadIdx.x; f < cnt; f += blockDim.x) {
    s_v[f] = ld_stream(val + e0 + f);
    s_c[f] = ld_stream(icol + e0 + f);
  }
  for (int t = threadIdx.x; t < kFlatRows; t += blockDim.x)
    if (r0 + t < n) out_count[r0 + t] = s_ptr[t + 1] - s_ptr[t];
  __syncthreads();
  const int slots = nz * kFlatRows;
  for (int f = threadIdx.x; f < slots; f += blockDim.x) {
    const int k = f / kFlatRows, row = f % kFlatRows;
    const int64_t i = r0 + row;
    if (i >= ld) continue;
    const int32_t a = s_ptr[row], len = s_ptr[row + 1] - a;
    const bool real = k < len;
    const int64_t slot = static_cast<int64_t>(k) * ld + i;
    st_stream(out_val + slot, real ? s_v[a - e0 + k] : 0.0);
    out_col[slot] = real ? s_c[a - e0 + k] : static_cast<int32_t>(pad_base + (i < n ? i : 0));
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
  for (uint32_t f = threadIdx.x; f < slots; f += blockDim.x) {
    const uint32_t row = div_nz.div(f);
    const int32_t k = static_cast<int32_t>(f - row * static_cast<uint32_t>(nz));
    const int32_t a = s_ptr[row], len = s_ptr[row + 1] - a;
    double v = 0.0;
    int32_t c = static_cast<int32_t>(pad_base + r0 + row);
    if (k < len) {
      v = ld_stream(val + a + k);
      c = ld_stream(icol + a + k);
    }
    st_stream(out_val + base + f, v);
    out_col[base + f] = c;
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

namespace {
struct BucketPlan {
  int shift;
  int nb;
};
BucketPlan bucket_plan(int64_t n, int64_t nnz) {
  const double per_col = n > 0 ? static_cast<double>(nnz) / static_cast<double>(n) : 1.0;
  int shift = 0;
  while (shift < 12 && static_cast<double>(int64_t(1) << (shift + 1)) * per_col <= 4096.0) ++shift;
  while (((n + (int64_t(1) << shift) - 1) >> shift) > 32768) ++shift;
  return {shift, static_cast<int>((n + (int64_t(1) << shift) - 1) >> shift)};
}
size_t align256(size_t v) { return (v + 255) & ~static_cast<size_t>(255); }
}  // namespace

size_t spmvtk_k_ccs_scratch_bytes(int64_t n, int64_t nnz) {
  const BucketPlan bp = bucket_plan(n, nnz);
  const size_t t = static_cast<size_t>(bp.nb) * kSlices + 1;
  const size_t bucketed = align256(static_cast<size_t>(nnz) * 16) + align256((kSlices + 1) * 4) +
                          2 * align256(t * 4) + align256((static_cast<size_t>(bp.nb) + 1) * 4) +
                          align256(spmvtk_k_scan_scratch_bytes(static_cast<int64_t>(t))) + 1024;
  // the atomic-cursor variant needs count/cursor/queue over n columns
  const size_t atomic = static_cast<size_t>(nnz) * 16 +
                        (static_cast<size_t>(n + 1) * 3 + 4) * sizeof(int32_t) +
                        spmvtk_k_scan_scratch_bytes(n + 1) + 1024;
  return bucketed > atomic ? bucketed : atomic;
}

int spmvtk_k_crs_to_ccs(int64_t n, int64_t nnz, const int32_t* irp, const int32_t* icol,
                        const double* val, int32_t* col_ptr, int32_t* row_idx,
                        double* out_val, void* scratch, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) SPMVTK_LAUNCH_RETURN();
  if (nnz == 0) {
    cudaMemsetAsync(col_ptr, 0, static_cast<size_t>(n + 1) * sizeof(int32_t), s);
    SPMVTK_LAUNCH_RETURN();
  }
  const BucketPlan bp = bucket_plan(n, nnz);
  const int64_t tlen = static_cast<int64_t>(bp.nb) * kSlices;
  uintptr_t cur = (reinterpret_cast<uintptr_t>(scratch) + 255) & ~static_cast<uintptr_t>(255);
  auto take = [&](size_t bytes) {
    void* p = reinterpret_cast<void*>(cur);
    cur += align256(bytes);
    return p;
  };
  int4* rec = static_cast<int4*>(take(static_cast<size_t>(nnz) * 16));
  int32_t* slice_row = static_cast<int32_t*>(take((kSlices + 1) * 4));
  int32_t* T = static_cast<int32_t*>(take(static_cast<size_t>(tlen + 1) * 4));
  int32_t* Toff = static_cast<int32_t*>(take(static_cast<size_t>(tlen + 1) * 4));
  int32_t* big = static_cast<int32_t*>(take((static_cast<size_t>(bp.nb) + 1) * 4));
  int32_t* big_len = big + bp.nb;
  void* scan_scratch = take(spmvtk_k_scan_scratch_bytes(tlen + 1));

  const size_t hist_smem = static_cast<size_t>(bp.nb) * 4;
  const int cb = 1 << bp.shift;
  const size_t sort_smem = ((static_cast<size_t>(cb + 1) * 4 + 15) & ~static_cast<size_t>(15)) +
                           static_cast<size_t>(kBktCap) * 12;
  static const bool attrs = [] {  // thread-safe one-time setup
    cudaFuncSetAttribute(k_bkt_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4);
    cudaFuncSetAttribute(k_bkt_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4);
    cudaFuncSetAttribute(k_bkt_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(((4097 * 4 + 15) & ~15) + kBktCap * 12));
    return true;
  }();
  (void)attrs;
  cudaMemsetAsync(big_len, 0, sizeof(int32_t), s);
  k_slice_rows<<<(kSlices + 128) / 128, 128, 0, s>>>(irp, n, slice_row);
  k_bkt_count<<<kSlices, kBktThreads, hist_smem, s>>>(irp, icol, slice_row, bp.shift, bp.nb, T);
  int rc = spmvtk_k_exclusive_scan(T, Toff, tlen, scan_scratch, stream);
  if (rc) return rc;
  k_bkt_scatter<<<kSlices, kBktThreads, hist_smem, s>>>(irp, icol, val, slice_row, bp.shift,
                                                         bp.nb, Toff, rec);
  k_bkt_sort<<<bp.nb, kBktThreads, sort_smem, s>>>(rec, Toff, n, bp.shift, bp.nb, col_ptr,
                                                    row_idx, out_val, big, big_len);
  k_bkt_sort_big<<<kSMs, 512, 0, s>>>(col_ptr, n, bp.shift, row_idx, out_val, big, big_len);
  SPMVTK_LAUNCH_RETURN();
}

// the previous, atomic-cursor formulation (kept for comparison / tuning)
int spmvtk_k_crs_to_ccs_atomic(int64_t n, int64_t nnz, const int32_t* irp, const int32_t* icol,
                               const double* val, int32_t* col_ptr, int32_t* row_idx,
                               double* out_val, void* scratch, void* stream) {
  cudaStream_t s = as_stream(stream);
  uintptr_t base = (reinterpret_cast<uintptr_t>(scratch) + 255) & ~static_cast<uintptr_t>(255);
  int4* rec = reinterpret_cast<int4*>(base);
  int32_t* count = reinterpret_cast<int32_t*>(rec + nnz);
  int32_t* cursor = count + (n + 1);
  int32_t* queue = cursor + (n + 1);
  int32_t* queue_len = queue + n;
  // keep the scan scratch aligned
  uintptr_t sp = reinterpret_cast<uintptr_t>(queue_len + 4);
  sp = (sp + 255) & ~static_cast<uintptr_t>(255);
  void* scan_scratch = reinterpret_cast<void*>(sp);

  cudaMemsetAsync(count, 0, static_cast<size_t>(n + 1) * sizeof(int32_t), s);
  cudaMemsetAsync(queue_len, 0, sizeof(int32_t), s);
  if (nnz > 0) k_col_hist<<<grid_for(nnz, 256), 256, 0, s>>>(icol, nnz, count);
  int rc = spmvtk_k_exclusive_scan(count, col_ptr, n, scan_scratch, stream);
  if (rc) return rc;
  if (nnz == 0 || n == 0) SPMVTK_LAUNCH_RETURN();
  cudaMemcpyAsync(cursor, col_ptr, static_cast<size_t>(n) * sizeof(int32_t),
                  cudaMemcpyDeviceToDevice, s);
  int rpw = rows_per_warp_for(n, nnz);
  int64_t warps = (n + rpw - 1) / rpw;
  int64_t blocks = (warps * 32 + 255) / 256;
  k_ccs_scatter<<<static_cast<unsigned>(blocks), 256, 0, s>>>(irp, icol, val, n, rpw, cursor,
                                                             rec);
  k_ccs_fix_short<<<grid_for(n * 32, 256, 16), 256, 0, s>>>(col_ptr, n, rec, row_idx, out_val,
                                                            queue, queue_len,
                                                            n < (int64_t(1) << 26));
  k_ccs_fix_long<<<kSMs * 2, 512, 0, s>>>(col_ptr, rec, row_idx, out_val, queue, queue_len);
  SPMVTK_LAUNCH_RETURN();
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
    unsigned blocks = static_cast<unsigned>((ld + kFlatRows - 1) / kFlatRows);
    k_crs_to_ell_cm_flat<<<blocks, 256, 0, s>>>(n, nz, ld, irp, icol, val, out_val, out_col,
                                                out_count, pad_base);
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
  // ~4096 slots per block, at least one row
  int rows = nz > 0 ? static_cast<int>(4096 / nz) : 4096;
  if (rows < 1) rows = 1;
  if (rows > 4096) rows = 4096;
  unsigned blocks = static_cast<unsigned>((n + rows - 1) / rows);
  size_t smem = static_cast<size_t>(rows + 1) * sizeof(int32_t);
  k_crs_to_ell_rm<<<blocks, 256, smem, s>>>(n, nz, FastDiv(static_cast<uint32_t>(nz > 0 ? nz : 1)),
                                           rows, irp, icol, val, out_val, out_col, out_count,
                                           pad_base);
  SPMVTK_LAUNCH_RETURN();
}

}  // extern "C"
