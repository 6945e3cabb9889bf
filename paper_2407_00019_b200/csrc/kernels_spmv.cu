// kernels_spmv.cu -- SpMV in CRS, COO (row- and column-ordered) and ELL
// (band-major "inner"/"outer", row-major) on sm_100a.
//
// Every kernel here is HBM-bound (~0.17 flop/byte): no tensor cores, the
// design levers are coalescing, 128-bit loads, enough bytes in flight per SM
// (unrolled independent loads) and keeping x cacheable while the matrix
// streams through with L1::no_allocate.  Reference kernels are in
// /root/reference/proj/src/spmv.cpp; each kernel below names the one it
// replaces.  Summation orders differ from the reference (fp64, FMA), which the
// contract allows (max-norm relative 1e-12, BASELINE.json north_star).
#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "spmvtk/spmvtk.h"
#include "spmvtk/spmvtk_kernels.h"

using namespace spmvtk_dev;

namespace {

__device__ __forceinline__ unsigned subwarp_mask(int W) {
  if (W == 32) return kFull;
  const int lane = threadIdx.x & 31;
  return ((1u << W) - 1u) << (lane & ~(W - 1));
}

// ---- where a result row goes -------------------------------------------
// PlainOut: y[r].  PushOut: the row-block multi-GPU exchange folded into the
// epilogue -- row r is stored to every rank that reads it (dst[w] points at
// this shard's rows inside rank w's next-x buffer, peer memory over NVLink),
// and each thread fences at system scope before it exits so a later flag
// store (spmvtk_k_flags_signal) orders after all of its pushes.
struct PlainOut {
  double* __restrict__ y;
  __device__ __forceinline__ void begin() const {}
  __device__ __forceinline__ void put(int64_t r, double v) const { y[r] = v; }
  __device__ __forceinline__ void done() const {}
};

__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct PushOut {
  spmvtk_push p;
  spmvtk_push_sync s;  // nwait = 0 / counter = NULL switch the pieces off
  // every thread of every CTA, before x is read: the step's flag wait
  __device__ __forceinline__ void begin() const {
    if (s.nwait <= 0) return;
    if (threadIdx.x == 0 && *reinterpret_cast<volatile uint32_t*>(s.status) == 0) {
      const uint64_t t0 = globaltimer_ns();
      for (int w = 0; w < s.nwait; ++w)
        while (ld_acquire_sys_u64(s.wait_flags + w) < s.wait_value) {
          if (globaltimer_ns() - t0 > s.timeout_ns) {
            atomicOr(s.status, 1u);
            break;
          }
          __nanosleep(32);
        }
    }
    __syncthreads();
  }
  __device__ __forceinline__ void put(int64_t r, double v) const {
    const unsigned m = p.mask ? __ldg(p.mask + r) : 0xffu;
#pragma unroll
    for (int w = 0; w < SPMVTK_MAX_PEERS; ++w)
      if (w < p.ndst && ((m >> w) & 1u)) p.dst[w][r] = v;
  }
  // every thread of every CTA, at the end: fence the pushes at system scope;
  // the last CTA to arrive stores the step flag to every rank
  __device__ __forceinline__ void done() const {
    if (p.ndst > 1) __threadfence_system();
    if (s.counter == nullptr) return;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned prev = atomicAdd(s.counter, 1u);
      if (prev == gridDim.x - 1) {
        *s.counter = 0;
        __threadfence_system();
        for (int w = 0; w < s.signal.n; ++w)
          asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(s.signal.ptr[w]),
                       "l"(s.signal_value)
                       : "memory");
      }
    }
  }
};

// ---- vector CRS: W lanes per row (spmv_crs, spmv.cpp:64-75) --------------
// Row extents come from a policy so the same kernel serves CRS (irp) and
// row-major ELL (fixed stride nz).  Rows longer than long_limit are handed to
// a block-per-row pass through a device queue (power-law rows would
// otherwise serialise one sub-warp).
struct CrsRows {
  const int32_t* irp;
  __device__ __forceinline__ void get(int64_t r, int64_t& a, int64_t& b) const {
    a = __ldg(irp + r);
    b = __ldg(irp + r + 1);
  }
};
struct EllRowMajorRows {
  int32_t nz;
  __device__ __forceinline__ void get(int64_t r, int64_t& a, int64_t& b) const {
    a = r * nz;
    b = a + nz;
  }
};

template <int W, int U, typename Rows, typename Out = PlainOut>
__global__ void __launch_bounds__(256) k_spmv_vec(int64_t n, Rows rows,
                                                  const int32_t* __restrict__ col,
                                                  const double* __restrict__ val,
                                                  const double* __restrict__ x,
                                                  Out y, int64_t long_limit,
                                                  int32_t* long_rows, bool hint) {
  y.begin();
  const int lane = threadIdx.x & (W - 1);
  const unsigned mask = subwarp_mask(W);
  const int64_t nsub = (static_cast<int64_t>(gridDim.x) * blockDim.x) / W;
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / W; r < n;
       r += nsub) {
    int64_t a, b;
    rows.get(r, a, b);
    if (b - a > long_limit) {
      if (lane == 0) long_rows[1 + atomicAdd(long_rows, 1)] = static_cast<int32_t>(r);
      continue;
    }
    double acc = 0.0;
    for (int64_t p = a + lane; p < b; p += W * U) {
      int32_t c[U];
      double v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int64_t q = p + static_cast<int64_t>(j) * W;
        if (q < b) {
          c[j] = hint ? ld_stream_hint(col + q, pf) : ld_stream(col + q);
          v[j] = hint ? ld_stream_hint(val + q, pf) : ld_stream(val + q);
        }
      }
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (p + static_cast<int64_t>(j) * W < b)
          acc = fma(v[j], hint ? ld_x_hint(x + c[j], pl) : ld_x(x + c[j]), acc);
    }
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(mask, acc, o, W);
    if (lane == 0) y.put(r, acc);
  }
  y.done();
}

// ---- multi-row vector CRS -------------------------------------------------
// A sub-warp of W lanes owns R consecutive rows at a time and issues the
// loads of all R rows before consuming any (R x (entries/W) independent
// col/val loads and x gathers in flight per lane -- the single-row vector
// kernel was latency-bound).  The R partial sums are then reduced with a
// transpose-reduction: R-1 + log2(W/R) shuffles leave lane l holding row
// l / (W/R), instead of R*log2(W).
template <int W, int R>
__device__ __forceinline__ double transpose_reduce(double (&acc)[R], int lane, unsigned mask) {
  static_assert(R <= W, "R rows need at least R lanes");
  int off = W / 2;
#pragma unroll
  for (int s = R / 2; s >= 1; s /= 2, off /= 2) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int k = 0; k < s; ++k) {
      const double send = upper ? acc[k] : acc[k + s];
      const double keep = upper ? acc[k + s] : acc[k];
      acc[k] = keep + __shfl_xor_sync(mask, send, off, W);
    }
  }
  double v = acc[0];
#pragma unroll
  for (; off >= 1; off /= 2) v += __shfl_xor_sync(mask, v, off, W);
  return v;
}

template <int W, int R, typename Rows>
__global__ void __launch_bounds__(256) k_spmv_multi(int64_t n, Rows rows,
                                                    const int32_t* __restrict__ col,
                                                    const double* __restrict__ val,
                                                    const double* __restrict__ x,
                                                    double* __restrict__ y, int64_t long_limit,
                                                    int32_t* long_rows) {
  const int lane = threadIdx.x & (W - 1);
  const unsigned mask = subwarp_mask(W);
  const int64_t nsub = (static_cast<int64_t>(gridDim.x) * blockDim.x) / W;
  for (int64_t rb = ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / W) * R;
       rb < n; rb += nsub * R) {
    int64_t a[R], b[R];
    int64_t maxlen = 0;
    unsigned long_mask = 0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (rb + k < n) {
        rows.get(rb + k, a[k], b[k]);
      } else {
        a[k] = b[k] = 0;
      }
      if (b[k] - a[k] > long_limit) {
        if (lane == 0) long_rows[1 + atomicAdd(long_rows, 1)] = static_cast<int32_t>(rb + k);
        b[k] = a[k];  // handled by the block-per-row pass
        long_mask |= 1u << k;
      }
      maxlen = max(maxlen, b[k] - a[k]);
    }
    double acc[R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = 0.0;
    for (int64_t off = lane; off < maxlen; off += W) {
      int32_t c[R];
      double v[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int64_t p = a[k] + off;
        if (p < b[k]) {
          c[k] = ld_stream(col + p);
          v[k] = ld_stream(val + p);
        }
      }
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (a[k] + off < b[k]) acc[k] = fma(v[k], ld_x(x + c[k]), acc[k]);
    }
    const double total = transpose_reduce<W, R>(acc, lane, mask);
    constexpr int kLanesPerRow = W / R;
    if ((lane & (kLanesPerRow - 1)) == 0) {
      const int k = lane / kLanesPerRow;
      if (rb + k < n && !((long_mask >> k) & 1u)) y[rb + k] = total;
    }
  }
}

// ---- tiled CRS ("stream" phase + per-row reduction from shared memory) ----
// A block owns 256 consecutive rows.  Phase 1 streams the block's entries in
// chunks of kTileC with one entry per thread (coalesced col/val loads, the x
// gather, one multiply) into shared memory; phase 2 sums each row's products
// out of shared memory, one thread per row for short segments, one warp per
// segment for long ones.  ~8 warp instructions per 32 entries instead of ~90
// for the sub-warp-per-row kernel, and the entry stream is perfectly balanced
// inside a block whatever the row lengths.  Products are stored at a padded
// index (p + p/16) so that rows 16 doubles apart do not share a bank.
constexpr int kTileRows = 256;
constexpr int kTileC = 4096;
constexpr int kLongSeg = 48;

__device__ __forceinline__ int tile_idx(int p) { return p + (p >> 4); }

template <typename Rows>
__global__ void __launch_bounds__(256) k_spmv_tile(int64_t n, Rows rows,
                                                   const int32_t* __restrict__ col,
                                                   const double* __restrict__ val,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ y) {
  __shared__ double s_prod[kTileC + kTileC / 16];
  __shared__ int64_t s_ptr[kTileRows + 1];
  __shared__ double s_extra[kTileRows];
  __shared__ int s_list[kTileRows];
  __shared__ int s_nlist;
  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kTileRows;
  const int rows_here = static_cast<int>(min(static_cast<int64_t>(kTileRows), n - r0));
  for (int k = t; k <= kTileRows; k += blockDim.x) {
    int64_t a, b;
    const int64_t r = r0 + min(k, rows_here);
    if (k < rows_here) {
      rows.get(r, a, b);
    } else {
      rows.get(r0 + rows_here - 1, a, b);
      a = b;
    }
    s_ptr[k] = a;
  }
  s_extra[t] = 0.0;
  __syncthreads();
  const int64_t e0 = s_ptr[0], e1 = s_ptr[rows_here];
  const int64_t my_a = s_ptr[t < rows_here ? t : rows_here];
  const int64_t my_b = s_ptr[t < rows_here ? t + 1 : rows_here];
  double acc = 0.0;
  for (int64_t c0 = e0; c0 < e1; c0 += kTileC) {
    const int len = static_cast<int>(min(static_cast<int64_t>(kTileC), e1 - c0));
    // phase 1: products of the chunk, U = 4 entries per thread in flight
    for (int base = 0; base < len; base += 4 * 256) {
      int32_t c[4];
      double v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int q = base + j * 256 + t;
        if (q < len) {
          c[j] = ld_stream(col + c0 + q);
          v[j] = ld_stream(val + c0 + q);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int q = base + j * 256 + t;
        if (q < len) s_prod[tile_idx(q)] = v[j] * ld_x(x + c[j]);
      }
    }
    if (t == 0) s_nlist = 0;
    __syncthreads();
    // phase 2a: short segments, one thread per row
    const int lo = static_cast<int>(max(my_a, c0) - c0);
    const int hi = static_cast<int>(min(my_b, c0 + len) - c0);
    if (hi - lo > kLongSeg) {
      s_list[atomicAdd(&s_nlist, 1)] = t;
    } else {
      for (int q = lo; q < hi; ++q) acc += s_prod[tile_idx(q)];
    }
    __syncthreads();
    // phase 2b: long segments, one warp each
    const int nl = s_nlist;
    for (int i = warp; i < nl; i += blockDim.x >> 5) {
      const int owner = s_list[i];
      const int a = static_cast<int>(max(s_ptr[owner], c0) - c0);
      const int b = static_cast<int>(min(s_ptr[owner + 1], c0 + len) - c0);
      double s = 0.0;
      for (int q = a + lane; q < b; q += 32) s += s_prod[tile_idx(q)];
      s = warp_sum(s);
      if (lane == 0) s_extra[owner] += s;
    }
    __syncthreads();
  }
  if (t < rows_here) y[r0 + t] = acc + s_extra[t];
}

// ---- vector CRS with 128-bit loads ----------------------------------------
// Same sub-warp-per-row scheme, but each lane consumes aligned entry PAIRS
// (one double2 value load + one int2 index load): half the load
// instructions and L1 wavefronts per entry of the scalar kernel.  A row
// starting at an odd position has its first entry taken by lane 0 alone.
template <int W, int U, typename Rows, typename Out = PlainOut>
__global__ void __launch_bounds__(256) k_spmv_vec2(int64_t n, Rows rows,
                                                   const int32_t* __restrict__ col,
                                                   const double* __restrict__ val,
                                                   const double* __restrict__ x,
                                                   Out y, int64_t long_limit,
                                                   int32_t* long_rows) {
  y.begin();
  const int lane = threadIdx.x & (W - 1);
  const unsigned mask = subwarp_mask(W);
  const int64_t nsub = (static_cast<int64_t>(gridDim.x) * blockDim.x) / W;
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / W; r < n;
       r += nsub) {
    int64_t a, b;
    rows.get(r, a, b);
    if (b - a > long_limit) {
      if (lane == 0) long_rows[1 + atomicAdd(long_rows, 1)] = static_cast<int32_t>(r);
      continue;
    }
    // row-relative 32-bit offsets from 64-bit row bases (64-bit induction
    // variables cost ~25% on the 27-point stencil)
    const double* __restrict__ vr = val + a;
    const int32_t* __restrict__ cr = col + a;
    const int32_t len = static_cast<int32_t>(b - a);
    double acc = 0.0;
    int32_t k0 = 0;
    if ((a & 1) && len > 0) {  // odd start: peel one entry
      if (lane == 0) acc = ld_stream(vr) * ld_x(x + ld_stream(cr));
      k0 = 1;
    }
    for (int32_t p = k0 + 2 * lane; p < len; p += 2 * W * U) {
      double2 v[U];
      int2 c[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int32_t q = p + 2 * W * j;
        if (q + 1 < len) {
          v[j] = ld_stream2(reinterpret_cast<const double2*>(vr + q));
          c[j] = ld_stream2(reinterpret_cast<const int2*>(cr + q));
        } else if (q < len) {
          v[j].x = ld_stream(vr + q);
          c[j].x = ld_stream(cr + q);
        }
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int32_t q = p + 2 * W * j;
        if (q < len) acc = fma(v[j].x, ld_x(x + c[j].x), acc);
        if (q + 1 < len) acc = fma(v[j].y, ld_x(x + c[j].y), acc);
      }
    }
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(mask, acc, o, W);
    if (lane == 0) y.put(r, acc);
  }
  y.done();
}

// block per long row (queue filled by k_spmv_vec / k_spmv_multi)
template <typename Out = PlainOut>
__global__ void __launch_bounds__(256) k_spmv_crs_long(const int32_t* __restrict__ irp,
                                                       const int32_t* __restrict__ col,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ x,
                                                       Out y,
                                                       const int32_t* long_rows) {
  __shared__ double s_part[8];
  const int32_t count = *long_rows;
  for (int32_t q = blockIdx.x; q < count; q += gridDim.x) {
    const int32_t r = long_rows[1 + q];
    const int32_t a = __ldg(irp + r), b = __ldg(irp + r + 1);
    double acc = 0.0;
    for (int32_t p = a + threadIdx.x; p < b; p += blockDim.x * 4) {
      int32_t c[4];
      double v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int32_t pp = p + j * blockDim.x;
        if (pp < b) {
          c[j] = ld_stream(col + pp);
          v[j] = ld_stream(val + pp);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (p + j * static_cast<int32_t>(blockDim.x) < b) acc = fma(v[j], ld_x(x + c[j]), acc);
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += s_part[w];
      y.put(r, t);
    }
    __syncthreads();
  }
  y.done();
}

// ---- COO row-ordered: deterministic warp-segmented reduction -------------
// (spmv_coo_row_outer, spmv.cpp:79-101, :111-115).  Each warp owns the
// entries of whole rows: its nominal chunk [w*C, (w+1)*C) is moved to the
// first row start at or after the nominal bound, so no partial sums cross
// warps and no atomics or fix-up pass are needed.  Inside a warp, 32 entries
// at a time are reduced by an inclusive segmented scan keyed by row; the
// running row at the end of a group is carried to the next.  Empty rows are
// written as 0 by the warp owning the preceding non-empty row (warp 0 also
// owns the rows before the first entry).
__device__ __forceinline__ int64_t coo_row_chunk_start(const int32_t* __restrict__ row,
                                                       int64_t nnz, int64_t p0, int lane) {
  if (p0 <= 0) return 0;
  for (int64_t q0 = p0; q0 < nnz; q0 += 32) {
    const int64_t q = q0 + lane;
    bool start = false;
    if (q < nnz) start = __ldg(row + q) != __ldg(row + q - 1);
    const unsigned bal = __ballot_sync(kFull, start);
    if (bal) return q0 + __ffs(bal) - 1;
  }
  return nnz;
}

__device__ __forceinline__ void zero_fill(double* y, int64_t from, int64_t to) {
  for (int64_t r = from; r < to; ++r) y[r] = 0.0;
}

__global__ void __launch_bounds__(256) k_spmv_coo_row(int64_t n, int64_t nnz, int64_t chunk,
                                                      const int32_t* __restrict__ row,
                                                      const int32_t* __restrict__ col,
                                                      const double* __restrict__ val,
                                                      const double* __restrict__ x,
                                                      double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t st = coo_row_chunk_start(row, nnz, w * chunk, lane);
  const int64_t en = coo_row_chunk_start(row, nnz, (w + 1) * chunk, lane);
  if (st >= en) return;
  if (w == 0 && lane == 0) zero_fill(y, 0, __ldg(row));

  int32_t carry_row = -1;
  double carry_val = 0.0;
  for (int64_t base = st; base < en; base += 32) {
    const int64_t p = base + lane;
    const bool valid = p < en;
    int32_t rr = INT_MAX;
    double v = 0.0;
    if (valid) {
      rr = ld_stream(row + p);
      v = ld_stream(val + p) * ld_x(x + ld_stream(col + p));
    }
    // inclusive segmented scan keyed by row (rows are nondecreasing)
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double t = __shfl_up_sync(kFull, v, d);
      const int32_t tr = __shfl_up_sync(kFull, rr, d);
      if (lane >= d && tr == rr) v += t;
    }
    const int32_t first = __shfl_sync(kFull, rr, 0);
    if (carry_row >= 0) {
      if (rr == carry_row) v += carry_val;
      if (first != carry_row && lane == 0) {  // carried row ended at the group edge
        y[carry_row] = carry_val;
        zero_fill(y, carry_row + 1, first);
      }
    }
    const int32_t nr = __shfl_down_sync(kFull, rr, 1);
    if (valid && lane < 31 && nr != rr) {
      y[rr] = v;
      if (nr != INT_MAX) zero_fill(y, static_cast<int64_t>(rr) + 1, nr);
    }
    carry_row = __shfl_sync(kFull, rr, 31);
    carry_val = __shfl_sync(kFull, v, 31);
    if (carry_row == INT_MAX) carry_row = -1;
  }
  if (lane == 0) {
    if (carry_row >= 0) y[carry_row] = carry_val;
    const int64_t last = __ldg(row + en - 1);
    const int64_t next = en < nnz ? static_cast<int64_t>(__ldg(row + en)) : n;
    zero_fill(y, last + 1, next);
  }
}

// ---- COO row-ordered, 4 entries per lane ----------------------------------
// Same ownership rules as k_spmv_coo_row (row-aligned warp chunks, no
// atomics, deterministic), but each lane takes 4 consecutive entries with
// 128-bit loads (int4 rows, int4 columns, 2 x double2 values), reduces them
// locally, and one segmented shuffle scan per 128 entries joins the lanes:
// 4x fewer load instructions and shuffles per entry.  Invalid entries (before
// the chunk start / after its end inside the aligned quads) carry row -1 /
// INT_MAX and are never written.
__device__ __forceinline__ void fill_gap(double* y, int32_t a, int32_t b) {
  // rows strictly between two real rows a < b are empty
  if (a >= 0 && b != INT_MAX)
    for (int64_t r = static_cast<int64_t>(a) + 1; r < b; ++r) y[r] = 0.0;
}

__global__ void __launch_bounds__(256) k_spmv_coo_row4(int64_t n, int64_t nnz, int64_t chunk,
                                                       const int32_t* __restrict__ row,
                                                       const int32_t* __restrict__ col,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ x,
                                                       double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t st = coo_row_chunk_start(row, nnz, w * chunk, lane);
  const int64_t en = coo_row_chunk_start(row, nnz, (w + 1) * chunk, lane);
  if (st >= en) return;
  if (w == 0 && lane == 0)
    for (int64_t r = 0; r < __ldg(row); ++r) y[r] = 0.0;
  int32_t carry_row = -1;
  double carry_val = 0.0;
  for (int64_t base = st & ~int64_t(3); base < en; base += 128) {
    const int64_t q = base + 4 * lane;
    int32_t r[4];
    double p[4];
    if (q >= st && q + 3 < en) {
      const int4 rv = ld_stream4(reinterpret_cast<const int4*>(row + q));
      const int4 cv = ld_stream4(reinterpret_cast<const int4*>(col + q));
      const double2 v0 = ld_stream2(reinterpret_cast<const double2*>(val + q));
      const double2 v1 = ld_stream2(reinterpret_cast<const double2*>(val + q + 2));
      r[0] = rv.x; r[1] = rv.y; r[2] = rv.z; r[3] = rv.w;
      p[0] = v0.x * ld_x(x + cv.x);
      p[1] = v0.y * ld_x(x + cv.y);
      p[2] = v1.x * ld_x(x + cv.z);
      p[3] = v1.y * ld_x(x + cv.w);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t e = q + k;
        if (e < st) {
          r[k] = -1;
          p[k] = 0.0;
        } else if (e >= en) {
          r[k] = INT_MAX;
          p[k] = 0.0;
        } else {
          r[k] = ld_stream(row + e);
          p[k] = ld_stream(val + e) * ld_x(x + ld_stream(col + e));
        }
      }
    }
    // lane-local runs: the first run may continue from the left, the last
    // may continue to the right, the ones in between are complete
    double first_sum = p[0], run = p[0];
    bool in_first = true;
#pragma unroll
    for (int k = 1; k < 4; ++k) {
      if (r[k] != r[k - 1]) {
        if (!in_first && r[k - 1] >= 0 && r[k - 1] != INT_MAX) y[r[k - 1]] = run;
        fill_gap(y, r[k - 1], r[k]);
        in_first = false;
        run = p[k];
      } else {
        run += p[k];
        if (in_first) first_sum += p[k];
      }
    }
    const int32_t head = r[0], tail = r[3];
    const bool single = head == tail;
    const double tail_sum = run;
    // segmented inclusive scan of tail sums across lanes
    const int32_t prev_tail = __shfl_up_sync(kFull, tail, 1);
    bool flag = !single || lane == 0 || head != prev_tail;
    double s = tail_sum;
    if (lane == 0 && single && head == carry_row) s += carry_val;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double ts = __shfl_up_sync(kFull, s, d);
      const bool tf = __shfl_up_sync(kFull, flag, d);
      if (lane >= d && !flag) s += ts;
      if (lane >= d) flag = flag || tf;
    }
    const double s_prev = __shfl_up_sync(kFull, s, 1);
    // head run completing inside this lane
    if (!single && head >= 0) {
      double tot = first_sum;
      if (lane > 0 && head == prev_tail) tot += s_prev;
      if (lane == 0 && head == carry_row) tot += carry_val;
      y[head] = tot;
    }
    // a carried row that the group does not continue is complete
    const int32_t head0 = __shfl_sync(kFull, head, 0);
    if (lane == 0 && carry_row >= 0 && head0 != carry_row) {
      y[carry_row] = carry_val;
      fill_gap(y, carry_row, head0);
    }
    // tail run completing at the lane boundary
    const int32_t next_head = __shfl_down_sync(kFull, head, 1);
    if (lane < 31 && next_head != tail) {
      if (tail >= 0 && tail != INT_MAX) y[tail] = s;
      fill_gap(y, tail, next_head);
    }
    carry_row = __shfl_sync(kFull, tail, 31);
    carry_val = __shfl_sync(kFull, s, 31);
    if (carry_row == INT_MAX || carry_row < 0) carry_row = -1;
  }
  if (lane == 0) {
    if (carry_row >= 0) y[carry_row] = carry_val;
    const int64_t last = __ldg(row + en - 1);
    const int64_t next = en < nnz ? static_cast<int64_t>(__ldg(row + en)) : n;
    for (int64_t r = last + 1; r < next; ++r) y[r] = 0.0;
  }
}

// ---- COO column-ordered (spmv_coo_col_outer, spmv.cpp:105-109) ------------
// Rows are scattered, so partial sums go to y through fp64 reductions
// (RED.ADD.F64 at L2); y is zeroed first.  4 entries per thread per step
// with 128-bit index loads.
__global__ void __launch_bounds__(256) k_spmv_coo_col(int64_t nnz,
                                                      const int32_t* __restrict__ row,
                                                      const int32_t* __restrict__ col,
                                                      const double* __restrict__ val,
                                                      const double* __restrict__ x,
                                                      double* __restrict__ y) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t quads = nnz >> 2;
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < quads;
       q += stride) {
    const int4 r = ld_stream4(reinterpret_cast<const int4*>(row) + q);
    const int4 c = ld_stream4(reinterpret_cast<const int4*>(col) + q);
    const double2 v0 = ld_stream2(reinterpret_cast<const double2*>(val) + 2 * q);
    const double2 v1 = ld_stream2(reinterpret_cast<const double2*>(val) + 2 * q + 1);
    atomicAdd(y + r.x, v0.x * ld_x(x + c.x));
    atomicAdd(y + r.y, v0.y * ld_x(x + c.y));
    atomicAdd(y + r.z, v1.x * ld_x(x + c.z));
    atomicAdd(y + r.w, v1.y * ld_x(x + c.w));
  }
  if (blockIdx.x == 0 && threadIdx.x < (nnz & 3)) {
    const int64_t p = (quads << 2) + threadIdx.x;
    atomicAdd(y + row[p], val[p] * ld_x(x + col[p]));
  }
}

// ---- ELL band-major (spmv_ell_inner, spmv.cpp:117-136) --------------------
// One thread per row pair: each band is one double2 + one int2 load per
// thread, fully coalesced (ld is a multiple of 32 so every band starts
// 256-byte aligned).  Bands are walked in order with U loads in flight.
// Every slot is multiplied, padding included (the ELL contract).
// one row pair (i, i+1) over bands [k_begin, k_end)
template <int U, bool H>
__device__ __forceinline__ void ell_pair(int64_t i, int32_t k_begin, int32_t k_end, int64_t ld,
                                         const double* __restrict__ val,
                                         const int32_t* __restrict__ col,
                                         const double* __restrict__ x, double& a0, double& a1) {
  a0 = 0.0;
  a1 = 0.0;
  const double2* vp = reinterpret_cast<const double2*>(val + i);
  const int2* cp = reinterpret_cast<const int2*>(col + i);
  const int64_t step = ld >> 1;  // in double2 / int2 units
  uint64_t pf = 0, pl = 0;
  if (H) {
    pf = policy_evict_first();
    pl = policy_evict_last();
  }
  auto lv = [&](int64_t off) { return H ? ld_stream2_hint(vp + off, pf) : ld_stream2(vp + off); };
  auto lc = [&](int64_t off) { return H ? ld_stream2_hint(cp + off, pf) : ld_stream2(cp + off); };
  auto lx = [&](int32_t c) { return H ? ld_x_hint(x + c, pl) : ld_x(x + c); };
  int32_t k = k_begin;
  for (; k + U <= k_end; k += U) {
    double2 v[U];
    int2 c[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      v[j] = lv(static_cast<int64_t>(k + j) * step);
      c[j] = lc(static_cast<int64_t>(k + j) * step);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      a0 = fma(v[j].x, lx(c[j].x), a0);
      a1 = fma(v[j].y, lx(c[j].y), a1);
    }
  }
  for (; k < k_end; ++k) {
    const double2 v = lv(static_cast<int64_t>(k) * step);
    const int2 c = lc(static_cast<int64_t>(k) * step);
    a0 = fma(v.x, lx(c.x), a0);
    a1 = fma(v.y, lx(c.y), a1);
  }
}

template <int U, bool H, typename Out = PlainOut>
__global__ void __launch_bounds__(256) k_spmv_ell_cm(int64_t n, int32_t k_begin, int32_t k_end,
                                                     int64_t ld, const double* __restrict__ val,
                                                     const int32_t* __restrict__ col,
                                                     const double* __restrict__ x,
                                                     Out y) {
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double a0, a1;
  if constexpr (std::is_same_v<Out, PlainOut>) {
    // one pair per thread, the grid covers every pair
    const int64_t i = 2 * t0;
    if (i >= n) return;
    ell_pair<U, H>(i, k_begin, k_end, ld, val, col, x, a0, a1);
    // rows past n in the last pair are ld padding: their result is dropped
    y.put(i, a0);
    if (i + 1 < n) y.put(i + 1, a1);
  } else {
    // pushed results: a capped grid walks the pairs, so the per-CTA step
    // handshake (flag wait, arrival count) stays cheap; no early return,
    // done() synchronises the CTA
    y.begin();
    for (int64_t t = t0; 2 * t < n; t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int64_t i = 2 * t;
      ell_pair<U, H>(i, k_begin, k_end, ld, val, col, x, a0, a1);
      y.put(i, a0);
      if (i + 1 < n) y.put(i + 1, a1);
    }
    y.done();
  }
}

// ---- ELL band-major with the matrix streamed by the TMA engine ------------
// The bands of a CTA's 256 rows are contiguous 2 KB (values) / 1 KB (column)
// runs: one elected thread moves them into a shared-memory ring with 1-D bulk
// copies (cp.async.bulk, completion counted on an mbarrier), so the matrix
// stream never occupies the LSU / L1 request path that the random x gathers
// saturate; threads read their row pair's slots from shared memory and keep
// KB bands of gathers in flight.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int THREADS, int KB, int STAGES>
__global__ void __launch_bounds__(THREADS) k_spmv_ell_bulk(int64_t n, int32_t nz, int64_t ld,
                                                           const double* __restrict__ val,
                                                           const int32_t* __restrict__ col,
                                                           const double* __restrict__ x,
                                                           double* __restrict__ y) {
  // persistent: the CTA walks row blocks blockIdx, +gridDim, ... and its
  // ring of STAGES x KB bands runs continuously across them
  constexpr int R = 2 * THREADS;  // rows per block (2 per thread)
  extern __shared__ __align__(128) unsigned char s_raw[];
  double* s_val = reinterpret_cast<double*>(s_raw);                 // [STAGES][KB][R]
  int32_t* s_col = reinterpret_cast<int32_t*>(s_val + STAGES * KB * R);
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int tid = threadIdx.x, lane = tid & 31;
  const int T = (nz + KB - 1) / KB;                       // band chunks per row block
  const int64_t nblocks = (ld + R - 1) / R;
  const int64_t my_blocks = blockIdx.x < nblocks ? (nblocks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = my_blocks * T;                    // ring items of this CTA
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], THREADS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t g) {
    const int s = static_cast<int>(g % STAGES);
    const int64_t rb = blockIdx.x + (g / T) * gridDim.x;
    const int k0 = static_cast<int>(g % T) * KB, kb = min(KB, nz - k0);
    const int64_t r0 = rb * R;
    const int rows = static_cast<int>(min(static_cast<int64_t>(R), ld - r0));
    mbar_expect_tx(&full[s], static_cast<uint32_t>(kb * rows * 12));
    for (int j = 0; j < kb; ++j) {
      const int64_t off = static_cast<int64_t>(k0 + j) * ld + r0;
      bulk_g2s(s_val + (s * KB + j) * R, val + off, rows * 8, &full[s]);
      bulk_g2s(s_col + (s * KB + j) * R, col + off, rows * 4, &full[s]);
    }
  };
  if (tid == 0)
    for (int64_t g = 0; g < min(static_cast<int64_t>(STAGES), total); ++g) issue(g);
  double a0 = 0.0, a1 = 0.0;
  for (int64_t g = 0; g < total; ++g) {
    const int s = static_cast<int>(g % STAGES);
    const uint32_t parity = static_cast<uint32_t>((g / STAGES) & 1);
    const int t = static_cast<int>(g % T);
    const int64_t r0 = (blockIdx.x + (g / T) * gridDim.x) * R;
    const int rows = static_cast<int>(min(static_cast<int64_t>(R), ld - r0));
    mbar_wait(&full[s], parity);
    const int kb = min(KB, nz - t * KB);
    if (2 * tid < rows) {
      double2 v[KB];
      int2 c[KB];
#pragma unroll
      for (int j = 0; j < KB; ++j)
        if (j < kb) {
          v[j] = reinterpret_cast<const double2*>(s_val + (s * KB + j) * R)[tid];
          c[j] = reinterpret_cast<const int2*>(s_col + (s * KB + j) * R)[tid];
        }
#pragma unroll
      for (int j = 0; j < KB; ++j)
        if (j < kb) {
          a0 = fma(v[j].x, ld_x(x + c[j].x), a0);
          a1 = fma(v[j].y, ld_x(x + c[j].y), a1);
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (tid == 0 && g + STAGES < total) {
      mbar_wait(&empty[s], parity);
      issue(g + STAGES);
    }
    if (t == T - 1) {  // row block done
      const int64_t i = r0 + 2 * tid;
      if (i < n) y[i] = a0;
      if (i + 1 < n) y[i + 1] = a1;
      a0 = a1 = 0.0;
    }
  }
}

// band-split variant (spmv_ell_outer): chunk s of the bands writes
// partial[s*n + i]; then an ascending-chunk reduction (reduce_partials,
// spmv.cpp:56-62) makes the result independent of scheduling.
template <int U>
__global__ void __launch_bounds__(256) k_spmv_ell_cm_part(int64_t n, int32_t nz, int32_t splits,
                                                          int64_t ld,
                                                          const double* __restrict__ val,
                                                          const int32_t* __restrict__ col,
                                                          const double* __restrict__ x,
                                                          double* __restrict__ partial) {
  const int32_t s = blockIdx.y;
  // partition_range (spmv.cpp:36-54), 0-based
  const int32_t base = nz / splits, rem = nz % splits;
  const int32_t kb = s * base + min(s, rem);
  const int32_t ke = kb + base + (s < rem ? 1 : 0);
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t i = 2 * t;
  if (i >= n) return;
  double a0 = 0.0, a1 = 0.0;
  const double2* vp = reinterpret_cast<const double2*>(val + i);
  const int2* cp = reinterpret_cast<const int2*>(col + i);
  const int64_t step = ld >> 1;
  int32_t k = kb;
  for (; k + U <= ke; k += U) {
    double2 v[U];
    int2 c[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      v[j] = ld_stream2(vp + static_cast<int64_t>(k + j) * step);
      c[j] = ld_stream2(cp + static_cast<int64_t>(k + j) * step);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      a0 = fma(v[j].x, ld_x(x + c[j].x), a0);
      a1 = fma(v[j].y, ld_x(x + c[j].y), a1);
    }
  }
  for (; k < ke; ++k) {
    const double2 v = ld_stream2(vp + static_cast<int64_t>(k) * step);
    const int2 c = ld_stream2(cp + static_cast<int64_t>(k) * step);
    a0 = fma(v.x, ld_x(x + c.x), a0);
    a1 = fma(v.y, ld_x(x + c.y), a1);
  }
  double* out = partial + static_cast<int64_t>(s) * n;
  out[i] = a0;
  if (i + 1 < n) out[i + 1] = a1;
}

__global__ void k_reduce_partials(int64_t n, int32_t splits, const double* __restrict__ partial,
                                  double* __restrict__ y) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    double acc = 0.0;
    for (int32_t s = 0; s < splits; ++s) acc += partial[static_cast<int64_t>(s) * n + i];
    y[i] = acc;
  }
}

int g_l2_hint = 0;  // L2 evict_first (matrix) / evict_last (x) policies
int g_coo_variant = 1;  // 1: 4 entries per lane (k_spmv_coo_row4), 0: scalar
int g_coo_chunk = 2048;  // entries per warp of k_spmv_coo_row4 (multiple of 128)
bool g_coo_chunk_auto = true;  // wave-aware choice between 2048 and 1024
int64_t g_coo_cap = 0;          // resident warps of k_spmv_coo_row4 (occupancy API)
void coo_row4_capacity() {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv_coo_row4, 256, 0);
  g_coo_cap = static_cast<int64_t>(kSMs) * std::max(per_sm, 1) * 8;
}
int g_rm_variant = -1;  // row-major ELL variant override (tuning)
int g_ell_variant = 0;  // band-major ELL: 0 = LSU loads, 1/2 = TMA bulk-copy ring (8x3 / 4x4)

template <int W, int U, typename Rows, typename Out>
void launch_vec(int64_t n, Rows rows, const int32_t* col, const double* val, const double* x,
                Out y, int64_t long_limit, int32_t* long_rows, cudaStream_t s) {
  const int64_t threads = n * W;
  k_spmv_vec<W, U, Rows, Out><<<grid_for(threads, 256, 8), 256, 0, s>>>(
      n, rows, col, val, x, y, long_limit, long_rows, g_l2_hint != 0);
}

template <int W, int R, typename Rows>
void launch_multi(int64_t n, Rows rows, const int32_t* col, const double* val, const double* x,
                  double* y, int64_t long_limit, int32_t* long_rows, cudaStream_t s) {
  const int64_t threads = (n + R - 1) / R * W;
  k_spmv_multi<W, R, Rows><<<grid_for(threads, 256, 8), 256, 0, s>>>(n, rows, col, val, x, y,
                                                                     long_limit, long_rows);
}

int g_crs_variant = -1;  // tuning override (spmvtk_k_tune), -1 = heuristic

template <typename Rows, typename Out>
void dispatch_vec(double mean, int64_t max_row, int64_t n, Rows rows, const int32_t* col,
                  const double* val, const double* x, Out y, int64_t long_limit,
                  int32_t* long_rows, cudaStream_t s) {
  int v = g_crs_variant;
  if (v < 0) {
    // measured on B200 (tools/tune_crs.py, profiles/r01_tune_crs.txt): few
    // lanes per row (more rows in flight) win unless the rows are skewed
    // (profiles/r01_tune_crs2.txt): 128-bit pair loads from 6 entries/row up
    if (static_cast<double>(max_row) > 8.0 * mean + 8.0) v = 16;  // W=8 pairs
    else if (mean <= 6.0) v = 12;                               // W=4 scalar
    else if (mean <= 30.0) v = 18;                              // W=4 pairs
    else if (mean <= 64.0) v = 16;                              // W=8 pairs
    else v = 17;                                                // W=16 pairs
    if constexpr (!std::is_same_v<Rows, CrsRows>) {
      // row-major ELL takes the same choice (profiles/r01_tune_rm2.txt: the
      // pair kernel also wins at odd band counts once its offsets are 32-bit)
      if (g_rm_variant >= 0) v = g_rm_variant;
    }
  }
  if constexpr (!std::is_same_v<Out, PlainOut>) {
    // pushed results: the multi-row / tiled variants have no push epilogue
    if (v < 11 && v != 0) v = 18;
  }
  switch (v) {
    case 15: case 16: case 17: case 18: case 19: {
      const int64_t W = v == 15 ? 4 : v == 16 ? 8 : v == 17 ? 16 : v == 18 ? 4 : 8;
      const int blocks = grid_for(n * W, 256, 8);
      if (v == 15) k_spmv_vec2<4, 2, Rows, Out><<<blocks, 256, 0, s>>>(n, rows, col, val, x, y, long_limit, long_rows);
      if (v == 16) k_spmv_vec2<8, 1, Rows, Out><<<blocks, 256, 0, s>>>(n, rows, col, val, x, y, long_limit, long_rows);
      if (v == 17) k_spmv_vec2<16, 1, Rows, Out><<<blocks, 256, 0, s>>>(n, rows, col, val, x, y, long_limit, long_rows);
      if (v == 18) k_spmv_vec2<4, 1, Rows, Out><<<blocks, 256, 0, s>>>(n, rows, col, val, x, y, long_limit, long_rows);
      if (v == 19) k_spmv_vec2<8, 2, Rows, Out><<<blocks, 256, 0, s>>>(n, rows, col, val, x, y, long_limit, long_rows);
      break;
    }
    case 11: launch_vec<8, 2>(n, rows, col, val, x, y, long_limit, long_rows, s); break;
    case 12: launch_vec<4, 2>(n, rows, col, val, x, y, long_limit, long_rows, s); break;
    case 13: launch_vec<32, 4>(n, rows, col, val, x, y, long_limit, long_rows, s); break;
    case 14: launch_vec<32, 2>(n, rows, col, val, x, y, long_limit, long_rows, s); break;
    case 0: launch_vec<16, 2>(n, rows, col, val, x, y, long_limit, long_rows, s); break;
    default:
      if constexpr (std::is_same_v<Out, PlainOut>) {
        double* yy = y.y;
        switch (v) {
          case 1: launch_multi<4, 4>(n, rows, col, val, x, yy, long_limit, long_rows, s); break;
          case 2: launch_multi<8, 4>(n, rows, col, val, x, yy, long_limit, long_rows, s); break;
          case 3: launch_multi<16, 4>(n, rows, col, val, x, yy, long_limit, long_rows, s); break;
          case 4: launch_multi<32, 4>(n, rows, col, val, x, yy, long_limit, long_rows, s); break;
          case 5: launch_multi<8, 2>(n, rows, col, val, x, yy, long_limit, long_rows, s); break;
          case 6: launch_multi<8, 8>(n, rows, col, val, x, yy, long_limit, long_rows, s); break;
          case 7: launch_multi<16, 8>(n, rows, col, val, x, yy, long_limit, long_rows, s); break;
          case 8: launch_multi<4, 2>(n, rows, col, val, x, yy, long_limit, long_rows, s); break;
          case 9: launch_multi<16, 2>(n, rows, col, val, x, yy, long_limit, long_rows, s); break;
          case 10:
            k_spmv_tile<Rows><<<static_cast<unsigned>((n + kTileRows - 1) / kTileRows), kTileRows,
                                0, s>>>(n, rows, col, val, x, yy);
            break;
          default: launch_multi<8, 4>(n, rows, col, val, x, yy, long_limit, long_rows, s); break;
        }
      }
      break;
  }
}

}  // namespace

extern "C" {

int spmvtk_k_spmv_crs(int64_t n, const int32_t* irp, const int32_t* icol, const double* val,
                      const double* x, double* y, double mean_row, int32_t max_row,
                      int32_t* long_rows, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) SPMVTK_LAUNCH_RETURN();
  const int64_t long_limit = spmvtk_k_crs_long_limit(mean_row);
  const bool use_long = long_rows != nullptr && max_row > long_limit;
  if (use_long) cudaMemsetAsync(long_rows, 0, sizeof(int32_t), s);
  dispatch_vec(mean_row, max_row, n, CrsRows{irp}, icol, val, x, PlainOut{y},
               use_long ? long_limit : INT64_MAX, long_rows, s);
  if (use_long)
    k_spmv_crs_long<<<kSMs * 4, 256, 0, s>>>(irp, icol, val, x, PlainOut{y}, long_rows);
  SPMVTK_LAUNCH_RETURN();
}

namespace {
spmvtk_push_sync no_sync() {
  spmvtk_push_sync z{};
  return z;
}
// an empty shard launches no SpMV: its step still waits and signals
int sync_only(const spmvtk_push_sync* sync, void* stream) {
  if (sync == nullptr) SPMVTK_LAUNCH_RETURN();
  if (sync->nwait > 0) {
    const int rc = spmvtk_k_flags_wait(sync->wait_flags, sync->nwait, sync->wait_value,
                                       sync->timeout_ns, sync->status, stream);
    if (rc) return rc;
  }
  if (sync->counter != nullptr) return spmvtk_k_flags_signal(&sync->signal, sync->signal_value, stream);
  SPMVTK_LAUNCH_RETURN();
}
bool bad_push(const spmvtk_push* push, const spmvtk_push_sync* sync) {
  if (push == nullptr || push->ndst < 1 || push->ndst > SPMVTK_MAX_PEERS) return true;
  if (sync && (sync->nwait < 0 || sync->nwait > SPMVTK_MAX_PEERS ||
               (sync->nwait > 0 && (sync->wait_flags == nullptr || sync->status == nullptr)) ||
               sync->signal.n < 0 || sync->signal.n > SPMVTK_MAX_PEERS))
    return true;
  return false;
}
}  // namespace

int spmvtk_k_spmv_crs_push(int64_t n, const int32_t* irp, const int32_t* icol,
                           const double* val, const double* x, const spmvtk_push* push,
                           const spmvtk_push_sync* sync, double mean_row, int32_t max_row,
                           int32_t* long_rows, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (bad_push(push, sync)) return static_cast<int>(cudaErrorInvalidValue);
  if (n <= 0) return sync_only(sync, stream);
  const int64_t long_limit = spmvtk_k_crs_long_limit(mean_row);
  const bool use_long = long_rows != nullptr && max_row > long_limit;
  if (use_long) cudaMemsetAsync(long_rows, 0, sizeof(int32_t), s);
  PushOut vec{*push, sync ? *sync : no_sync()};
  if (use_long) {
    // the long-row pass runs after the vector kernel: it signals, the
    // vector kernel only waits
    PushOut lng = vec;
    vec.s.counter = nullptr;
    vec.s.signal.n = 0;
    lng.s.nwait = 0;
    dispatch_vec(mean_row, max_row, n, CrsRows{irp}, icol, val, x, vec, long_limit, long_rows, s);
    k_spmv_crs_long<<<kSMs * 4, 256, 0, s>>>(irp, icol, val, x, lng, long_rows);
  } else {
    dispatch_vec(mean_row, max_row, n, CrsRows{irp}, icol, val, x, vec, INT64_MAX, long_rows, s);
  }
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_spmv_coo_row(int64_t n, int64_t nnz, const int32_t* row, const int32_t* col,
                          const double* val, const double* x, double* y, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) SPMVTK_LAUNCH_RETURN();
  if (nnz == 0) {
    cudaMemsetAsync(y, 0, static_cast<size_t>(n) * sizeof(double), s);
    SPMVTK_LAUNCH_RETURN();
  }
  const bool quad = g_coo_variant != 0 && (reinterpret_cast<uintptr_t>(row) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(col) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(val) & 15) == 0;
  int64_t chunk = quad ? g_coo_chunk : 1024;
  if (quad && g_coo_chunk_auto) {
    // wave quantisation: one warp per chunk, so pick the chunk (2048 or
    // 1024 entries) whose warp count fills the last wave of resident warps
    // best (config 2: 8192 warps = 1.15 waves at 2048 vs 2.3 at 1024;
    // profiles/r01_tune_coo_chunk.txt)
    if (g_coo_cap == 0) coo_row4_capacity();  // normally done by spmvtk_k_preload
    const int64_t cap = g_coo_cap;
    auto eff = [&](int64_t c) {
      const int64_t w = (nnz + c - 1) / c;
      return static_cast<double>(w) / static_cast<double>(((w + cap - 1) / cap) * cap);
    };
    chunk = eff(1024) > eff(2048) + 0.05 ? 1024 : 2048;
  }
  const int64_t warps = (nnz + chunk - 1) / chunk;
  const int64_t blocks = (warps * 32 + 255) / 256;
  if (quad)
    k_spmv_coo_row4<<<static_cast<unsigned>(blocks), 256, 0, s>>>(n, nnz, chunk, row, col, val,
                                                                  x, y);
  else
    k_spmv_coo_row<<<static_cast<unsigned>(blocks), 256, 0, s>>>(n, nnz, chunk, row, col, val,
                                                                 x, y);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_spmv_coo_col(int64_t n, int64_t nnz, const int32_t* row, const int32_t* col,
                          const double* val, const double* x, double* y, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) SPMVTK_LAUNCH_RETURN();
  cudaMemsetAsync(y, 0, static_cast<size_t>(n) * sizeof(double), s);
  if (nnz > 0)
    k_spmv_coo_col<<<grid_for((nnz + 3) / 4, 256, 8), 256, 0, s>>>(nnz, row, col, val, x, y);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_spmv_ell_cm(int64_t n, int32_t nz, int64_t ld, const double* val,
                         const int32_t* col, const double* x, double* y, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) SPMVTK_LAUNCH_RETURN();
  if (nz == 0) {
    cudaMemsetAsync(y, 0, static_cast<size_t>(n) * sizeof(double), s);
    SPMVTK_LAUNCH_RETURN();
  }
  if (g_ell_variant >= 1 && g_ell_variant <= 4) {  // matrix streamed by TMA bulk copies
    auto go = [&](auto kern, int threads, int kb, int stages, int ctas_per_sm) {
      const int smem = stages * kb * 2 * threads * 12;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const int64_t nblocks = (ld + 2 * threads - 1) / (2 * threads);
      const unsigned grid =
          static_cast<unsigned>(std::min<int64_t>(nblocks, int64_t(kSMs) * ctas_per_sm));
      kern<<<grid, threads, smem, s>>>(n, nz, ld, val, col, x, y);
    };
    if (g_ell_variant == 1) go(k_spmv_ell_bulk<128, 8, 4>, 128, 8, 4, 2);
    if (g_ell_variant == 2) go(k_spmv_ell_bulk<256, 4, 4>, 256, 4, 4, 2);
    if (g_ell_variant == 3) go(k_spmv_ell_bulk<256, 4, 3>, 256, 4, 3, 3);
    if (g_ell_variant == 4) go(k_spmv_ell_bulk<512, 2, 4>, 512, 2, 4, 2);
    SPMVTK_LAUNCH_RETURN();
  }
  const int64_t pairs = (n + 1) / 2;
  const unsigned blocks = static_cast<unsigned>((pairs + 255) / 256);
  if (g_l2_hint)
    k_spmv_ell_cm<4, true><<<blocks, 256, 0, s>>>(n, 0, nz, ld, val, col, x, PlainOut{y});
  else
    k_spmv_ell_cm<4, false><<<blocks, 256, 0, s>>>(n, 0, nz, ld, val, col, x, PlainOut{y});
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_spmv_ell_cm_push(int64_t n, int32_t nz, int64_t ld, const double* val,
                              const int32_t* col, const double* x, const spmvtk_push* push,
                              const spmvtk_push_sync* sync, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (bad_push(push, sync)) return static_cast<int>(cudaErrorInvalidValue);
  if (n <= 0) return sync_only(sync, stream);
  const int64_t pairs = (n + 1) / 2;
  const unsigned blocks = static_cast<unsigned>((pairs + 255) / 256);
  k_spmv_ell_cm<4, false, PushOut><<<std::min<unsigned>(blocks, kSMs * 8), 256, 0, s>>>(
      n, 0, nz, ld, val, col, x, PushOut{*push, sync ? *sync : no_sync()});
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_spmv_ell_cm_split(int64_t n, int32_t nz, int64_t ld, const double* val,
                               const int32_t* col, const double* x, double* y, int32_t splits,
                               double* partial, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (splits <= 1 || partial == nullptr || nz <= 1)
    return spmvtk_k_spmv_ell_cm(n, nz, ld, val, col, x, y, stream);
  if (splits > nz) splits = nz;
  const int64_t pairs = (n + 1) / 2;
  dim3 grid(static_cast<unsigned>((pairs + 255) / 256), static_cast<unsigned>(splits));
  k_spmv_ell_cm_part<4><<<grid, 256, 0, s>>>(n, nz, splits, ld, val, col, x, partial);
  k_reduce_partials<<<grid_for(n, 256), 256, 0, s>>>(n, splits, partial, y);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_spmv_ell_rm(int64_t n, int32_t nz, const double* val, const int32_t* col,
                         const double* x, double* y, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) SPMVTK_LAUNCH_RETURN();
  dispatch_vec(static_cast<double>(nz), nz, n, EllRowMajorRows{nz}, col, val, x, PlainOut{y}, INT64_MAX,
               nullptr, s);
  SPMVTK_LAUNCH_RETURN();
}

int64_t spmvtk_k_crs_long_limit(double mean_row) {
  // rows this much longer than average would serialise one sub-warp: they go
  // to the block-per-row pass (power-law rows, BASELINE config 4)
  const int64_t m = static_cast<int64_t>(mean_row + 0.999);
  return std::max<int64_t>(256, std::min<int64_t>(4096, 32 * m));
}

int spmvtk_k_tune(const char* key, int value) {
  if (key && std::string(key) == "crs_variant") {
    g_crs_variant = value;
    return 0;
  }
  if (key && std::string(key) == "l2_hint") {
    g_l2_hint = value;
    return 0;
  }
  if (key && std::string(key) == "coo_variant") {
    g_coo_variant = value;
    return 0;
  }
  if (key && std::string(key) == "ell_variant") {
    g_ell_variant = value;
    return 0;
  }
  if (key && std::string(key) == "coo_chunk") {  // <= 0: automatic
    g_coo_chunk_auto = value <= 0;
    g_coo_chunk = value >= 128 ? (value / 128) * 128 : 2048;
    return 0;
  }
  if (key && std::string(key) == "rm_variant") {
    g_rm_variant = value;
    return 0;
  }
  return spmvtk_k_tune_convert(key, value);
}

int spmvtk_k_preload(void) {
  // touching the attributes of every kernel forces module load
  spmvtk_dev::preload_convert();
  spmvtk_dev::preload_util();
  spmvtk_dev::preload_inverse();
  if (const char* c = std::getenv("SPMVTK_L1_CARVEOUT")) {  // experiment hook
    const int pct = std::atoi(c);
    cudaFuncSetAttribute(k_spmv_ell_cm<4, false>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaFuncSetAttribute(k_spmv_vec2<4, 1, CrsRows>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaFuncSetAttribute(k_spmv_vec2<8, 1, CrsRows>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaFuncSetAttribute(k_spmv_vec2<16, 1, CrsRows>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  }
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_spmv_crs_long<PlainOut>);
  cudaFuncGetAttributes(&a, k_spmv_crs_long<PushOut>);
  cudaFuncGetAttributes(&a, k_spmv_ell_cm<4, false, PushOut>);
  cudaFuncGetAttributes(&a, k_spmv_vec2<4, 1, CrsRows, PushOut>);
  cudaFuncGetAttributes(&a, k_spmv_vec2<8, 1, CrsRows, PushOut>);
  cudaFuncGetAttributes(&a, k_spmv_vec2<16, 1, CrsRows, PushOut>);
  cudaFuncGetAttributes(&a, k_spmv_vec<4, 2, CrsRows, PushOut>);
  cudaFuncGetAttributes(&a, k_spmv_coo_row);
  cudaFuncGetAttributes(&a, k_spmv_coo_row4);
  coo_row4_capacity();
  cudaFuncGetAttributes(&a, k_spmv_coo_col);
  cudaFuncGetAttributes(&a, k_spmv_ell_cm<4, false>);
  cudaFuncGetAttributes(&a, k_spmv_ell_cm<4, true>);
  cudaFuncGetAttributes(&a, k_spmv_ell_cm_part<4>);
  cudaFuncGetAttributes(&a, k_reduce_partials);
  cudaFuncGetAttributes(&a, k_spmv_vec<2, 2, CrsRows>);
  cudaFuncGetAttributes(&a, k_spmv_vec<4, 2, CrsRows>);
  cudaFuncGetAttributes(&a, k_spmv_vec<8, 2, CrsRows>);
  cudaFuncGetAttributes(&a, k_spmv_vec<16, 2, CrsRows>);
  cudaFuncGetAttributes(&a, k_spmv_vec<32, 4, CrsRows>);
#define PRELOAD_MULTI(ROWS)                                 \
  cudaFuncGetAttributes(&a, k_spmv_multi<4, 4, ROWS>);      \
  cudaFuncGetAttributes(&a, k_spmv_multi<8, 4, ROWS>);      \
  cudaFuncGetAttributes(&a, k_spmv_multi<16, 4, ROWS>);     \
  cudaFuncGetAttributes(&a, k_spmv_multi<32, 4, ROWS>);
  PRELOAD_MULTI(CrsRows)
  PRELOAD_MULTI(EllRowMajorRows)
#undef PRELOAD_MULTI
  cudaFuncGetAttributes(&a, k_spmv_vec<2, 2, EllRowMajorRows>);
  cudaFuncGetAttributes(&a, k_spmv_vec<4, 2, EllRowMajorRows>);
  cudaFuncGetAttributes(&a, k_spmv_vec<8, 2, EllRowMajorRows>);
  cudaFuncGetAttributes(&a, k_spmv_vec<16, 2, EllRowMajorRows>);
  cudaFuncGetAttributes(&a, k_spmv_vec<32, 4, EllRowMajorRows>);
  SPMVTK_LAUNCH_RETURN();
}

}  // extern "C"
