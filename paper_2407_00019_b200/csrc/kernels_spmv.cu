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
#include "spmv_out.cuh"
#include "spmvtk/spmvtk.h"
#include "spmvtk/spmvtk_kernels.h"

using namespace spmvtk_dev;

namespace {

__device__ __forceinline__ unsigned subwarp_mask(int W) {
  if (W == 32) return kFull;
  const int lane = threadIdx.x & 31;
  return ((1u << W) - 1u) << (lane & ~(W - 1));
}

int g_ell_banded = -1;  // tuning: SM-local band-major ELL (-1 auto from the band shape)

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
    double acc = 0.0;
    for (int64_t p = a + lane; p < b; p += W * U) {
      int32_t c[U];
      double v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int64_t q = p + static_cast<int64_t>(j) * W;
        if (q < b) {
          c[j] = ld_stream(col + q);
          v[j] = ld_stream(val + q);
        }
      }
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (p + static_cast<int64_t>(j) * W < b)
          acc = fma(v[j], ld_x(x + c[j]), acc);
    }
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(mask, acc, o, W);
    if (lane == 0) y.put(r, acc);
  }
  y.done();
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

// W lanes per row, aligned entry QUADS: a lane's four values come in one
// 256-bit L2-evict-first load, its four columns in one 128-bit load (the
// base arrays must be 32- / 16-byte aligned: checked at launch).  The row's
// first (4 - a % 4) % 4 entries are peeled, one per lane.
template <int W, typename Rows, typename Out = PlainOut>
__global__ void __launch_bounds__(256) k_spmv_vec4(int64_t n, Rows rows,
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
    const int32_t len = static_cast<int32_t>(b - a);
    const int32_t head = min(len, static_cast<int32_t>((4 - (a & 3)) & 3));
    double acc = 0.0;
    for (int32_t t = lane; t < head; t += W)
      acc = fma(ld_stream(val + a + t), ld_x(x + ld_stream(col + a + t)), acc);
    const double* __restrict__ vr = val + a + head;  // 32-byte aligned
    const int32_t* __restrict__ cr = col + a + head;
    const int32_t body = len - head;
    for (int32_t q = 4 * lane; q < body; q += 4 * W) {
      if (q + 3 < body) {
        double2 lo, hi;
        ld4_stream_first(vr + q, lo, hi);
        const int4 c = ld_stream4(reinterpret_cast<const int4*>(cr + q));
        acc = fma(lo.x, ld_x(x + c.x), acc);
        acc = fma(lo.y, ld_x(x + c.y), acc);
        acc = fma(hi.x, ld_x(x + c.z), acc);
        acc = fma(hi.y, ld_x(x + c.w), acc);
      } else {
        for (int32_t t = q; t < body; ++t) acc = fma(ld_stream(vr + t), ld_x(x + ld_stream(cr + t)), acc);
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
      double2 v0, v1;
      ld4_stream_first(val + q, v0, v1);
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
template <int U>
__device__ __forceinline__ void ell_pair(int64_t i, int32_t k_begin, int32_t k_end, int64_t ld,
                                         const double* __restrict__ val,
                                         const int32_t* __restrict__ col,
                                         const double* __restrict__ x, double& a0, double& a1) {
  a0 = 0.0;
  a1 = 0.0;
  const double2* vp = reinterpret_cast<const double2*>(val + i);
  const int2* cp = reinterpret_cast<const int2*>(col + i);
  const int64_t step = ld >> 1;  // in double2 / int2 units
  auto lv = [&](int64_t off) { return ld_stream2(vp + off); };
  auto lc = [&](int64_t off) { return ld_stream2(cp + off); };
  auto lx = [&](int32_t c) { return ld_x(x + c); };
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

template <int U, typename Out = PlainOut>
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
    ell_pair<U>(i, k_begin, k_end, ld, val, col, x, a0, a1);
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
      ell_pair<U>(i, k_begin, k_end, ld, val, col, x, a0, a1);
      y.put(i, a0);
      if (i + 1 < n) y.put(i + 1, a1);
    }
    y.done();
  }
}

// Banded matrices (SM-local regions): ONE 1024-thread CTA per SM (grid =
// kSMs; the block scheduler places them breadth-first, one per SM), each CTA
// sweeping one contiguous region of row pairs.  A band-major ELL thread walks
// its rows band by band, so at any moment an SM's threads gather band k of a
// few thousand consecutive rows: for columns scattered inside a band window
// of x (config 5) those gathers stay inside a slice of x that L1 holds,
// instead of the interleaved grid's 8 CTAs per SM each pulling a different
// window through L2 (config 5 D = 0: L1 sector hit rate 14 % -> 51 %, L2
// requests 58.7 M -> 25.8 M).  Same per-row band order as k_spmv_ell_cm, so
// the results are bitwise equal.  (Four rows per thread with 256-bit value
// loads measured no faster; profiles/r02_ell_banded.txt.)
template <int U>
__global__ void __launch_bounds__(1024, 1) k_spmv_ell_cm_local(int64_t n, int32_t nz, int64_t ld,
                                                               const double* __restrict__ val,
                                                               const int32_t* __restrict__ col,
                                                               const double* __restrict__ x,
                                                               double* __restrict__ y) {
  const int64_t pairs = (n + 1) / 2;
  const int64_t per = ((pairs + gridDim.x - 1) / gridDim.x + blockDim.x - 1) / blockDim.x *
                      blockDim.x;
  const int64_t g_end = min(pairs, static_cast<int64_t>(blockIdx.x + 1) * per);
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * per + threadIdx.x; g < g_end;
       g += blockDim.x) {
    const int64_t i = 2 * g;
    double a0, a1;
    ell_pair<U>(i, 0, nz, ld, val, col, x, a0, a1);
    y[i] = a0;
    if (i + 1 < n) y[i + 1] = a1;
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

int g_coo_variant = 1;  // 1: 4 entries per lane (k_spmv_coo_row4), 0: scalar
int g_seg_chunk = 0;  // entries per warp of the segmented CRS plan (0: SPMVTK_SEG_CHUNK)
int g_coo_chunk = 2048;  // entries per warp of k_spmv_coo_row4 (multiple of 128)
bool g_coo_chunk_auto = true;  // wave-aware choice between 2048 and 1024
int64_t g_coo_cap = 0;          // resident warps of k_spmv_coo_row4 (occupancy API)
void coo_row4_capacity() {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv_coo_row4, 256, 0);
  g_coo_cap = static_cast<int64_t>(kSMs) * std::max(per_sm, 1) * 8;
}
int g_rm_variant = -1;  // row-major ELL variant override (tuning)
int g_crs_variant = -1;  // tuning override (spmvtk_k_tune), -1 = heuristic
int g_ell_splits = 0;    // ell-outer band chunks forced (0 = by occupancy)

// The sub-warp CRS kernels (row-major ELL runs the same code on fixed-stride
// rows).  Variants: 12 = k_spmv_vec<4,2> (scalar loads), 16/17/18 =
// k_spmv_vec2 with 8/16/4 lanes per row (128-bit entry pairs), 21/22 =
// k_spmv_vec4 with 4/8 lanes (256-bit evict-first value quads; 2 and 16
// lanes measured slower everywhere, r02_tune_spmv_quads.txt, and removed).
// Measured on B200 (profiles/r01_tune_crs*.txt, r02_tune_spmv_quads.txt):
// few lanes per row (more rows in flight) win unless rows are long; pair
// loads from ~6 entries per row up; quads with 8 lanes for rows of ~32
// (config 5 at D = 0: 286 -> 269 us) and for row-major ELL with nz % 4 == 0
// (config 2, nz = 24: 91 -> 83 us).
template <typename Rows, typename Out>
void dispatch_vec(double mean, int64_t max_row, int64_t n, Rows rows, const int32_t* col,
                  const double* val, const double* x, Out y, int64_t long_limit,
                  int32_t* long_rows, cudaStream_t s) {
  int v = g_crs_variant;
  if (v < 0 || v == 20) {
    if (static_cast<double>(max_row) > 8.0 * mean + 8.0) v = 16;  // skewed: W=8 pairs
    else if (mean <= 6.0) v = 12;                               // W=4 scalar
    else if (mean <= 30.0) v = 18;                              // W=4 pairs
    else if (mean <= 64.0) v = 22;                              // W=8 quads
    else v = 17;                                                // W=16 pairs
    if constexpr (!std::is_same_v<Rows, CrsRows>) {
      // row-major ELL: rows of exactly nz slots; when nz % 4 == 0 every row
      // starts on a quad, so the quad kernel has no peeled entries
      if (max_row % 4 == 0 && max_row >= 12 && max_row <= 64) v = max_row <= 16 ? 21 : 22;
      if (g_rm_variant >= 0) v = g_rm_variant;
    }
  }
  const bool quads = (reinterpret_cast<uintptr_t>(val) & 31) == 0 &&
                     (reinterpret_cast<uintptr_t>(col) & 15) == 0;
  if (!quads && (v == 21 || v == 22)) v = 18;
  switch (v) {
    case 21:
      k_spmv_vec4<4, Rows, Out><<<grid_for(n * 4, 256, 8), 256, 0, s>>>(
          n, rows, col, val, x, y, long_limit, long_rows);
      break;
    case 22:
      k_spmv_vec4<8, Rows, Out><<<grid_for(n * 8, 256, 8), 256, 0, s>>>(
          n, rows, col, val, x, y, long_limit, long_rows);
      break;
    case 12:
      k_spmv_vec<4, 2, Rows, Out><<<grid_for(n * 4, 256, 8), 256, 0, s>>>(
          n, rows, col, val, x, y, long_limit, long_rows);
      break;
    case 17:
      k_spmv_vec2<16, 1, Rows, Out><<<grid_for(n * 16, 256, 8), 256, 0, s>>>(
          n, rows, col, val, x, y, long_limit, long_rows);
      break;
    case 18:
      k_spmv_vec2<4, 1, Rows, Out><<<grid_for(n * 4, 256, 8), 256, 0, s>>>(
          n, rows, col, val, x, y, long_limit, long_rows);
      break;
    default:
      k_spmv_vec2<8, 1, Rows, Out><<<grid_for(n * 8, 256, 8), 256, 0, s>>>(
          n, rows, col, val, x, y, long_limit, long_rows);
      break;
  }
  count_launches(1);
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
  if (use_long) {
    k_spmv_crs_long<<<kSMs * 4, 256, 0, s>>>(irp, icol, val, x, PlainOut{y}, long_rows);
    count_launches(1);
  }
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
  if (push == nullptr || push->ndst < 1 || push->ndst > SPMVTK_MAX_PEERS || push->local < 0 ||
      push->local >= push->ndst)
    return true;
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
    count_launches(1);
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
                    (reinterpret_cast<uintptr_t>(val) & 31) == 0;  // 256-bit value loads
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
  count_launches(1);
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
  if (nnz > 0) {
    k_spmv_coo_col<<<grid_for((nnz + 3) / 4, 256, 8), 256, 0, s>>>(nnz, row, col, val, x, y);
    count_launches(1);
  }
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
  const int64_t pairs = (n + 1) / 2;
  const unsigned blocks = static_cast<unsigned>((pairs + 255) / 256);
  k_spmv_ell_cm<4><<<blocks, 256, 0, s>>>(n, 0, nz, ld, val, col, x, PlainOut{y});
  count_launches(1);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_spmv_ell_cm_banded(int64_t n, int32_t nz, int64_t ld, const double* val,
                                const int32_t* col, const double* x, double* y, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) SPMVTK_LAUNCH_RETURN();
  if (nz == 0) {
    cudaMemsetAsync(y, 0, static_cast<size_t>(n) * sizeof(double), s);
    SPMVTK_LAUNCH_RETURN();
  }
  // 1024 threads x 64 registers: one CTA per SM, so the kSMs CTAs land on
  // distinct SMs.  Two bands in flight per thread (a tighter band front
  // across the SM's threads) measured 2-7 % faster than four; four rows per
  // thread with 256-bit loads no faster (profiles/r02_ell_banded.txt)
  k_spmv_ell_cm_local<2><<<kSMs, 1024, 0, s>>>(n, nz, ld, val, col, x, y);
  count_launches(1);
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
  k_spmv_ell_cm<4, PushOut><<<std::min<unsigned>(blocks, kSMs * 8), 256, 0, s>>>(
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
  count_launches(2);
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

int32_t spmvtk_k_seg_chunk(void) { return g_seg_chunk > 0 ? g_seg_chunk : SPMVTK_SEG_CHUNK; }

int spmvtk_k_crs_use_seg(double mean_row, int64_t max_row) {
  if (g_crs_variant >= 0) return g_crs_variant == 20 ? 1 : 0;
  // row-skewed matrices (power-law rows, config 4): the entry-balanced kernel
  // (366 vs 436 us on config 4); otherwise the sub-warp kernels win (config 2
  // 93 vs 95, config 3 135 vs 230, config 5 269 (quads) vs 303 us;
  // profiles/r02_tune_spmv_seg.txt, r02_tune_spmv_quads.txt)
  return (static_cast<double>(max_row) > 8.0 * mean_row + 8.0 && mean_row >= 4.0) ? 1 : 0;
}

int spmvtk_k_ell_splits_forced(void) { return g_ell_splits; }
int spmvtk_k_ell_banded_forced(void) { return g_ell_banded; }

int64_t spmvtk_k_crs_long_limit(double mean_row) {
  // rows this much longer than average would serialise one sub-warp: they go
  // to the block-per-row pass (power-law rows, BASELINE config 4)
  const int64_t m = static_cast<int64_t>(mean_row + 0.999);
  return std::max<int64_t>(256, std::min<int64_t>(4096, 32 * m));
}

int spmvtk_k_tune(const char* key, int value) {
  if (key && std::string(key) == "ell_banded") {  // SM-local ELL: -1 auto, 0 never, 1 always
    g_ell_banded = value < 0 ? -1 : value > 0 ? 1 : 0;
    return 0;
  }
  if (key && std::string(key) == "crs_variant") {
    g_crs_variant = value;
    return 0;
  }
  if (key && std::string(key) == "coo_variant") {
    g_coo_variant = value;
    return 0;
  }
  if (key && std::string(key) == "coo_chunk") {  // <= 0: automatic
    g_coo_chunk_auto = value <= 0;
    g_coo_chunk = value >= 128 ? (value / 128) * 128 : 2048;
    return 0;
  }
  if (key && std::string(key) == "ell_splits") {  // force ell-outer's band chunks (testing)
    g_ell_splits = value > 0 ? value : 0;
    return 0;
  }
  if (key && std::string(key) == "seg_chunk") {
    g_seg_chunk = value > 0 ? (value / 128) * 128 : 0;
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
  spmvtk_dev::preload_seg();
  spmvtk_dev::preload_ccs();
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_spmv_crs_long<PlainOut>);
  cudaFuncGetAttributes(&a, k_spmv_crs_long<PushOut>);
  cudaFuncGetAttributes(&a, k_spmv_ell_cm<4, PushOut>);
  cudaFuncGetAttributes(&a, k_spmv_ell_cm<4>);
  cudaFuncGetAttributes(&a, k_spmv_ell_cm_local<2>);
  cudaFuncGetAttributes(&a, k_spmv_ell_cm_part<4>);
  cudaFuncGetAttributes(&a, k_reduce_partials);
  cudaFuncGetAttributes(&a, k_spmv_coo_row);
  cudaFuncGetAttributes(&a, k_spmv_coo_row4);
  coo_row4_capacity();
  cudaFuncGetAttributes(&a, k_spmv_coo_col);
#define PRELOAD_VEC(ROWS, OUT)                                 \
  cudaFuncGetAttributes(&a, k_spmv_vec<4, 2, ROWS, OUT>);      \
  cudaFuncGetAttributes(&a, k_spmv_vec2<4, 1, ROWS, OUT>);     \
  cudaFuncGetAttributes(&a, k_spmv_vec2<8, 1, ROWS, OUT>);     \
  cudaFuncGetAttributes(&a, k_spmv_vec2<16, 1, ROWS, OUT>);
  PRELOAD_VEC(CrsRows, PlainOut)
  PRELOAD_VEC(CrsRows, PushOut)
  PRELOAD_VEC(EllRowMajorRows, PlainOut)
#undef PRELOAD_VEC
  SPMVTK_LAUNCH_RETURN();
}

}  // extern "C"
