// kernels_spmv_seg.cu -- entry-balanced ("segmented") CRS SpMV on sm_100a
// (spmv_crs, spmv.cpp:64-75), the kernel for row-skewed matrices.
//
// Why: on matrices with scattered columns every x gather is its own L2
// request, and the SM's L1->L2 request path (~1 request per SM-cycle,
// profiles/r02_microbench_gather_tma.txt) is the roofline.  Two things keep a
// kernel below it: (1) matrix-stream requests that carry less than a full
// 128-byte line (a sub-warp per row reads each row's unaligned run: ~3x the
// line count, profiles/r02_ncu_cfg4_spmv_vec2.txt), and (2) too few gathers in
// flight while a warp waits on its next column indices (long-scoreboard
// stalls).  Here every warp owns a contiguous, row-aligned run of ~C entries
// (a per-handle plan: warp w owns the rows whose first entry lies in
// [wC, (w+1)C)), lanes take 4 consecutive entries each (one int4 + two
// double2 loads: a warp's 128 entries are 12 full lines), the loads of the
// NEXT 128 entries are issued before the current ones' gathers are consumed,
// and rows are resolved against a window of 32 row ends held one per lane
// (CRS: no row array is read).  Row sums come out of a segmented shuffle
// scan, so the result is deterministic (the order of additions is fixed by
// the plan) and needs no atomics.
#include <algorithm>
#include <climits>
#include <cstdint>
#include <string>

#include "common.cuh"
#include "spmv_out.cuh"
#include "spmvtk/spmvtk.h"
#include "spmvtk/spmvtk_kernels.h"

using namespace spmvtk_dev;

namespace {
constexpr int kSegWarps = 8;  // warps per CTA

__device__ __forceinline__ bool real_row(int32_t r) { return r >= 0 && r != INT_MAX; }

// Entries of one lane: K (4 or 8) consecutive positions q..q+K-1 (q a
// multiple of K), masked to [a, b).  Out-of-range slots read nothing.  Full
// groups use 256-bit L2-evict-first loads where the width allows.
template <int K>
struct Group {
  int32_t c[K];
  double v[K];
};

__device__ __forceinline__ void ld8_cols_first(const int32_t* p, int32_t (&c)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]), "=r"(c[4]), "=r"(c[5]),
                 "=r"(c[6]), "=r"(c[7])
               : "l"(p));
}

template <int K>
__device__ __forceinline__ void load_group(const int32_t* __restrict__ col,
                                           const double* __restrict__ val, int32_t q, int32_t a,
                                           int32_t b, bool wide, Group<K>& o) {
  if (wide && q >= a && q + K - 1 < b) {
    if constexpr (K == 8) {
      ld8_cols_first(col + q, o.c);
    } else {
      const int4 c4 = ld_stream4(reinterpret_cast<const int4*>(col + q));
      o.c[0] = c4.x; o.c[1] = c4.y; o.c[2] = c4.z; o.c[3] = c4.w;
    }
#pragma unroll
    for (int k = 0; k < K; k += 4) {
      double2 lo, hi;
      ld4_stream_first(val + q + k, lo, hi);
      o.v[k] = lo.x; o.v[k + 1] = lo.y; o.v[k + 2] = hi.x; o.v[k + 3] = hi.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool in = q + k >= a && q + k < b;
      o.c[k] = in ? ld_stream(col + q + k) : 0;
      o.v[k] = in ? ld_stream(val + q + k) : 0.0;
    }
  }
}

template <int K>
__device__ __forceinline__ void products(const Group<K>& g, int32_t q, int32_t a, int32_t b,
                                         const double* __restrict__ x, double (&p)[K]) {
  // gathers only for real entries; they are independent
#pragma unroll
  for (int k = 0; k < K; ++k) p[k] = (q + k >= a && q + k < b) ? g.v[k] * ld_x(x + g.c[k]) : 0.0;
}

// One group of 32*K entries (K per lane, r[k] = row or -1 before / INT_MAX
// after the warp's range) reduced into row sums: lane-local runs, then a
// segmented inclusive scan of the lanes' tail runs; a row still open at the
// end of the group is carried to the next.  Empty rows are written from the
// row window (load_window), not here.
template <int K, typename Out>
__device__ __forceinline__ void seg_reduce(const int32_t (&r)[K], const double (&p)[K], int lane,
                                           int32_t& carry_row, double& carry_val, const Out& y) {
  double first_sum = p[0], run = p[0];
  bool in_first = true;
#pragma unroll
  for (int k = 1; k < K; ++k) {
    if (r[k] != r[k - 1]) {
      if (!in_first && real_row(r[k - 1])) y.put_local(r[k - 1], run);
      in_first = false;
      run = p[k];
    } else {
      run += p[k];
      if (in_first) first_sum += p[k];
    }
  }
  const int32_t head = r[0], tail = r[K - 1];
  const bool single = head == tail;
  const int32_t prev_tail = __shfl_up_sync(kFull, tail, 1);
  bool flag = !single || lane == 0 || head != prev_tail;
  double s = run;
  if (lane == 0 && single && head == carry_row) s += carry_val;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double ts = __shfl_up_sync(kFull, s, d);
    const bool tf = __shfl_up_sync(kFull, flag, d);
    if (lane >= d && !flag) s += ts;
    if (lane >= d) flag = flag || tf;
  }
  const double s_prev = __shfl_up_sync(kFull, s, 1);
  if (!single && head >= 0) {  // head run completes inside this lane
    double tot = first_sum;
    if (lane > 0 && head == prev_tail) tot += s_prev;
    if (lane == 0 && head == carry_row) tot += carry_val;
    y.put_local(head, tot);
  }
  const int32_t head0 = __shfl_sync(kFull, head, 0);
  if (lane == 0 && carry_row >= 0 && head0 != carry_row) {  // carried row ended at the edge
    y.put_local(carry_row, carry_val);
  }
  const int32_t next_head = __shfl_down_sync(kFull, head, 1);
  if (lane < 31 && next_head != tail) {  // tail run completes at the lane boundary
    if (real_row(tail)) y.put_local(tail, s);
  }
  carry_row = __shfl_sync(kFull, tail, 31);
  carry_val = __shfl_sync(kFull, s, 31);
  if (!real_row(carry_row)) carry_row = -1;
}

// Row window: lane j holds E = end of row t+j (exclusive entry index), or
// INT_MAX past the window; rows of the window that are empty are zeroed when
// the window is loaded (every row of the warp's range passes through exactly
// one window position).
template <typename Out>
__device__ __forceinline__ void load_window(const int32_t* __restrict__ irp, int32_t t,
                                            int32_t r_end, int lane, int32_t& E, int32_t& nrw,
                                            int32_t& Elast, const Out& y) {
  nrw = min(32, r_end - t);
  E = lane < nrw ? __ldg(irp + t + lane + 1) : INT_MAX;
  const int32_t up = __shfl_up_sync(kFull, E, 1);
  const int32_t start = lane == 0 ? __ldg(irp + t) : up;
  if (lane < nrw && E == start) y.put_local(int64_t(t) + lane, 0.0);
  Elast = __shfl_sync(kFull, E, 31);
}

// number of window row ends <= e (0..32)
__device__ __forceinline__ int window_rank(int32_t E, int32_t Elast, int32_t e) {
  int lo = 0;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const int32_t v = __shfl_sync(kFull, E, lo + s - 1);
    if (v <= e) lo += s;
  }
  return Elast <= e ? 32 : lo;
}

// CRS.  plan[w] = first row whose start >= w*C (plan[nwarps] = n); warp
// w_base + w owns rows [plan[w], plan[w+1]) clipped to [row_lo, row_hi).
// (K = 8 entries per lane, 120 registers at 2 CTAs/SM, measured 14-30 %
// slower on configs 2-5: profiles/r02_tune_spmv_evict_first.txt)
template <int K, typename Out>
__global__ void __launch_bounds__(kSegWarps * 32, 4) k_spmv_crs_seg(const int32_t* __restrict__ irp,
                                                         const int32_t* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ x, Out y,
                                                         const int32_t* __restrict__ plan,
                                                         int32_t w_base, int32_t w_end,
                                                         int32_t row_lo, int32_t row_hi) {
  // wide loads need 32-byte aligned values and 16-byte aligned columns
  // (pool allocations are; arrays handed in through the lower ABI may not be)
  const bool wide = ((reinterpret_cast<uintptr_t>(val) & 31) | (reinterpret_cast<uintptr_t>(col) & 15)) == 0;
  y.begin();
  const int lane = threadIdx.x & 31;
  // one pass for a full grid; a capped grid (the pushed SpMV: one flag wait
  // and one counter arrival per resident CTA) strides over the tiles of
  // kSegWarps consecutive warps, whose rows are one contiguous range
  const int32_t tiles = (w_end - w_base + kSegWarps - 1) / kSegWarps;
  for (int32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int32_t t0 = w_base + tile * kSegWarps;
    const int32_t w = t0 + static_cast<int32_t>(threadIdx.x >> 5);
    if (w < w_end) {
    const int32_t R0 = max(__ldg(plan + w), row_lo), R1 = min(__ldg(plan + w + 1), row_hi);
    if (R0 < R1) {
      const int32_t a = __ldg(irp + R0), b = __ldg(irp + R1);
      int32_t t = R0, E, nrw, Elast;
      constexpr int G = 32 * K;  // entries per warp step
      int32_t g = a & ~(K - 1);
      Group<K> cur;
      load_group<K>(col, val, g + K * lane, a, b, wide, cur);
      load_window(irp, t, R1, lane, E, nrw, Elast, y);
      int32_t carry_row = -1;
      double carry_val = 0.0;
      for (; g < b; g += G) {
        Group<K> nxt;
        if (g + G < b) load_group<K>(col, val, g + G + K * lane, a, b, wide, nxt);
        const int32_t q = g + K * lane;
        double p[K];
        products<K>(cur, q, a, b, x, p);
        int32_t r[K];
        bool pend[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int32_t e = q + k;
          pend[k] = e >= a && e < b;
          r[k] = e < a ? -1 : INT_MAX;
        }
        while (true) {
          bool any = false;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const int o = window_rank(E, Elast, q + k);
            if (pend[k] && o < nrw) {
              r[k] = t + o;
              pend[k] = false;
            }
            any = any || pend[k];
          }
          if (!__any_sync(kFull, any)) break;
          t += 32;
          load_window(irp, t, R1, lane, E, nrw, Elast, y);
        }
        seg_reduce<K>(r, p, lane, carry_row, carry_val, y);
        cur = nxt;
      }
      if (lane == 0 && carry_row >= 0) y.put_local(carry_row, carry_val);
      // trailing rows of the range (empty) still pass through a window
      while (t + 32 < R1) {
        t += 32;
        load_window(irp, t, R1, lane, E, nrw, Elast, y);
      }
    }
    }
    y.tile(max(__ldg(plan + t0), row_lo), min(__ldg(plan + min(t0 + kSegWarps, w_end)), row_hi));
  }
  y.done();
}

__global__ void k_seg_plan(const int32_t* __restrict__ irp, int32_t n, int32_t chunk,
                           int32_t nwarps, int32_t* __restrict__ plan) {
  const int32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w > nwarps) return;
  if (w == nwarps) {
    plan[w] = n;
    return;
  }
  const int64_t target = static_cast<int64_t>(w) * chunk;
  int32_t lo = 0, hi = n;  // first r in [0, n] with irp[r] >= target
  while (lo < hi) {
    const int32_t mid = lo + (hi - lo) / 2;
    if (__ldg(irp + mid) >= target) hi = mid;
    else lo = mid + 1;
  }
  plan[w] = lo;
}



template <typename Out>
int launch_crs_seg(const int32_t* irp, const int32_t* icol, const double* val, const double* x,
                   Out y, const int32_t* plan, int32_t w_base, int32_t w_end, int32_t row_lo,
                   int32_t row_hi, int32_t nnz, cudaStream_t s) {
  const int32_t warps = w_end - w_base;
  if (warps <= 0) SPMVTK_LAUNCH_RETURN();
  unsigned blocks = static_cast<unsigned>((warps + kSegWarps - 1) / kSegWarps);
  (void)nnz;  // (the array length: bounds of stream prefetchers; unused here)
  if (y.synced()) blocks = std::min<unsigned>(blocks, kSMs * 4);
  k_spmv_crs_seg<4, Out><<<blocks, kSegWarps * 32, 0, s>>>(irp, icol, val, x, y, plan, w_base,
                                                            w_end, row_lo, row_hi);
  count_launches(1);
  SPMVTK_LAUNCH_RETURN();
}

}  // namespace

namespace spmvtk_dev {
void preload_seg() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_spmv_crs_seg<4, PlainOut>);
  cudaFuncGetAttributes(&a, k_spmv_crs_seg<4, PushOut>);
  cudaFuncGetAttributes(&a, k_seg_plan);
}
}  // namespace spmvtk_dev

extern "C" {

int32_t spmvtk_k_seg_plan_warps(int64_t nnz, int32_t chunk) {
  if (chunk <= 0) chunk = SPMVTK_SEG_CHUNK;
  return static_cast<int32_t>(std::max<int64_t>(1, (nnz + chunk - 1) / chunk));
}

int spmvtk_k_seg_plan(int64_t n, int64_t nnz, const int32_t* irp, int32_t chunk, int32_t* plan,
                      void* stream) {
  cudaStream_t s = as_stream(stream);
  if (chunk <= 0) chunk = SPMVTK_SEG_CHUNK;
  const int32_t nw = spmvtk_k_seg_plan_warps(nnz, chunk);
  k_seg_plan<<<(nw + 1 + 255) / 256, 256, 0, s>>>(irp, static_cast<int32_t>(n), chunk, nw, plan);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_spmv_crs_seg(const int32_t* irp, const int32_t* icol, const double* val,
                          const double* x, double* y, const int32_t* plan, int32_t w_base,
                          int32_t w_end, int64_t row_lo, int64_t row_hi, int64_t nnz,
                          void* stream) {
  return launch_crs_seg(irp, icol, val, x, PlainOut{y}, plan, w_base, w_end,
                        static_cast<int32_t>(row_lo), static_cast<int32_t>(row_hi),
                        static_cast<int32_t>(nnz), as_stream(stream));
}

int spmvtk_k_spmv_crs_seg_push(const int32_t* irp, const int32_t* icol, const double* val,
                               const double* x, const struct spmvtk_push* push,
                               const struct spmvtk_push_sync* sync, const int32_t* plan,
                               int32_t nwarps, int64_t n, int64_t nnz, void* stream) {
  if (push == nullptr || push->ndst < 1 || push->ndst > SPMVTK_MAX_PEERS || push->local < 0 ||
      push->local >= push->ndst)
    return static_cast<int>(cudaErrorInvalidValue);
  spmvtk_push_sync none{};
  PushOut out{*push, sync ? *sync : none};
  return launch_crs_seg(irp, icol, val, x, out, plan, 0, nwarps, 0, static_cast<int32_t>(n),
                        static_cast<int32_t>(nnz), as_stream(stream));
}

}  // extern "C"
