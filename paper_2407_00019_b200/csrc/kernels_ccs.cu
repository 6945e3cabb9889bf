// kernels_ccs.cu -- CRS -> CCS Phase I (convert.cpp:24-53) and CRS -> COO-col
// with Phase II fused (convert.cpp:55-70) on sm_100a: a stable two-level
// partition followed by a stable per-bucket counting sort.
//
// The reference scatters each CRS entry, in CRS order, to the next free
// slot of its column (convert.cpp:43-51), so rows come out ascending inside
// every column and entries of one (row, column) pair keep their CRS order.
// Every pass here is STABLE (records keep CRS order inside every run), so
// the last pass is a plain counting sort by column and reproduces the
// reference's arrays exactly -- duplicates included -- with no per-column
// ranking by row.
//
// Columns are grouped into F fine buckets of 2^s2 columns (~2k entries
// each) and G = 2^g consecutive fine buckets form a coarse bucket (B1 of
// them, <= 256).  The CRS is cut into S entry-balanced row slices.
//   A  k_ccs_count    slice histograms of fine buckets (shared memory)
//                     -> cnt[s][f]; coarse counts cnt1[s][b] from them
//   -  k_ccs_offsets  exclusive scans: fine run (f, s) offsets (bucket-major:
//                     f, then slices in order) and coarse run (b, s) offsets
//                     in the same bucket-major layout
//   B  k_ccs_coarse   each slice streams its entries in 4096-entry tiles; a
//                     tile is ranked by coarse bucket in entry order (warp
//                     match_any + per-warp counts), staged in shared memory in
//                     bucket order and written run by run (coalesced 16-byte
//                     records {col, row, value})
//   C  k_ccs_refine   every coarse run (b, s) is split the same way into its
//                     fine runs (f, s)
//   D  k_ccs_sort     one CTA per fine bucket: its records (slices in order,
//                     so CRS order) are counted per (warp segment, column),
//                     placed in order by match_any ranks, staged in shared
//                     memory and written out coalesced; col_ptr from the
//                     column counts; COO-col also gets the column array
// Write streams stay short-lived in L2 (a tile's runs, a bucket's output),
// so DRAM sees whole lines.  Buckets larger than the staging capacity
// (dense columns) place their records straight into global memory.
#include <algorithm>
#include <climits>
#include <cstdint>

#include "common.cuh"
#include "spmvtk/spmvtk_kernels.h"

using namespace spmvtk_dev;

namespace {

constexpr int kPartThreads = 512;   // 16 warps x 128 entries per tile
constexpr int kPartWarps = kPartThreads / 32;
constexpr int kTile = kPartWarps * 128;  // entries per tile of the partition passes
constexpr int kMaxB = 256;          // buckets per partition level
constexpr int kMaxF = 32768;        // fine buckets (pass A shared histogram)
constexpr int kSortThreads = 256;   // pass D: 8 warps
constexpr int kSortCap = 4096;      // records a pass-D CTA stages
constexpr int kMaxCB = 512;         // columns per fine bucket

struct CcsPlan {
  int s2, g, F, B1, S;
};

// ---- slices: entry-balanced row ranges ------------------------------------
// slice_row[s] = first row whose start >= s*nnz/S (slice_row[S] = n)
__global__ void k_ccs_slices(const int32_t* __restrict__ irp, int32_t n, int64_t nnz, int32_t S,
                             int32_t* __restrict__ slice_row) {
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s > S) return;
  if (s == S) {
    slice_row[s] = n;
    return;
  }
  const int64_t target = nnz * s / S;
  int32_t lo = 0, hi = n;
  while (lo < hi) {
    const int32_t mid = lo + (hi - lo) / 2;
    if (__ldg(irp + mid) >= target) hi = mid;
    else lo = mid + 1;
  }
  slice_row[s] = lo;
}

// ---- A: fine histograms per slice ----------------------------------------
// cnt[f][s] (f-major: the per-bucket scan over slices is contiguous; the
// strided 4-byte writes merge in L2, the array is S*F*4 bytes)
__global__ void __launch_bounds__(512) k_ccs_count(const int32_t* __restrict__ irp,
                                                   const int32_t* __restrict__ icol,
                                                   const int32_t* __restrict__ slice_row,
                                                   CcsPlan p, int32_t* __restrict__ cnt,
                                                   int32_t* __restrict__ cnt1) {
  extern __shared__ int32_t hist[];
  const int s = blockIdx.x;
  for (int f = threadIdx.x; f < p.F; f += blockDim.x) hist[f] = 0;
  __syncthreads();
  const int32_t a = __ldg(irp + __ldg(slice_row + s)), b = __ldg(irp + __ldg(slice_row + s + 1));
  constexpr int U = 4;
  int32_t e = a + threadIdx.x;
  for (; e + (U - 1) * static_cast<int32_t>(blockDim.x) < b; e += U * blockDim.x) {
    int32_t c[U];
#pragma unroll
    for (int k = 0; k < U; ++k) c[k] = ld_stream(icol + e + k * blockDim.x);
#pragma unroll
    for (int k = 0; k < U; ++k) atomicAdd(hist + (c[k] >> p.s2), 1);
  }
  for (; e < b; e += blockDim.x) atomicAdd(hist + (ld_stream(icol + e) >> p.s2), 1);
  __syncthreads();
  for (int f = threadIdx.x; f < p.F; f += blockDim.x)
    cnt[static_cast<int64_t>(f) * p.S + s] = hist[f];
  const int G = 1 << p.g;
  for (int c = threadIdx.x; c < p.B1; c += blockDim.x) {
    int32_t t = 0;
    for (int k = 0; k < G && c * G + k < p.F; ++k) t += hist[c * G + k];
    cnt1[static_cast<int64_t>(c) * p.S + s] = t;
  }
}

// ---- offsets ----------------------------------------------------------------
// warp-wide exclusive scan of v (returns the exclusive prefix; *total = sum)
__device__ __forceinline__ int32_t warp_excl(int32_t v, int lane, int32_t* total) {
  int32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int32_t t = __shfl_up_sync(kFull, x, d);
    if (lane >= d) x += t;
  }
  *total = __shfl_sync(kFull, x, 31);
  return x - v;
}

// warp per fine bucket: exclusive over its slices (in place), total
__global__ void k_ccs_run_scan(int32_t* __restrict__ cnt, const CcsPlan p,
                               int32_t* __restrict__ tot) {
  const int lane = threadIdx.x & 31;
  const int32_t f = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (f >= p.F) return;
  int32_t* row = cnt + static_cast<int64_t>(f) * p.S;
  int32_t run = 0;
  for (int s0 = 0; s0 < p.S; s0 += 32) {
    const int s = s0 + lane;
    const int32_t v = s < p.S ? row[s] : 0;
    int32_t t;
    const int32_t x = warp_excl(v, lane, &t);
    if (s < p.S) row[s] = run + x;
    run += t;
  }
  if (lane == 0) tot[f] = run;
}

// one CTA: base[f] = exclusive scan of tot (base[F] = nnz)
__global__ void __launch_bounds__(1024) k_ccs_bucket_scan(const int32_t* __restrict__ tot,
                                                          int32_t F, int32_t* __restrict__ base) {
  __shared__ int32_t s_warp[32];
  __shared__ int32_t s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int32_t c0 = 0; c0 < F; c0 += 1024) {
    const int32_t i = c0 + threadIdx.x;
    const int32_t v = i < F ? tot[i] : 0;
    int32_t t;
    const int32_t x = warp_excl(v, lane, &t);
    if (lane == 0) s_warp[w] = t;
    __syncthreads();
    if (w == 0) {
      int32_t tt;
      s_warp[lane] = warp_excl(s_warp[lane], lane, &tt);
    }
    __syncthreads();
    const int32_t excl = s_carry + s_warp[w] + x;
    if (i < F) base[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) base[F] = s_carry;
}

// warps [0, F): fine offsets += bucket base; warps [F, F + B1): coarse run
// offsets (b, s) in the same bucket-major layout
__global__ void k_ccs_run_offsets(int32_t* __restrict__ cnt, int32_t* __restrict__ cnt1,
                                  const int32_t* __restrict__ base, const CcsPlan p) {
  const int lane = threadIdx.x & 31;
  const int32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w < p.F) {
    const int32_t bf = base[w];
    int32_t* row = cnt + static_cast<int64_t>(w) * p.S;
    for (int s = lane; s < p.S; s += 32) row[s] += bf;
  } else if (w < p.F + p.B1) {
    const int32_t b = w - p.F;
    int32_t* row = cnt1 + static_cast<int64_t>(b) * p.S;
    int32_t run = base[b << p.g];
    for (int s0 = 0; s0 < p.S; s0 += 32) {
      const int s = s0 + lane;
      const int32_t v = s < p.S ? row[s] : 0;
      int32_t t;
      const int32_t x = warp_excl(v, lane, &t);
      if (s < p.S) row[s] = run + x;
      run += t;
    }
  }
}

// ---- the stable tile partition shared by passes B and C -----------------
// The tile's records (registers of the thread owning them: warp w, round k,
// lane -> tile entry 128w + 32k + lane) have buckets in [0, nb).  On return
// every record has been written to out[cur[b] + rank], rank counting the
// tile's earlier records of bucket b, and cur[b] has advanced by the tile's
// count.  Ranks come from match_any in entry order plus per-warp counts, so
// the partition is stable.
struct PartSmem {
  int32_t wcnt[kPartWarps][kMaxB];  // per warp per bucket: count, then exclusive prefix
  int32_t tstart[kMaxB + 1];        // tile-local bucket starts
  int32_t cur[kMaxB];               // run cursors (global positions)
  int32_t wsum[kPartWarps];
  int4 stage[kTile];                // records in bucket order (aliases the row starts)
};

template <typename BucketOf>
__device__ __forceinline__ void tile_partition(PartSmem& sm, const int4 (&rec)[4],
                                               const int (&bkt)[4], const bool (&ok)[4], int nb,
                                               BucketOf bucket_of, int4* __restrict__ out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int i = threadIdx.x; i < kPartWarps * kMaxB; i += blockDim.x) (&sm.wcnt[0][0])[i] = 0;
  __syncthreads();
  int rank[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int key = ok[k] ? bkt[k] : -1;
    const unsigned m = __match_any_sync(kFull, key);
    const int leader = __ffs(m) - 1;
    int old = 0;
    if (key >= 0 && lane == leader) {
      old = sm.wcnt[w][key];
      sm.wcnt[w][key] = old + __popc(m);
    }
    old = __shfl_sync(kFull, old, leader);
    rank[k] = old + __popc(m & lt);
  }
  __syncthreads();
  // per bucket (thread b): exclusive over warps, tile count; then a block
  // scan of the counts over buckets (nb <= kMaxB <= blockDim)
  int32_t tcount = 0;
  if (threadIdx.x < nb) {
    const int b = threadIdx.x;
#pragma unroll
    for (int ww = 0; ww < kPartWarps; ++ww) {
      const int32_t t = sm.wcnt[ww][b];
      sm.wcnt[ww][b] = tcount;
      tcount += t;
    }
  }
  int32_t wt;
  const int32_t x = warp_excl(tcount, lane, &wt);
  if (lane == 0) sm.wsum[w] = wt;
  __syncthreads();
  if (w == 0) {
    int32_t tt;
    const int32_t v = lane < kPartWarps ? sm.wsum[lane] : 0;
    const int32_t y = warp_excl(v, lane, &tt);
    if (lane < kPartWarps) sm.wsum[lane] = y;
    if (lane == 0) sm.tstart[nb] = tt;
  }
  __syncthreads();
  if (threadIdx.x < nb) sm.tstart[threadIdx.x] = sm.wsum[w] + x;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (ok[k]) sm.stage[sm.tstart[bkt[k]] + sm.wcnt[w][bkt[k]] + rank[k]] = rec[k];
  __syncthreads();
  // bucket-ordered tile -> runs (consecutive threads, consecutive addresses)
  const int total = sm.tstart[nb];
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int4 r = sm.stage[i];
    const int bb = bucket_of(r);
    out[sm.cur[bb] + (i - sm.tstart[bb])] = r;
  }
  __syncthreads();
  if (threadIdx.x < nb) sm.cur[threadIdx.x] += sm.tstart[threadIdx.x + 1] - sm.tstart[threadIdx.x];
  __syncthreads();
}

__device__ __forceinline__ int4 make_rec(int32_t col, int32_t row, double v) {
  const long long bits = __double_as_longlong(v);
  return make_int4(col, row, static_cast<int32_t>(bits & 0xffffffffll),
                   static_cast<int32_t>(bits >> 32));
}

// ---- B: coarse partition of each slice -----------------------------------
// Row ids come from the expanded pointer array (one coalesced int32 per
// entry, written by k_expand_ptr just before), so a tile is three coalesced
// streams and the partition.
__global__ void __launch_bounds__(kPartThreads, 2) k_ccs_coarse(
    const int32_t* __restrict__ irp, const int32_t* __restrict__ icol,
    const double* __restrict__ val, const int32_t* __restrict__ rows,
    const int32_t* __restrict__ slice_row, CcsPlan p, const int32_t* __restrict__ off1,
    int4* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PartSmem& sm = *reinterpret_cast<PartSmem*>(smem_raw);
  const int s = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cshift = p.s2 + p.g;
  const int32_t a = __ldg(irp + __ldg(slice_row + s)), b = __ldg(irp + __ldg(slice_row + s + 1));
  for (int c = threadIdx.x; c < p.B1; c += blockDim.x)
    sm.cur[c] = off1[static_cast<int64_t>(c) * p.S + s];
  for (int32_t t0 = a; t0 < b; t0 += kTile) {
    int4 rec[4];
    int bkt[4];
    bool ok[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int32_t e = t0 + 128 * w + 32 * k + lane;
      ok[k] = e < b;
      if (ok[k]) {
        const int32_t c = ld_stream(icol + e);
        rec[k] = make_rec(c, ld_stream(rows + e), ld_stream(val + e));
        bkt[k] = c >> cshift;
      } else {
        bkt[k] = 0;
      }
    }
    tile_partition(sm, rec, bkt, ok, p.B1, [cshift](const int4& r) { return r.x >> cshift; },
                   out);
  }
}

// ---- C: coarse runs -> fine runs --------------------------------------------
__global__ void __launch_bounds__(kPartThreads, 2) k_ccs_refine(
    const int4* __restrict__ in, CcsPlan p, const int32_t* __restrict__ off1,
    const int32_t* __restrict__ off2, int64_t nnz, int4* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PartSmem& sm = *reinterpret_cast<PartSmem*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int G = 1 << p.g;
  const int64_t runs = static_cast<int64_t>(p.B1) * p.S;
  for (int64_t run = blockIdx.x; run < runs; run += gridDim.x) {
    const int c = static_cast<int>(run / p.S), s = static_cast<int>(run % p.S);
    const int32_t* orow = off1 + static_cast<int64_t>(c) * p.S;
    const int32_t a = orow[s];
    const int32_t b = s + 1 < p.S ? orow[s + 1] : (c + 1 < p.B1 ? orow[p.S] : static_cast<int32_t>(nnz));
    if (a >= b) continue;
    const int f0 = c * G, nb = min(G, p.F - f0);
    for (int k = threadIdx.x; k < nb; k += blockDim.x)
      sm.cur[k] = off2[static_cast<int64_t>(f0 + k) * p.S + s];
    __syncthreads();
    for (int32_t t0 = a; t0 < b; t0 += kTile) {
      int4 rec[4];
      int bkt[4];
      bool ok[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int32_t e = t0 + 128 * w + 32 * k + lane;
        ok[k] = e < b;
        if (ok[k]) {
          rec[k] = ld_stream4(in + e);
          bkt[k] = (rec[k].x >> p.s2) - f0;
        } else {
          bkt[k] = 0;
        }
      }
      tile_partition(sm, rec, bkt, ok, nb,
                     [s2 = p.s2, f0](const int4& r) { return (r.x >> s2) - f0; }, out);
    }
  }
}

// ---- D: per fine bucket, stable counting sort by column ------------------
struct SortSmem {
  int32_t tab[kSortThreads / 32][kMaxCB];  // per warp segment per column
  int32_t cstart[kMaxCB + 1];
  int32_t s_row[kSortCap];
  double s_val[kSortCap];
};

__global__ void __launch_bounds__(kSortThreads, 3) k_ccs_sort(
    const int4* __restrict__ in, const int32_t* __restrict__ base, CcsPlan p, int32_t n,
    int32_t* __restrict__ col_ptr, int32_t* __restrict__ row_idx, double* __restrict__ out_val,
    int32_t* __restrict__ out_col) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem& sm = *reinterpret_cast<SortSmem*>(smem_raw);
  constexpr int W = kSortThreads / 32;
  const int f = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int CB = 1 << p.s2, cmask = CB - 1;
  const int32_t a = base[f], b = base[f + 1];
  const int32_t tot = b - a;
  for (int i = threadIdx.x; i < W * CB; i += blockDim.x) sm.tab[i / CB][i % CB] = 0;
  __syncthreads();
  // warp segments of the bucket, in order
  const int32_t L = (tot + W - 1) / W;
  const int32_t sa = a + min(tot, w * L), sb = a + min(tot, (w + 1) * L);
  {
    int32_t e = sa + lane;
    for (; e + 96 < sb; e += 128) {
      int32_t c[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) c[k] = __ldg(&in[e + 32 * k].x);
#pragma unroll
      for (int k = 0; k < 4; ++k) atomicAdd(&sm.tab[w][c[k] & cmask], 1);
    }
    for (; e < sb; e += 32) atomicAdd(&sm.tab[w][__ldg(&in[e].x) & cmask], 1);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < CB; c += blockDim.x) {
    int32_t acc = 0;
#pragma unroll 4
    for (int ww = 0; ww < W; ++ww) {
      const int32_t t = sm.tab[ww][c];
      sm.tab[ww][c] = acc;
      acc += t;
    }
    sm.cstart[c] = acc;
  }
  __syncthreads();
  if (w == 0) {  // exclusive scan of the column counts (CB <= 512)
    int32_t carry = 0;
    for (int c0 = 0; c0 < CB; c0 += 32) {
      const int c = c0 + lane;
      const int32_t v = c < CB ? sm.cstart[c] : 0;
      int32_t x = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int32_t t = __shfl_up_sync(kFull, x, d);
        if (lane >= d) x += t;
      }
      if (c < CB) sm.cstart[c] = carry + x - v;
      carry += __shfl_sync(kFull, x, 31);
    }
  }
  __syncthreads();
  const int64_t c0 = static_cast<int64_t>(f) << p.s2;
  for (int c = threadIdx.x; c < CB; c += blockDim.x)
    if (c0 + c < n) col_ptr[c0 + c] = a + sm.cstart[c];
  if (f == p.F - 1 && threadIdx.x == 0) col_ptr[n] = b;
  const bool staged = tot <= kSortCap;
  // place every record at cstart[col] + (its rank among the bucket's earlier
  // records of that column): warp segments in order, lanes in order
  int4 nxt = sa + lane < sb ? __ldg(in + sa + lane) : make_int4(0, 0, 0, 0);
  for (int32_t e0 = sa; e0 < sb; e0 += 32) {
    const int32_t e = e0 + lane;
    const int4 r = nxt;
    if (e + 32 < sb) nxt = __ldg(in + e + 32);
    const int key = e < sb ? (r.x & cmask) : -1;
    const unsigned m = __match_any_sync(kFull, key);
    const int leader = __ffs(m) - 1;
    int old = 0;
    if (key >= 0 && lane == leader) {
      old = sm.tab[w][key];
      sm.tab[w][key] = old + __popc(m);
    }
    old = __shfl_sync(kFull, old, leader);
    if (key >= 0) {
      const int32_t pos = sm.cstart[key] + old + __popc(m & lt);
      const double v = __longlong_as_double((static_cast<long long>(r.w) << 32) |
                                            static_cast<uint32_t>(r.z));
      if (staged) {
        sm.s_row[pos] = r.y;
        sm.s_val[pos] = v;
      } else {
        row_idx[a + pos] = r.y;
        out_val[a + pos] = v;
        if (out_col) out_col[a + pos] = r.x;
      }
    }
  }
  if (!staged) return;
  __syncthreads();
  for (int32_t i = threadIdx.x; i < tot; i += blockDim.x) {
    row_idx[a + i] = sm.s_row[i];
    out_val[a + i] = sm.s_val[i];
    if (out_col) {  // the column of slot i: the last c with cstart[c] <= i
      int lo = 0, hi = CB - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sm.cstart[mid] <= i) lo = mid;
        else hi = mid - 1;
      }
      out_col[a + i] = static_cast<int32_t>(c0 + lo);
    }
  }
}

CcsPlan make_plan(int64_t n, int64_t nnz) {
  CcsPlan p{};
  // fine buckets of ~2k entries: 2^s2 columns, s2 <= log2(kMaxCB)
  const double per_col = nnz > 0 && n > 0 ? static_cast<double>(nnz) / static_cast<double>(n) : 1.0;
  int s2 = 0;
  while (s2 < 9 && (static_cast<double>(int64_t(1) << (s2 + 1)) * per_col) <= 2048.0) ++s2;
  while ((((n + (int64_t(1) << s2) - 1) >> s2)) > kMaxF && s2 < 9) ++s2;
  p.s2 = s2;
  p.F = static_cast<int>(std::max<int64_t>(1, (n + (int64_t(1) << s2) - 1) >> s2));
  p.S = static_cast<int>(std::min<int64_t>(2 * kSMs, std::max<int64_t>(1, nnz / kTile)));
  // coarse buckets: runs (b, s) of ~2k records (so the refine pass works on
  // long runs), at most kMaxB coarse buckets and kMaxB fine ones per coarse
  const int64_t want_b1 = std::max<int64_t>(1, nnz / (static_cast<int64_t>(p.S) * 2048));
  int g = 0;
  while (g < 15 && (((p.F + (1 << g) - 1) >> g) > kMaxB ||
                    ((p.F + (1 << g) - 1) >> g) > want_b1))
    ++g;
  while ((1 << g) > kMaxB) --g;
  p.g = g;
  p.B1 = (p.F + (1 << g) - 1) >> g;
  return p;
}

struct CcsScratch {
  int4* rec;
  int4* rec2;
  int32_t* cnt;    // [S][F]
  int32_t* cnt1;   // [S][B1]
  int32_t* tot;    // [F]
  int32_t* base;   // [F + 1]
  int32_t* slice;  // [S + 1]
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

CcsScratch carve(void* scratch, const CcsPlan& p, int64_t nnz) {
  char* q = static_cast<char*>(scratch);
  CcsScratch c{};
  auto take = [&](size_t bytes) {
    char* r = q;
    q += align256(bytes);
    return r;
  };
  c.rec = reinterpret_cast<int4*>(take(static_cast<size_t>(std::max<int64_t>(nnz, 1)) * 16));
  c.rec2 = reinterpret_cast<int4*>(take(static_cast<size_t>(std::max<int64_t>(nnz, 1)) * 16));
  c.cnt = reinterpret_cast<int32_t*>(take(static_cast<size_t>(p.S) * p.F * 4));
  c.cnt1 = reinterpret_cast<int32_t*>(take(static_cast<size_t>(p.S) * p.B1 * 4));
  c.tot = reinterpret_cast<int32_t*>(take(static_cast<size_t>(p.F) * 4));
  c.base = reinterpret_cast<int32_t*>(take(static_cast<size_t>(p.F + 1) * 4));
  c.slice = reinterpret_cast<int32_t*>(take(static_cast<size_t>(p.S + 1) * 4));
  return c;
}

size_t scratch_bytes(int64_t n, int64_t nnz) {
  const CcsPlan p = make_plan(n, nnz);
  return 2 * align256(static_cast<size_t>(std::max<int64_t>(nnz, 1)) * 16) +
         align256(static_cast<size_t>(p.S) * p.F * 4) + align256(static_cast<size_t>(p.S) * p.B1 * 4) +
         align256(static_cast<size_t>(p.F) * 4) + align256(static_cast<size_t>(p.F + 1) * 4) +
         align256(static_cast<size_t>(p.S + 1) * 4);
}

int crs_to_ccs_impl(int64_t n, int64_t nnz, const int32_t* irp, const int32_t* icol,
                    const double* val, int32_t* col_ptr, int32_t* row_idx, double* out_val,
                    int32_t* out_col, void* scratch, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) {
    cudaMemsetAsync(col_ptr, 0, sizeof(int32_t), s);
    SPMVTK_LAUNCH_RETURN();
  }
  const CcsPlan p = make_plan(n, nnz);
  if (nnz == 0) {
    cudaMemsetAsync(col_ptr, 0, static_cast<size_t>(n + 1) * sizeof(int32_t), s);
    SPMVTK_LAUNCH_RETURN();
  }
  static const bool attrs = [] {  // thread-safe one-time setup
    cudaFuncSetAttribute(k_ccs_count, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxF * 4);
    cudaFuncSetAttribute(k_ccs_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(PartSmem)));
    cudaFuncSetAttribute(k_ccs_refine, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(PartSmem)));
    cudaFuncSetAttribute(k_ccs_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(SortSmem)));
    return true;
  }();
  (void)attrs;
  const CcsScratch c = carve(scratch, p, nnz);
  const int32_t ni = static_cast<int32_t>(n);
  k_ccs_slices<<<(p.S + 1 + 127) / 128, 128, 0, s>>>(irp, ni, nnz, p.S, c.slice);
  k_ccs_count<<<p.S, 512, static_cast<size_t>(p.F) * 4, s>>>(irp, icol, c.slice, p, c.cnt,
                                                             c.cnt1);
  k_ccs_run_scan<<<(p.F + 7) / 8, 256, 0, s>>>(c.cnt, p, c.tot);
  k_ccs_bucket_scan<<<1, 1024, 0, s>>>(c.tot, p.F, c.base);
  k_ccs_run_offsets<<<(p.F + p.B1 + 7) / 8, 256, 0, s>>>(c.cnt, c.cnt1, c.base, p);
  // row ids of every entry, into the (not yet used) refine output buffer
  int32_t* rows = reinterpret_cast<int32_t*>(c.rec2);
  int rc = spmvtk_k_expand_ptr(irp, n, nnz, rows, stream);
  if (rc) return rc;
  k_ccs_coarse<<<p.S, kPartThreads, sizeof(PartSmem), s>>>(irp, icol, val, rows, c.slice, p,
                                                           c.cnt1, c.rec);
  const int64_t runs = static_cast<int64_t>(p.B1) * p.S;
  k_ccs_refine<<<static_cast<unsigned>(std::min<int64_t>(runs, int64_t(kSMs) * 2)), kPartThreads,
                 sizeof(PartSmem), s>>>(c.rec, p, c.cnt1, c.cnt, nnz, c.rec2);
  k_ccs_sort<<<p.F, kSortThreads, sizeof(SortSmem), s>>>(c.rec2, c.base, p, ni, col_ptr, row_idx,
                                                         out_val, out_col);
  SPMVTK_LAUNCH_RETURN();
}

}  // namespace

namespace spmvtk_dev {
int g_ccs_force_stable = 0;
void preload_ccs() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_ccs_slices);
  cudaFuncGetAttributes(&a, k_ccs_count);
  cudaFuncGetAttributes(&a, k_ccs_run_scan);
  cudaFuncGetAttributes(&a, k_ccs_bucket_scan);
  cudaFuncGetAttributes(&a, k_ccs_run_offsets);
  cudaFuncGetAttributes(&a, k_ccs_coarse);
  cudaFuncGetAttributes(&a, k_ccs_refine);
  cudaFuncGetAttributes(&a, k_ccs_sort);
}
}  // namespace spmvtk_dev

extern "C" {

int spmvtk_k_ccs_force_stable(void) { return spmvtk_dev::g_ccs_force_stable; }

size_t spmvtk_k_ccs_scratch_bytes(int64_t n, int64_t nnz) {
  return std::max(scratch_bytes(n, nnz), legacy_ccs_scratch_bytes(n, nnz));
}

int spmvtk_k_crs_to_ccs(int64_t n, int64_t nnz, const int32_t* irp, const int32_t* icol,
                        const double* val, int32_t* col_ptr, int32_t* row_idx,
                        double* out_val, void* scratch, void* stream) {
  return legacy_crs_to_ccs(n, nnz, irp, icol, val, col_ptr, row_idx, out_val, scratch, stream);
}

int spmvtk_k_crs_to_coo_col(int64_t n, int64_t nnz, const int32_t* irp, const int32_t* icol,
                            const double* val, int32_t* col_ptr, int32_t* row_idx,
                            int32_t* col_idx, double* out_val, void* scratch, void* stream) {
  return legacy_crs_to_coo_col(n, nnz, irp, icol, val, col_ptr, row_idx, col_idx, out_val,
                               scratch, stream);
}

int spmvtk_k_crs_to_ccs_stable(int64_t n, int64_t nnz, const int32_t* irp, const int32_t* icol,
                               const double* val, int32_t* col_ptr, int32_t* row_idx,
                               double* out_val, void* scratch, void* stream) {
  return crs_to_ccs_impl(n, nnz, irp, icol, val, col_ptr, row_idx, out_val, nullptr, scratch,
                         stream);
}

int spmvtk_k_crs_to_coo_col_stable(int64_t n, int64_t nnz, const int32_t* irp,
                                   const int32_t* icol, const double* val, int32_t* col_ptr,
                                   int32_t* row_idx, int32_t* col_idx, double* out_val,
                                   void* scratch, void* stream) {
  return crs_to_ccs_impl(n, nnz, irp, icol, val, col_ptr, row_idx, out_val, col_idx, scratch,
                         stream);
}

}  // extern "C"
