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
                                                     int32_t* __restrict__ row_idx,
                                                     double* __restrict__ out_val) {
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
      int32_t slot = atomicAdd(cursor + c, 1);
      row_idx[slot] = row;
      out_val[slot] = v;
    }
  }
}

// Columns of length <= 32: one warp per column, bitonic sort in registers on
// a packed key (row << 5 | source lane); values follow by shuffle.  Sorted
// columns (the common case) exit after one ballot.  Longer columns are queued
// for the block-level passes.
constexpr int kShortCol = 32;
constexpr int kMediumCol = 4096;

__global__ void __launch_bounds__(256) k_ccs_fix_short(const int32_t* __restrict__ col_ptr,
                                                       int64_t n, int32_t* row_idx,
                                                       double* vals, int32_t* queue,
                                                       int32_t* queue_len, bool packed_ok) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < n;
       j += warps) {
    const int32_t a = __ldg(col_ptr + j), b = __ldg(col_ptr + j + 1);
    const int32_t len = b - a;
    if (len <= 1) continue;
    if (len > kShortCol || !packed_ok) {
      if (lane == 0) queue[atomicAdd(queue_len, 1)] = static_cast<int32_t>(j);
      continue;
    }
    int32_t r = lane < len ? row_idx[a + lane] : INT_MAX;
    int32_t rn = __shfl_down_sync(kFull, r, 1);
    bool desc = (lane + 1 < len) && rn < r;
    if (!__any_sync(kFull, desc)) continue;
    double v = lane < len ? vals[a + lane] : 0.0;
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
        s_key[t] = row_idx[a + t];
        s_val[t] = vals[a + t];
      }
      __syncthreads();
      block_bitonic(s_key, s_val, len);
      for (int32_t t = threadIdx.x; t < len; t += blockDim.x) {
        row_idx[a + t] = s_key[t];
        vals[a + t] = s_val[t];
      }
    } else {
      // very long column: same network directly in global memory (L2)
      block_bitonic(row_idx + a, vals + a, len);
    }
    __syncthreads();
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

size_t spmvtk_k_ccs_scratch_bytes(int64_t n) {
  // count[n+1], cursor[n+1], queue[n], queue_len[1], scan tiles
  size_t ints = static_cast<size_t>(n + 1) * 2 + static_cast<size_t>(n) + 4;
  return ints * sizeof(int32_t) + spmvtk_k_scan_scratch_bytes(n + 1) + 256;
}

int spmvtk_k_crs_to_ccs(int64_t n, int64_t nnz, const int32_t* irp, const int32_t* icol,
                        const double* val, int32_t* col_ptr, int32_t* row_idx,
                        double* out_val, void* scratch, void* stream) {
  cudaStream_t s = as_stream(stream);
  int32_t* count = static_cast<int32_t*>(scratch);
  int32_t* cursor = count + (n + 1);
  int32_t* queue = cursor + (n + 1);
  int32_t* queue_len = queue + n;
  // keep the scan scratch 16-byte aligned
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
                                                             row_idx, out_val);
  k_ccs_fix_short<<<grid_for(n * 32, 256, 16), 256, 0, s>>>(col_ptr, n, row_idx, out_val,
                                                            queue, queue_len,
                                                            n < (int64_t(1) << 26));
  k_ccs_fix_long<<<kSMs * 2, 512, 0, s>>>(col_ptr, row_idx, out_val, queue, queue_len);
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
