// kernels_inverse.cu -- the inverse conversions on sm_100a (SURVEY.md §8f
// rank 2): any handle back to CANONICAL CRS (columns ascending inside each
// row), refusing duplicate positions, as the reference's
// triplets_to_canonical_crs (convert.cpp:119-154) does for coo_to_crs /
// ell_to_crs, and canonicalize (formats.cpp:228-244).
//
//   k_seg_sort      sort every segment of a pointer array by key (payload
//                   follows): one warp per segment <= 32 (register bitonic,
//                   sorted segments exit after one ballot), block bitonic
//                   beyond; adjacent equal keys = duplicate -> the smallest
//                   (segment, key) pair is reported through an atomicMin.
//   k_ell_gather    band-major ELL -> row-ordered CRS (padding dropped by
//                   row_entry_count, never by value, convert.cpp:166-183)
//   k_coo_*         COO triplets -> CRS: row histogram, scan, cursor scatter
#include <climits>

#include "common.cuh"
#include "spmvtk/spmvtk_kernels.h"

using namespace spmvtk_dev;

namespace {

constexpr int kSegShort = 32;

__device__ void report_dup(unsigned long long* dup, int64_t seg, int32_t key) {
  atomicMin(dup, (static_cast<unsigned long long>(seg) << 32) | static_cast<uint32_t>(key));
}

template <typename KeyPtr, typename ValPtr>
__device__ void block_bitonic_kv(KeyPtr key, ValPtr val, int32_t len) {
  int32_t P = 1;
  while (P < len) P <<= 1;
  const int32_t half = P >> 1;
  for (int32_t size = 2; size <= P; size <<= 1) {
    const int32_t h = size >> 1;
    for (int32_t t = threadIdx.x; t < half; t += blockDim.x) {
      const int32_t blk = t / h, off = t - blk * h;
      const int32_t i = blk * size + off, j = blk * size + size - 1 - off;
      if (j < len && key[i] > key[j]) {
        auto k = key[i]; key[i] = key[j]; key[j] = k;
        auto v = val[i]; val[i] = val[j]; val[j] = v;
      }
    }
    __syncthreads();
    for (int32_t d = h >> 1; d > 0; d >>= 1) {
      for (int32_t t = threadIdx.x; t < half; t += blockDim.x) {
        const int32_t blk = t / d, off = t - blk * d;
        const int32_t i = blk * 2 * d + off, j = i + d;
        if (j < len && key[i] > key[j]) {
          auto k = key[i]; key[i] = key[j]; key[j] = k;
          auto v = val[i]; val[i] = val[j]; val[j] = v;
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(256) k_seg_sort_short(const int32_t* __restrict__ ptr,
                                                        int64_t nseg, int32_t* key, double* val,
                                                        int32_t* queue, int32_t* queue_len,
                                                        unsigned long long* dup, bool packed_ok) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t sgi = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
       sgi < nseg; sgi += warps) {
    const int32_t a = __ldg(ptr + sgi), len = __ldg(ptr + sgi + 1) - a;
    if (len <= 1) continue;
    if (len > kSegShort || !packed_ok) {
      if (lane == 0) queue[atomicAdd(queue_len, 1)] = static_cast<int32_t>(sgi);
      continue;
    }
    int32_t k = lane < len ? key[a + lane] : INT_MAX;
    const int32_t kn = __shfl_down_sync(kFull, k, 1);
    if (__any_sync(kFull, lane + 1 < len && kn < k)) {
      double v = lane < len ? val[a + lane] : 0.0;
      uint32_t pk = lane < len ? (static_cast<uint32_t>(k) << 5) | lane : 0xffffffffu;
#pragma unroll
      for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int d = size >> 1; d > 0; d >>= 1) {
          const uint32_t o = __shfl_xor_sync(kFull, pk, d);
          const bool up = (lane & size) == 0, lower = (lane & d) == 0;
          pk = (lower == up) ? min(pk, o) : max(pk, o);
        }
      }
      v = __shfl_sync(kFull, v, static_cast<int>(pk & 31u));
      k = lane < len ? static_cast<int32_t>(pk >> 5) : INT_MAX;
      if (lane < len) {
        key[a + lane] = k;
        val[a + lane] = v;
      }
    }
    const int32_t k2 = __shfl_down_sync(kFull, k, 1);
    if (lane + 1 < len && k2 == k) report_dup(dup, sgi, k);
  }
}

__global__ void __launch_bounds__(512) k_seg_sort_long(const int32_t* __restrict__ ptr,
                                                       int32_t* key, double* val,
                                                       const int32_t* queue,
                                                       const int32_t* queue_len,
                                                       unsigned long long* dup) {
  const int32_t count = *queue_len;
  for (int32_t q = blockIdx.x; q < count; q += gridDim.x) {
    const int32_t sgi = queue[q];
    const int32_t a = ptr[sgi], len = ptr[sgi + 1] - a;
    block_bitonic_kv(key + a, val + a, len);
    for (int32_t t = threadIdx.x + 1; t < len; t += blockDim.x)
      if (key[a + t] == key[a + t - 1]) report_dup(dup, sgi, key[a + t]);
    __syncthreads();
  }
}

// band-major ELL -> CRS rows in ELL order (thread per row; for a fixed band
// the reads of consecutive rows are coalesced)
__global__ void __launch_bounds__(256) k_ell_gather(int64_t n, int64_t stride_k,
                                                    int64_t stride_i,
                                                    const double* __restrict__ eval,
                                                    const int32_t* __restrict__ ecol,
                                                    const int32_t* __restrict__ cnt,
                                                    const int32_t* __restrict__ irp,
                                                    int32_t* __restrict__ icol,
                                                    double* __restrict__ val) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const int32_t c = cnt[i], base = irp[i];
    for (int32_t k = 0; k < c; ++k) {
      const int64_t s = static_cast<int64_t>(k) * stride_k + i * stride_i;
      icol[base + k] = ld_stream(ecol + s);
      val[base + k] = ld_stream(eval + s);
    }
  }
}

__global__ void k_hist_keys(const int32_t* __restrict__ key, int64_t len, int32_t* count) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < len;
       p += stride)
    atomicAdd(count + ld_stream(key + p), 1);
}

// COO -> CRS scatter by row with atomic cursors (order inside a row fixed
// afterwards by k_seg_sort on the column)
__global__ void k_coo_scatter(const int32_t* __restrict__ row, const int32_t* __restrict__ col,
                              const double* __restrict__ v, int64_t nnz, int32_t* cursor,
                              int32_t* __restrict__ icol, double* __restrict__ val) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < nnz;
       p += stride) {
    const int32_t slot = atomicAdd(cursor + ld_stream(row + p), 1);
    icol[slot] = ld_stream(col + p);
    val[slot] = ld_stream(v + p);
  }
}

}  // namespace

extern "C" {

size_t spmvtk_k_canon_scratch_bytes(int64_t nseg) {
  return static_cast<size_t>(nseg + 1) * 2 * sizeof(int32_t) +
         spmvtk_k_scan_scratch_bytes(nseg + 1) + 1024;
}

int spmvtk_k_sort_segments(const int32_t* ptr, int64_t nseg, int64_t key_bound, int32_t* key,
                           double* val, unsigned long long* dup, void* scratch, void* stream) {
  cudaStream_t s = as_stream(stream);
  int32_t* queue = static_cast<int32_t*>(scratch);
  int32_t* queue_len = queue + nseg;
  cudaMemsetAsync(queue_len, 0, sizeof(int32_t), s);
  cudaMemsetAsync(dup, 0xff, sizeof(unsigned long long), s);
  if (nseg <= 0) SPMVTK_LAUNCH_RETURN();
  k_seg_sort_short<<<grid_for(nseg * 32, 256, 16), 256, 0, s>>>(
      ptr, nseg, key, val, queue, queue_len, dup, key_bound < (int64_t(1) << 27));
  k_seg_sort_long<<<kSMs * 2, 512, 0, s>>>(ptr, key, val, queue, queue_len, dup);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_ell_to_crs(int64_t n, int64_t ncols, int64_t stride_k, int64_t stride_i,
                        const double* eval, const int32_t* ecol, const int32_t* cnt,
                        int32_t* irp, int32_t* icol, double* val, unsigned long long* dup,
                        void* scratch, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) SPMVTK_LAUNCH_RETURN();
  // row pointers: exclusive scan of the per-row entry counts
  char* sc = static_cast<char*>(scratch);
  int rc = spmvtk_k_exclusive_scan(cnt, irp, n, sc, stream);
  if (rc) return rc;
  k_ell_gather<<<grid_for(n, 256), 256, 0, s>>>(n, stride_k, stride_i, eval, ecol, cnt, irp,
                                                icol, val);
  return spmvtk_k_sort_segments(irp, n, ncols, icol, val, dup,
                                sc + ((spmvtk_k_scan_scratch_bytes(n + 1) + 255) & ~size_t(255)),
                                stream);
}

int spmvtk_k_coo_to_crs(int64_t n, int64_t ncols, int64_t nnz, const int32_t* row,
                        const int32_t* col, const double* v, int32_t* irp, int32_t* icol,
                        double* val, unsigned long long* dup, void* scratch, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) SPMVTK_LAUNCH_RETURN();
  int32_t* count = static_cast<int32_t*>(scratch);
  char* rest = reinterpret_cast<char*>(count + ((n + 1 + 63) & ~int64_t(63)));
  cudaMemsetAsync(count, 0, static_cast<size_t>(n + 1) * sizeof(int32_t), s);
  if (nnz > 0) k_hist_keys<<<grid_for(nnz, 256), 256, 0, s>>>(row, nnz, count);
  int rc = spmvtk_k_exclusive_scan(count, irp, n, rest, stream);
  if (rc) return rc;
  if (nnz > 0) {
    cudaMemcpyAsync(count, irp, static_cast<size_t>(n) * sizeof(int32_t),
                    cudaMemcpyDeviceToDevice, s);
    k_coo_scatter<<<grid_for(nnz, 256), 256, 0, s>>>(row, col, v, nnz, count, icol, val);
  }
  return spmvtk_k_sort_segments(irp, n, ncols, icol, val, dup,
                                rest + ((spmvtk_k_scan_scratch_bytes(n + 1) + 255) & ~size_t(255)),
                                stream);
}

}  // extern "C"

namespace spmvtk_dev {
void preload_inverse() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_seg_sort_short);
  cudaFuncGetAttributes(&a, k_seg_sort_long);
  cudaFuncGetAttributes(&a, k_ell_gather);
  cudaFuncGetAttributes(&a, k_hist_keys);
  cudaFuncGetAttributes(&a, k_coo_scatter);
}
}  // namespace spmvtk_dev
