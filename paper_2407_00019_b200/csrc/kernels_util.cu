// kernels_util.cu -- row statistics, index-width conversion, validation
// scans and the device exclusive scan used by the CCS transform.
//
// HBM-bound integer work: grid-stride loops sized to a multiple of the 148
// SMs, warp-shuffle reductions, one atomic per warp.
#include <atomic>

#include <climits>

#include "common.cuh"
#include "spmvtk/spmvtk.h"
#include "spmvtk/spmvtk_kernels.h"

using namespace spmvtk_dev;

namespace {

// ---- row statistics ------------------------------------------------------
// Reference: row_histogram (formats.cpp:184-192) feeds Welford in
// stats_from_histogram (stats.cpp:9-29); max row length as in
// estimate_ell_bytes / crs_to_ell (convert.cpp:74-76, :91-96).  The device
// computes the exact integer moments {max, sum c, sum c^2}; the host turns
// them into mu / sigma / d_mat (runtime.cpp: stats_from_moments).
// One pass over the pointer array with 128-bit loads (4 rows per thread per
// step), block-level reduction in shared memory, then 3 atomics per block on
// a grid of 2 blocks per SM (per-warp atomics on 3 addresses serialised at
// L2 and cost ~20 us at n = 2^20).
constexpr int kStatsThreads = 512;

__device__ __forceinline__ void stats_add(int32_t a, int32_t b, unsigned long long& mx,
                                          unsigned long long& s, unsigned long long& s2,
                                          bool& bad) {
  if (b < a) {
    bad = true;  // non-monotone pointer array
    return;
  }
  const unsigned long long c = static_cast<unsigned long long>(b - a);
  mx = c > mx ? c : mx;
  s += c;
  s2 += c * c;
}

// acc[0..2] = max | bad<<63, sum, sum of squares.  With `host` (mapped
// pinned memory) the last CTA to finish also publishes the totals there,
// clears acc[0..3] for the next call, then publishes `seq` in host[3]: the caller
// spins on host[3] instead of a memset + copy + stream synchronisation.
__global__ void __launch_bounds__(kStatsThreads) k_row_stats(const int32_t* __restrict__ ptr,
                                                             int64_t n,
                                                             unsigned long long* acc,
                                                             volatile unsigned long long* host,
                                                             unsigned long long seq) {
  __shared__ unsigned long long s_red[3][kStatsThreads / 32];
  __shared__ int s_bad;
  unsigned long long mx = 0, s = 0, s2 = 0;
  bool bad = false;
  if (threadIdx.x == 0) s_bad = 0;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const bool aligned = (reinterpret_cast<uintptr_t>(ptr) & 15) == 0;
  const int64_t quads = aligned ? n / 4 : 0;
  for (int64_t q = tid; q < quads; q += stride) {
    const int4 v = *reinterpret_cast<const int4*>(ptr + 4 * q);
    const int32_t e = __ldg(ptr + 4 * q + 4);
    stats_add(v.x, v.y, mx, s, s2, bad);
    stats_add(v.y, v.z, mx, s, s2, bad);
    stats_add(v.z, v.w, mx, s, s2, bad);
    stats_add(v.w, e, mx, s, s2, bad);
  }
  for (int64_t i = 4 * quads + tid; i < n; i += stride)
    stats_add(__ldg(ptr + i), __ldg(ptr + i + 1), mx, s, s2, bad);
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long om = __shfl_xor_sync(kFull, mx, o);
    mx = om > mx ? om : mx;
    s += __shfl_xor_sync(kFull, s, o);
    s2 += __shfl_xor_sync(kFull, s2, o);
  }
  bad = __any_sync(kFull, bad);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) {
    s_red[0][wid] = mx;
    s_red[1][wid] = s;
    s_red[2][wid] = s2;
    if (bad) s_bad = 1;
  }
  __syncthreads();
  if (wid == 0) {
    constexpr int kW = kStatsThreads / 32;
    mx = lane < kW ? s_red[0][lane] : 0;
    s = lane < kW ? s_red[1][lane] : 0;
    s2 = lane < kW ? s_red[2][lane] : 0;
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long om = __shfl_xor_sync(kFull, mx, o);
      mx = om > mx ? om : mx;
      s += __shfl_xor_sync(kFull, s, o);
      s2 += __shfl_xor_sync(kFull, s2, o);
    }
    if (lane == 0) {
      atomicMax(acc + 0, mx | (s_bad ? (1ull << 63) : 0ull));
      atomicAdd(acc + 1, s);
      atomicAdd(acc + 2, s2);
      if (host) {
        __threadfence();
        if (atomicAdd(acc + 3, 1ull) == gridDim.x - 1) {  // last CTA: totals are final
          const unsigned long long t0 = atomicAdd(acc + 0, 0ull), t1 = atomicAdd(acc + 1, 0ull),
                                   t2 = atomicAdd(acc + 2, 0ull);
          // clear the accumulators BEFORE publishing seq: the caller may
          // launch the next reduction (on another stream) as soon as it
          // sees seq, and its atomics must not race with this reset
          acc[0] = acc[1] = acc[2] = acc[3] = 0;
          __threadfence();
          host[0] = t0;
          host[1] = t1;
          host[2] = t2;
          __threadfence_system();
          host[3] = seq;
        }
      }
    }
  }
}

__global__ void k_narrow(const int64_t* __restrict__ src, int32_t* __restrict__ dst,
                         int64_t len, int64_t base) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < len;
       i += stride)
    dst[i] = static_cast<int32_t>(src[i] - base);
}

__global__ void k_widen(const int32_t* __restrict__ src, int64_t* __restrict__ dst,
                        int64_t len, int64_t base) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < len;
       i += stride)
    dst[i] = static_cast<int64_t>(src[i]) + base;
}

__global__ void k_out_of_range(const int32_t* __restrict__ idx, int64_t len, int64_t n,
                               unsigned long long* bad) {
  unsigned long long cnt = 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < len;
       i += stride) {
    int32_t v = __ldg(idx + i);
    cnt += (v < 0 || v >= n) ? 1 : 0;
  }
  cnt = warp_sum(cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(bad, cnt);
}

__global__ void k_descents(const int32_t* __restrict__ key, int64_t len,
                           unsigned long long* bad) {
  unsigned long long cnt = 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x + 1; i < len;
       i += stride)
    cnt += (__ldg(key + i) < __ldg(key + i - 1)) ? 1 : 0;
  cnt = warp_sum(cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(bad, cnt);
}

// entries whose column is not above the previous one IN THE SAME ROW (0 =
// columns strictly ascending in every row, so no duplicate (row, col) pair):
// a warp per 32-row group walks the group's entries 32 at a time; the row
// starts among them come from the group's row ends (one per lane) as a
// 32-bit mask
__global__ void k_row_descents(const int32_t* __restrict__ irp, int64_t n,
                               const int32_t* __restrict__ col, unsigned long long* bad) {
  unsigned long long cnt = 0;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r0 = ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 32;
       r0 < n; r0 += warps * 32) {
    const int64_t r1 = r0 + 32 < n ? r0 + 32 : n;
    const int32_t a = __ldg(irp + r0), b = __ldg(irp + r1);
    const int32_t end = r0 + lane < r1 ? __ldg(irp + r0 + lane + 1) : INT_MAX;
    for (int32_t p0 = a; p0 < b; p0 += 32) {
      const unsigned bit = (end >= p0 && end < p0 + 32) ? 1u << (end - p0) : 0u;
      const unsigned starts = __reduce_or_sync(kFull, bit);
      const int32_t p = p0 + lane;
      if (p > a && p < b && !((starts >> lane) & 1u) && __ldg(col + p) <= __ldg(col + p - 1))
        ++cnt;
    }
  }
  cnt = warp_sum(cnt);
  if (lane == 0 && cnt) atomicAdd(bad, cnt);
}

// Row order + band shape of a CRS in one pass over its columns (the upload's
// ordering check, extended): out[0] descents (as k_row_descents), out[1]
// entries whose column is the previous column + 1 in the same row (stencil-
// like runs), out[2] max over rows of (last column - global row) + 2^32,
// out[3] max of (global row - first column) + 2^32 (offsets keep the atomics
// unsigned; empty rows contribute nothing).
__global__ void k_row_order_stats(const int32_t* __restrict__ irp, int64_t n, int64_t row0,
                                  const int32_t* __restrict__ col, unsigned long long* out) {
  unsigned long long desc = 0, adj = 0;
  long long right = LLONG_MIN, left = LLONG_MIN;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r0 = ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 32;
       r0 < n; r0 += warps * 32) {
    const int64_t r1 = r0 + 32 < n ? r0 + 32 : n;
    const int32_t a = __ldg(irp + r0), b = __ldg(irp + r1);
    const int32_t end = r0 + lane < r1 ? __ldg(irp + r0 + lane + 1) : INT_MAX;
    if (r0 + lane < r1) {  // lane's own row: first and last column
      const int32_t beg = __ldg(irp + r0 + lane);
      if (end > beg) {
        const long long g = row0 + r0 + lane;
        right = max(right, static_cast<long long>(__ldg(col + end - 1)) - g);
        left = max(left, g - static_cast<long long>(__ldg(col + beg)));
      }
    }
    for (int32_t p0 = a; p0 < b; p0 += 32) {
      const unsigned bit = (end >= p0 && end < p0 + 32) ? 1u << (end - p0) : 0u;
      const unsigned starts = __reduce_or_sync(kFull, bit);
      const int32_t p = p0 + lane;
      if (p > a && p < b && !((starts >> lane) & 1u)) {
        const int32_t c = __ldg(col + p), cp = __ldg(col + p - 1);
        desc += c <= cp;
        adj += c == cp + 1;
      }
    }
  }
  desc = warp_sum(desc);
  adj = warp_sum(adj);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    right = max(right, __shfl_xor_sync(kFull, right, o));
    left = max(left, __shfl_xor_sync(kFull, left, o));
  }
  if (lane == 0) {
    if (desc) atomicAdd(out, desc);
    if (adj) atomicAdd(out + 1, adj);
    const long long off = 1LL << 32;
    if (right != LLONG_MIN) atomicMax(out + 2, static_cast<unsigned long long>(right + off));
    if (left != LLONG_MIN) atomicMax(out + 3, static_cast<unsigned long long>(left + off));
  }
}

// ---- exclusive scan (tiles of 4096) -----------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int32_t block_exclusive_scan(int32_t v, int32_t* s_warp,
                                                        int32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int32_t inc = v;
  for (int d = 1; d < 32; d <<= 1) {
    int32_t t = __shfl_up_sync(kFull, inc, d);
    if (lane >= d) inc += t;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int32_t w = (lane < kScanThreads / 32) ? s_warp[lane] : 0;
    int32_t wi = w;
    for (int d = 1; d < 32; d <<= 1) {
      int32_t t = __shfl_up_sync(kFull, wi, d);
      if (lane >= d) wi += t;
    }
    if (lane < kScanThreads / 32) s_warp[lane] = wi - w;
    if (lane == kScanThreads / 32 - 1) *total = wi;
  }
  __syncthreads();
  return s_warp[wid] + inc - v;
}

__device__ __forceinline__ void load_items(const int32_t* in, int64_t n, int64_t first,
                                           int32_t (&it)[kScanItems]) {
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    int64_t i = first + j;
    it[j] = i < n ? __ldg(in + i) : 0;
  }
}

// ---- single-pass exclusive scan (decoupled look-back) --------------------
// One launch: tiles take tickets in launch order, publish their aggregate,
// then walk back over predecessors (aggregate or inclusive prefix) and
// publish their inclusive prefix.  Status word per tile: bits 63:62 flag
// (0 none, 1 aggregate, 2 inclusive), bits 31:0 the value.
__device__ __forceinline__ void publish(unsigned long long* st, unsigned long long flag,
                                        int32_t v) {
  const unsigned long long w = (flag << 62) | static_cast<uint32_t>(v);
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(st), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long peek(const unsigned long long* st) {
  unsigned long long w;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(st) : "memory");
  return w;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_lookback(const int32_t* __restrict__ in,
                                                                int32_t* __restrict__ out,
                                                                int64_t n, int64_t tiles,
                                                                unsigned long long* status,
                                                                unsigned int* ticket) {
  __shared__ int32_t s_warp[kScanThreads / 32];
  __shared__ int32_t total;
  __shared__ int32_t s_prefix;
  __shared__ unsigned int s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  int32_t it[kScanItems];
  const int64_t first = tile * kScanTile + static_cast<int64_t>(threadIdx.x) * kScanItems;
  load_items(in, n, first, it);
  int32_t sum = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) sum += it[j];
  const int32_t ex = block_exclusive_scan(sum, s_warp, &total);
  if (threadIdx.x < 32) {
    // warp 0 looks back 32 predecessors at a time: the nearest one with an
    // inclusive prefix ends the walk, the aggregates before it add up
    const int lane = threadIdx.x;
    int32_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) publish(status, 2, total);
    } else {
      if (lane == 0) publish(status + tile, 1, total);
      int64_t end = tile;  // window = predecessors [end - 32, end)
      for (;;) {
        const int64_t p = end - 1 - lane;
        const unsigned long long w = p >= 0 ? peek(status + p) : (2ull << 62);  // p < 0: zero
        const unsigned long long flag = w >> 62;
        const unsigned incl = __ballot_sync(kFull, flag == 2);
        const unsigned none = __ballot_sync(kFull, flag == 0);
        const int stop = incl ? __ffs(incl) - 1 : 31;  // nearest inclusive predecessor
        const unsigned upto = stop == 31 ? kFull : ((2u << stop) - 1u);
        if (none & upto) continue;  // a needed predecessor is still scanning: re-read
        int32_t v = lane <= stop ? static_cast<int32_t>(static_cast<uint32_t>(w)) : 0;
        for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
        prefix += v;
        if (incl) break;
        end -= 32;
      }
      if (lane == 0) publish(status + tile, 2, prefix + total);
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  int32_t run = s_prefix + ex;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t i = first + j;
    if (i < n) out[i] = run;
    run += it[j];
  }
  if (tile == tiles - 1 && threadIdx.x == kScanThreads - 1) out[n] = run;
}

// ---- step flags of the pushed multi-GPU SpMV ------------------------------
// signal: one thread per target, system-scope release store of the step
// number into this rank's slot of a peer's flag array.  wait: one thread per
// source, acquire loads until the source's flag reaches the step; bounded by
// a timeout (globaltimer) so a lost peer cannot hang the GPU -- the caller
// reads *status afterwards.
__global__ void k_flags_signal(spmvtk_flag_targets t, uint64_t value) {
  const int w = threadIdx.x;
  if (w < t.n)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(t.ptr[w]), "l"(value) : "memory");
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_flags_wait(const uint64_t* flags, int n, uint64_t value, uint64_t timeout_ns,
                             uint32_t* status) {
  const int w = threadIdx.x;
  if (w >= n) return;
  // an earlier step already timed out: fail fast instead of once per step
  if (*reinterpret_cast<volatile uint32_t*>(status) != 0) return;
  if (ld_acquire_sys(flags + w) >= value) return;
  const uint64_t t0 = global_ns();
  while (ld_acquire_sys(flags + w) < value) {
    if (global_ns() - t0 > timeout_ns) {
      atomicOr(status, 1u);
      return;
    }
    __nanosleep(64);
  }
}

// ---- random-gather rate probe -------------------------------------------
// The roofline denominator of the x gathers: 8-byte loads at hashed
// addresses of an L2-resident vector, nothing else in flight (B200: ~1 per
// SM-cycle, profiles/r01_microbench_gather.txt).
__device__ __forceinline__ uint32_t probe_hash(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}
__global__ void __launch_bounds__(512) k_gather_probe(const double* __restrict__ x, uint32_t mask,
                                                      int iters, double* out) {
  double acc = 0.0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 8
  for (int i = 0; i < iters; ++i) {
    s = probe_hash(s + i);
    acc += __ldg(x + (s & mask));
  }
  if (acc == 1.2345) out[0] = acc;  // keeps the loads alive
}

}  // namespace

extern "C" {


int spmvtk_k_row_stats(const int32_t* ptr, int64_t n, unsigned long long* acc,
                       void* stream) {
  cudaStream_t s = as_stream(stream);
  if (cudaMemsetAsync(acc, 0, 3 * sizeof(unsigned long long), s) != cudaSuccess)
    SPMVTK_LAUNCH_RETURN();
  if (n > 0)
    k_row_stats<<<grid_for((n + 3) / 4, kStatsThreads, 2), kStatsThreads, 0, s>>>(ptr, n, acc,
                                                                                nullptr, 0);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_row_stats_mapped(const int32_t* ptr, int64_t n, unsigned long long* acc,
                              unsigned long long* host, unsigned long long seq, void* stream) {
  if (n <= 0) return static_cast<int>(cudaErrorInvalidValue);
  k_row_stats<<<grid_for((n + 3) / 4, kStatsThreads, 2), kStatsThreads, 0, as_stream(stream)>>>(
      ptr, n, acc, host, seq);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_narrow_index(const int64_t* src, int32_t* dst, int64_t len,
                          int64_t base, void* stream) {
  if (len > 0) k_narrow<<<grid_for(len, 256), 256, 0, as_stream(stream)>>>(src, dst, len, base);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_widen_index(const int32_t* src, int64_t* dst, int64_t len,
                         int64_t base, void* stream) {
  if (len > 0) k_widen<<<grid_for(len, 256), 256, 0, as_stream(stream)>>>(src, dst, len, base);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_count_out_of_range(const int32_t* idx, int64_t len, int64_t n,
                                unsigned long long* bad, void* stream) {
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(bad, 0, sizeof(unsigned long long), s);
  if (len > 0) k_out_of_range<<<grid_for(len, 256), 256, 0, s>>>(idx, len, n, bad);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_count_descents(const int32_t* key, int64_t len,
                            unsigned long long* bad, void* stream) {
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(bad, 0, sizeof(unsigned long long), s);
  if (len > 1) k_descents<<<grid_for(len, 256), 256, 0, s>>>(key, len, bad);
  SPMVTK_LAUNCH_RETURN();
}

// push exchange setup: need[c] = 1 for every column a shard references
__global__ void k_mark_columns(const int32_t* __restrict__ col, int64_t len, uint8_t* need) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < len;
       p += stride)
    need[__ldg(col + p)] = 1;
}

// mask[r] bit w = rank w references global row row_offset + r (own bit set)
__global__ void k_push_mask(const uint8_t* __restrict__ need_all, int32_t world, int64_t n,
                            int64_t row_offset, int64_t rows, int32_t rank, uint8_t* mask) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < rows;
       r += stride) {
    unsigned m = 1u << rank;
    for (int32_t w = 0; w < world; ++w)
      if (need_all[static_cast<int64_t>(w) * n + row_offset + r]) m |= 1u << w;
    mask[r] = static_cast<uint8_t>(m);
  }
}

int spmvtk_k_mark_columns(const int32_t* col, int64_t len, uint8_t* need, void* stream) {
  if (len > 0) k_mark_columns<<<grid_for(len, 256), 256, 0, as_stream(stream)>>>(col, len, need);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_push_mask(const uint8_t* need_all, int32_t world, int64_t n, int64_t row_offset,
                       int64_t rows, int32_t rank, uint8_t* mask, void* stream) {
  if (rows > 0)
    k_push_mask<<<grid_for(rows, 256), 256, 0, as_stream(stream)>>>(need_all, world, n, row_offset,
                                                                   rows, rank, mask);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_count_row_descents(const int32_t* irp, int64_t n, const int32_t* col,
                                unsigned long long* bad, void* stream) {
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(bad, 0, sizeof(unsigned long long), s);
  if (n > 0) k_row_descents<<<grid_for((n + 31) / 32 * 32, 256, 16), 256, 0, s>>>(irp, n, col, bad);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_row_order_stats(const int32_t* irp, int64_t n, int64_t row_offset,
                             const int32_t* col, unsigned long long* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(out, 0, 4 * sizeof(unsigned long long), s);
  if (n > 0)
    k_row_order_stats<<<grid_for((n + 31) / 32 * 32, 256, 16), 256, 0, s>>>(irp, n, row_offset,
                                                                            col, out);
  SPMVTK_LAUNCH_RETURN();
}

size_t spmvtk_k_scan_scratch_bytes(int64_t n) {
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  return static_cast<size_t>((tiles < 1 ? 1 : tiles) + 1) * sizeof(unsigned long long);
}

int spmvtk_k_exclusive_scan(const int32_t* in, int32_t* out, int64_t n,
                            void* scratch, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) {
    cudaMemsetAsync(out, 0, sizeof(int32_t), s);
    SPMVTK_LAUNCH_RETURN();
  }
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  auto* status = static_cast<unsigned long long*>(scratch);
  auto* ticket = reinterpret_cast<unsigned int*>(status + tiles);
  cudaMemsetAsync(status, 0, static_cast<size_t>(tiles + 1) * sizeof(unsigned long long), s);
  k_scan_lookback<<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, out, n, tiles,
                                                                       status, ticket);
  SPMVTK_LAUNCH_RETURN();
}

}  // extern "C"

namespace spmvtk_dev {
std::atomic<unsigned long long> g_spmv_launches{0};
void count_launches(int k) { g_spmv_launches.fetch_add(static_cast<unsigned long long>(k)); }

void preload_util() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_gather_probe);
  cudaFuncGetAttributes(&a, k_flags_signal);
  cudaFuncGetAttributes(&a, k_flags_wait);
  cudaFuncGetAttributes(&a, k_row_stats);
  cudaFuncGetAttributes(&a, k_narrow);
  cudaFuncGetAttributes(&a, k_widen);
  cudaFuncGetAttributes(&a, k_out_of_range);
  cudaFuncGetAttributes(&a, k_descents);
  cudaFuncGetAttributes(&a, k_row_order_stats);
  cudaFuncGetAttributes(&a, k_scan_lookback);
}
}  // namespace spmvtk_dev

extern "C" unsigned long long spmvtk_k_launch_count(void) {
  return spmvtk_dev::g_spmv_launches.load();
}

extern "C" {

int spmvtk_k_flags_signal(const spmvtk_flag_targets* targets, uint64_t value, void* stream) {
  if (targets == nullptr || targets->n < 0 || targets->n > SPMVTK_MAX_PEERS)
    return static_cast<int>(cudaErrorInvalidValue);
  if (targets->n == 0) SPMVTK_LAUNCH_RETURN();
  k_flags_signal<<<1, 32, 0, as_stream(stream)>>>(*targets, value);
  SPMVTK_LAUNCH_RETURN();
}

int spmvtk_k_flags_wait(const uint64_t* flags, int32_t n, uint64_t value, uint64_t timeout_ns,
                        uint32_t* status, void* stream) {
  if (n < 0 || n > SPMVTK_MAX_PEERS || (n > 0 && (flags == nullptr || status == nullptr)))
    return static_cast<int>(cudaErrorInvalidValue);
  if (n == 0) SPMVTK_LAUNCH_RETURN();
  k_flags_wait<<<1, 32, 0, as_stream(stream)>>>(flags, n, value, timeout_ns, status);
  SPMVTK_LAUNCH_RETURN();
}

}  // extern "C"

extern "C" int spmvtk_k_gather_probe(const double* x, int64_t n_pow2, int iters, double* out,
                                     void* stream) {
  if (n_pow2 <= 0 || (n_pow2 & (n_pow2 - 1)) != 0 || iters <= 0)
    return static_cast<int>(cudaErrorInvalidValue);
  k_gather_probe<<<kSMs * 2, 512, 0, as_stream(stream)>>>(x, static_cast<uint32_t>(n_pow2 - 1),
                                                          iters, out);
  SPMVTK_LAUNCH_RETURN();
}
