// spmv_out.cuh -- where an SpMV result row goes (shared by the SpMV kernels).
#pragma once

#include <cstdint>

#include "common.cuh"
#include "spmvtk/spmvtk.h"

namespace spmvtk_dev {

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
  __device__ __forceinline__ void put_local(int64_t r, double v) const { y[r] = v; }
  __device__ __forceinline__ void tile(int64_t, int64_t) const {}
  bool synced() const { return false; }
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
  // a flag wait or a counter arrival per CTA: launch one resident wave
  bool synced() const { return s.nwait > 0 || s.counter != nullptr; }
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
  // every destination whose mask bit is set (kernels with one put per
  // thread per row: ELL, the vector CRS kernels)
  __device__ __forceinline__ void put(int64_t r, double v) const {
    unsigned m = (p.mask ? __ldg(p.mask + r) : 0xffu) & ((1u << p.ndst) - 1u);
#pragma unroll 1
    while (m) {
      const int w = __ffs(m) - 1;
      m &= m - 1;
      p.dst[w][r] = v;
    }
  }
  // staged form, for kernels whose put sites are many and divergent (the
  // entry-balanced CRS SpMV, where a put to every destination at each site
  // cost ~15% at one rank): rows go to dst[local] only, then tile() copies
  // a finished contiguous range of rows to the other destinations with
  // coalesced loads and stores
  __device__ __forceinline__ void put_local(int64_t r, double v) const { p.dst[p.local][r] = v; }
  // every thread of the CTA, once the CTA's rows [r0, r1) are all put
  __device__ __forceinline__ void tile(int64_t r0, int64_t r1) const {
    if (p.ndst <= 1) return;
    __syncthreads();
    const double* src = p.dst[p.local];
    const unsigned others = ((1u << p.ndst) - 1u) & ~(1u << p.local);
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
      const double v = __ldcg(src + r);
      unsigned m = p.mask ? (__ldg(p.mask + r) & others) : others;
#pragma unroll 1
      while (m) {
        const int w = __ffs(m) - 1;
        m &= m - 1;
        p.dst[w][r] = v;
      }
    }
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


}  // namespace spmvtk_dev
