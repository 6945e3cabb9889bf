// runtime.cpp -- see runtime.hpp.
#include "runtime.hpp"

#include <cstdlib>
#include <cstring>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <mutex>

#include "spmvtk/spmvtk_kernels.h"

namespace spmvtk::rt {

namespace {
thread_local cudaStream_t t_stream = nullptr;
std::once_flag g_init;
}  // namespace

void check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();  // clear sticky non-fatal error state
  std::string msg = std::string(what) + ": CUDA error " + cudaGetErrorName(e) + " (" +
                    cudaGetErrorString(e) + ")";
  if (e == cudaErrorMemoryAllocation)
    throw Error(ErrorCode::MemoryLimit, msg + " -- device memory exhausted");
  throw Error(ErrorCode::Validation, msg);
}

cudaStream_t stream() { return t_stream; }
void set_stream(cudaStream_t s) { t_stream = s; }

void init() {
  std::call_once(g_init, [] {
    int dev = 0;
    check(cudaGetDevice(&dev), "cudaGetDevice");
    cudaMemPool_t pool;
    check(cudaDeviceGetDefaultMemPool(&pool, dev), "cudaDeviceGetDefaultMemPool");
    // keep up to kPoolKeepDefault bytes cached between conversions (so a
    // timed conversion of a mid-sized matrix sub-allocates instead of paying
    // cudaMalloc); anything above is returned to the driver at the next
    // synchronisation.  spmvtk_reserve_device_memory() raises the figure.
    uint64_t threshold = kPoolKeepDefault;
    check(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold),
          "cudaMemPoolSetAttribute");
    check(static_cast<cudaError_t>(spmvtk_k_preload()), "kernel preload");
    // test hook: force a CRS kernel variant for a whole process
    if (const char* v = std::getenv("SPMVTK_CRS_VARIANT")) spmvtk_k_tune("crs_variant", std::atoi(v));
  });
}

void set_pool_keep(std::uint64_t bytes) {
  init();
  int dev = 0;
  check(cudaGetDevice(&dev), "cudaGetDevice");
  cudaMemPool_t pool;
  check(cudaDeviceGetDefaultMemPool(&pool, dev), "cudaDeviceGetDefaultMemPool");
  uint64_t threshold = std::max<std::uint64_t>(bytes, kPoolKeepDefault);
  check(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold),
        "cudaMemPoolSetAttribute");
}

void* alloc_bytes(std::size_t bytes, const char* what) {
  init();
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, bytes, t_stream);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw Error(ErrorCode::MemoryLimit, std::string(what) + ": device allocation of " +
                                            std::to_string(bytes) +
                                            " bytes failed (out of device memory)");
  }
  check(e, what);
  return p;
}

void free_bytes(void* p) { cudaFreeAsync(p, t_stream); }

namespace {
// per-thread scratch of the row-statistics round trip: a device accumulator
// (zeroed once; the kernel clears it after use) and a mapped pinned landing
// slot the kernel's last CTA writes, allocated once (the conversion timing
// t_trans pays this round trip on every CRS -> ELL call)
struct StatsScratch {
  unsigned long long* dev = nullptr;
  unsigned long long* host = nullptr;
  unsigned long long seq = 0;
  ~StatsScratch() {
    if (dev) cudaFree(dev);
    if (host) cudaFreeHost(host);
  }
};
thread_local StatsScratch t_stats;
}  // namespace

Moments row_moments(const std::int32_t* ptr, std::int64_t n) {
  init();
  if (!t_stats.dev) {
    check(cudaMalloc(&t_stats.dev, 4 * sizeof(unsigned long long)), "row statistics scratch");
    check(cudaMemset(t_stats.dev, 0, 4 * sizeof(unsigned long long)), "row statistics scratch");
    check(cudaHostAlloc(&t_stats.host, 4 * sizeof(unsigned long long), cudaHostAllocMapped),
          "row statistics scratch");
    std::memset(t_stats.host, 0, 4 * sizeof(unsigned long long));
  }
  unsigned long long h[3] = {0, 0, 0};
  if (n > 0) {
    // the kernel publishes into mapped memory; spin briefly on its sequence
    // word (no memset, no copy, no stream synchronisation on the fast path),
    // then fall back to a stream synchronisation, which also surfaces errors
    const unsigned long long seq = ++t_stats.seq;
    void* host_dev = nullptr;
    check(cudaHostGetDevicePointer(&host_dev, t_stats.host, 0), "row statistics scratch");
    check_launch(spmvtk_k_row_stats_mapped(ptr, n, t_stats.dev,
                                           static_cast<unsigned long long*>(host_dev), seq,
                                           t_stream),
                 "row statistics kernel");
    volatile unsigned long long* flag = t_stats.host + 3;
    const auto t0 = std::chrono::steady_clock::now();
    while (*flag != seq &&
           std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(200)) {
    }
    if (*flag != seq) {
      sync();
      if (*flag != seq) throw Error(ErrorCode::Validation, "row statistics did not complete");
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    const volatile unsigned long long* v = t_stats.host;
    h[0] = v[0];
    h[1] = v[1];
    h[2] = v[2];
  }
  Moments m;
  m.monotone = (h[0] >> 63) == 0;
  m.max = h[0] & ~(1ull << 63);
  m.sum = h[1];
  m.sumsq = h[2];
  return m;
}

RowStatsD stats_from_moments(const Moments& m, std::int64_t n) {
  if (n <= 0) throw Error(ErrorCode::InvalidArgument, "empty histogram");
  if (m.sum == 0)
    throw Error(ErrorCode::InvalidArgument,
                "row statistics undefined for an empty matrix (mu = 0)");
  using u128 = unsigned __int128;
  const u128 num = static_cast<u128>(static_cast<std::uint64_t>(n)) * m.sumsq -
                   static_cast<u128>(m.sum) * m.sum;  // n^2 * variance, exact
  RowStatsD s;
  s.mu = static_cast<double>(m.sum) / static_cast<double>(n);
  s.sigma = std::sqrt(static_cast<double>(static_cast<long double>(num))) /
            static_cast<double>(n);
  s.d_mat = s.sigma / s.mu;
  return s;
}

EventTimer::EventTimer() {
  check(cudaEventCreate(&a_), "cudaEventCreate");
  check(cudaEventCreate(&b_), "cudaEventCreate");
}
EventTimer::~EventTimer() {
  if (a_) cudaEventDestroy(a_);
  if (b_) cudaEventDestroy(b_);
}
void EventTimer::start() { check(cudaEventRecord(a_, t_stream), "cudaEventRecord"); }
double EventTimer::stop_seconds() {
  check(cudaEventRecord(b_, t_stream), "cudaEventRecord");
  check(cudaEventSynchronize(b_), "cudaEventSynchronize");
  float ms = 0.f;
  check(cudaEventElapsedTime(&ms, a_, b_), "cudaEventElapsedTime");
  return static_cast<double>(ms) * 1e-3;
}

void copy_to_device(void* dst, const void* src, std::size_t bytes) {
  if (bytes == 0) return;
  check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, t_stream), "H2D copy");
}
void copy_to_host(void* dst, const void* src, std::size_t bytes) {
  if (bytes) check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, t_stream), "D2H copy");
  check(cudaStreamSynchronize(t_stream), "stream synchronize");
}
void sync() { check(cudaStreamSynchronize(t_stream), "stream synchronize"); }

}  // namespace spmvtk::rt
