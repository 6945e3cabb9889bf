// runtime.hpp -- host runtime around the kernels: error mapping, the
// per-thread stream, stream-ordered device buffers, event timing.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>

#include "spmvtk/error.hpp"

namespace spmvtk::rt {

// Throws spmvtk::Error for a failed CUDA call: allocation failures map to
// MemoryLimit (-> SPMVTK_ERR_MEMORY_LIMIT), everything else to Validation
// (-> SPMVTK_ERR_DATA).
void check(cudaError_t e, const char* what);
inline void check_launch(int rc, const char* what) {
  check(static_cast<cudaError_t>(rc), what);
}

// Current stream of the calling thread (default: legacy stream 0).
cudaStream_t stream();
void set_stream(cudaStream_t s);

// One-time: device selection check, memory-pool release threshold (so
// stream-ordered allocations are served from the pool after warm-up), and
// module preload so no timed call pays lazy kernel loading.
void init();

// Bytes the stream-ordered pool keeps cached after frees (the release
// threshold); set_pool_keep() raises it (spmvtk_reserve_device_memory).
inline constexpr std::uint64_t kPoolKeepDefault = 2ull << 30;
void set_pool_keep(std::uint64_t bytes);

void* alloc_bytes(std::size_t bytes, const char* what);
void free_bytes(void* p);

// Stream-ordered device buffer (cudaMallocAsync / cudaFreeAsync).
template <typename T>
class DevArray {
 public:
  DevArray() = default;
  explicit DevArray(std::size_t count, const char* what = "device buffer") { reset(count, what); }
  DevArray(const DevArray&) = delete;
  DevArray& operator=(const DevArray&) = delete;
  DevArray(DevArray&& o) noexcept
      : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)), own_(o.own_) {}
  DevArray& operator=(DevArray&& o) noexcept {
    if (this != &o) {
      release();
      p_ = std::exchange(o.p_, nullptr);
      n_ = std::exchange(o.n_, 0);
      own_ = o.own_;
    }
    return *this;
  }
  ~DevArray() { release(); }

  void reset(std::size_t count, const char* what = "device buffer") {
    release();
    if (count) p_ = static_cast<T*>(alloc_bytes(count * sizeof(T), what));
    n_ = count;
  }
  void release() {
    if (p_ && own_) free_bytes(p_);
    p_ = nullptr;
    n_ = 0;
    own_ = true;
  }
  // A non-owning view into another buffer (e.g. a slice of one allocation
  // that holds several arrays of a handle); the owner must outlive it.
  void view(T* p, std::size_t count) {
    release();
    p_ = p;
    n_ = count;
    own_ = false;
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  std::size_t bytes() const { return n_ * sizeof(T); }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
  bool own_ = true;
};

// Exact integer moments of the row lengths, from the GPU reduction.
struct Moments {
  std::uint64_t max = 0;
  std::uint64_t sum = 0;
  std::uint64_t sumsq = 0;
  bool monotone = true;
};
Moments row_moments(const std::int32_t* ptr, std::int64_t n);  // synchronises

struct RowStatsD {
  double mu = 0, sigma = 0, d_mat = 0;
};
// mu = sum/n, sigma = sqrt(n*sumsq - sum^2)/n evaluated exactly in 128-bit
// integers (one rounding), d_mat = sigma/mu.  Throws InvalidArgument when
// nnz == 0, with the reference's message (stats.cpp:21-23).
RowStatsD stats_from_moments(const Moments& m, std::int64_t n);

// Device timer on the current stream.
class EventTimer {
 public:
  EventTimer();
  ~EventTimer();
  void start();
  double stop_seconds();  // synchronises on the stop event
 private:
  cudaEvent_t a_ = nullptr, b_ = nullptr;
};

void copy_to_device(void* dst, const void* src, std::size_t bytes);
void copy_to_host(void* dst, const void* src, std::size_t bytes);  // synchronises
void sync();

}  // namespace spmvtk::rt
