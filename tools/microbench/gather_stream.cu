// Random-gather rate with a concurrent matrix stream: does streaming the
// matrix through the LSU (L1 miss tracking) cost gather throughput that a
// TMA bulk stream (cp.async.bulk into shared memory, tracked by mbarriers)
// would not?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_stream gather_stream.cu
//
// Per SM: 12 bytes of stream per gather (an SpMV's VAL + ICOL per entry).
//   lsu_only  gathers only (x = 32 MB, L2-resident)
//   lsu_lsu   each warp alternates 128 gathers with 1.5 KB of coalesced
//             128-bit stream loads (the CRS/COO kernels' pattern)
//   lsu_tma   warp 0 lane 0 streams the CTA's share with 1-D bulk copies into
//             a shared-memory ring; the other warps gather
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra W;\n}\n" ::"r"(smem_u32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ int4 ld_nc4(const int4* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// G gathers per thread per round; stream: 12*32*G bytes per warp per round
template <int G>
__global__ void k_lsu(const double* __restrict__ x, uint32_t mask, const int4* __restrict__ stream,
                      int64_t stream_words_per_warp, int rounds, int with_stream, double* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int4* sp = stream + warp * stream_words_per_warp;
  double acc = 0;
  int sacc = 0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  // per round per warp: 32*G gathers, 12*32*G bytes = 24*G int4 words
  constexpr int W = 24 * G / 32;  // int4 words per lane per round
  for (int r = 0; r < rounds; ++r) {
    int4 w[W > 0 ? W : 1];
    if (with_stream) {
#pragma unroll
      for (int k = 0; k < W; ++k) w[k] = ld_nc4(sp + (static_cast<int64_t>(r) * W + k) * 32 + lane);
    }
    double g[G];
#pragma unroll
    for (int k = 0; k < G; ++k) {
      s = hash(s + k);
      g[k] = __ldg(x + (s & mask));
    }
#pragma unroll
    for (int k = 0; k < G; ++k) acc += g[k];
    if (with_stream) {
#pragma unroll
      for (int k = 0; k < W; ++k) sacc += w[k].x ^ w[k].w;
    }
  }
  if (acc == 1.2345 || sacc == 12345) out[0] = acc + sacc;
}

// warp 0 lane 0: bulk stream of `bytes_per_cta` in CHUNK pieces through a
// ring of S slots; warps 1..: gathers
template <int G, int S, int CHUNK>
__global__ void k_tma(const double* __restrict__ x, uint32_t mask, const char* __restrict__ stream,
                      int64_t bytes_per_cta, int rounds, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  unsigned char* ring = sm + 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < S) mbar_init(full + threadIdx.x, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      const char* src = stream + static_cast<int64_t>(blockIdx.x) * bytes_per_cta;
      const int64_t nchunks = bytes_per_cta / CHUNK;
      for (int64_t c = 0; c < nchunks; ++c) {
        const int k = static_cast<int>(c % S);
        if (c >= S) mbar_wait(full + k, ((c / S) - 1) & 1);
        mbar_expect(full + k, CHUNK);
        bulk(ring + k * CHUNK, src + c * CHUNK, CHUNK, full + k);
      }
      for (int64_t c = (nchunks > S ? nchunks - S : 0); c < nchunks; ++c)
        mbar_wait(full + (c % S), (c / S) & 1);
    }
  } else {
    double acc = 0;
    uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    for (int r = 0; r < rounds; ++r) {
      double g[G];
#pragma unroll
      for (int k = 0; k < G; ++k) {
        s = hash(s + k);
        g[k] = __ldg(x + (s & mask));
      }
#pragma unroll
      for (int k = 0; k < G; ++k) acc += g[k];
    }
    if (acc == 1.2345) out[0] = acc;
  }
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double sm_hz = double(sms) * clk * 1e3;
  const uint32_t words = 1u << 22;  // 32 MB x
  double* x;
  double* out;
  char* stream;
  const size_t stream_bytes = size_t(2) << 30;  // 2 GB pool (larger than L2)
  cudaMalloc(&x, words * 8);
  cudaMemset(x, 0, words * 8);
  cudaMalloc(&out, 64);
  cudaMalloc(&stream, stream_bytes);
  cudaMemset(stream, 0, stream_bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e-3 / 5;
  };
  constexpr int G = 4;
  for (int tpb : {256, 512}) {
    for (int bps : {2, 4}) {
      if (tpb * bps > 2048) continue;
      const int blocks = sms * bps;
      const int64_t warps = int64_t(blocks) * tpb / 32;
      const int words_per_round = 24 * G;  // int4 per warp per round
      const int rounds = int(stream_bytes / 16 / warps / words_per_round);
      const int64_t spw = int64_t(rounds) * words_per_round;
      for (int ws : {0, 1}) {
        double t = timeit([&] {
          k_lsu<G><<<blocks, tpb>>>(x, words - 1, reinterpret_cast<const int4*>(stream), spw, rounds,
                                    ws, out);
        });
        const double gathers = double(warps) * 32 * G * rounds;
        const double sbytes = ws ? double(warps) * spw * 16 : 0;
        printf("lsu%s tpb=%d ctas/sm=%d: %.1f us  gathers %.3f/SM-cycle  stream %.0f GB/s\n",
               ws ? "+lsu-stream" : "           ", tpb, bps, t * 1e6, gathers / t / sm_hz,
               sbytes / t / 1e9);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e) printf("err %s\n", cudaGetErrorString(e));
  // TMA stream: bytes per CTA = 12 * gathers of the CTA
  constexpr int S = 8, CHUNK = 8192;
  for (int tpb : {256, 512, 1024}) {
    for (int bps : {1, 2}) {
      if (tpb * bps > 2048) continue;
      const int blocks = sms * bps;
      const int gwarps = tpb / 32 - 1;
      const int64_t per_cta_stream = (int64_t(stream_bytes) / blocks) / CHUNK * CHUNK;
      const int rounds = int(per_cta_stream / 12 / (int64_t(gwarps) * 32 * G));
      const size_t sh = 128 + S * CHUNK;
      cudaFuncSetAttribute(k_tma<G, S, CHUNK>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sh));
      for (int with : {0, 1}) {
        const int64_t bytes = with ? per_cta_stream : 0;
        double t = timeit([&] {
          k_tma<G, S, CHUNK><<<blocks, tpb, sh>>>(x, words - 1, stream, bytes, rounds, out);
        });
        const double gathers = double(blocks) * gwarps * 32 * G * rounds;
        printf("lsu%s tpb=%d ctas/sm=%d: %.1f us  gathers %.3f/SM-cycle  stream %.0f GB/s\n",
               with ? "+tma-stream" : "           ", tpb, bps, t * 1e6, gathers / t / sm_hz,
               double(blocks) * bytes / t / 1e9);
      }
    }
  }
  e = cudaGetLastError();
  if (e) printf("err %s\n", cudaGetErrorString(e));
  cudaDeviceSynchronize();
  printf("done\n");
  return 0;
}
