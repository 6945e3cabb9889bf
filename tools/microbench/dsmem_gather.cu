// Random 8-byte gather throughput on B200: L2-resident global (__ldg), local
// shared memory, and distributed shared memory across a thread-block cluster.
// Decides whether a cluster-resident x window pays for banded SpMV.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_gather dsmem_gather.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

constexpr int kWords = 16384;  // doubles per CTA's shared array (128 KB)
constexpr int kIters = 256;

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

__global__ void k_global(const double* __restrict__ x, uint32_t mask, double* out) {
  double acc = 0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 8
  for (int i = 0; i < kIters; ++i) {
    s = hash(s + i);
    acc += __ldg(x + (s & mask));
  }
  if (acc == 1.2345) out[0] = acc;
}

__global__ void k_local(double* out) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double acc = 0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 8
  for (int i = 0; i < kIters; ++i) {
    s = hash(s + i);
    acc += sm[s & (kWords - 1)];
  }
  if (acc == 1.2345) out[0] = acc;
}

template <int C>
__global__ void __cluster_dims__(C, 1, 1) k_dsmem(double* out) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) sm[i] = i;
  cl.sync();
  double* remote[C];
#pragma unroll
  for (int r = 0; r < C; ++r) remote[r] = cl.map_shared_rank(sm, r);
  double acc = 0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 8
  for (int i = 0; i < kIters; ++i) {
    s = hash(s + i);
    acc += remote[(s >> 20) % C][s & (kWords - 1)];
  }
  cl.sync();
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  double *x, *out;
  const size_t nx = 1 << 20;  // 8 MB (L2-resident)
  cudaMalloc(&x, nx * 8);
  cudaMemset(x, 0, nx * 8);
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 512, blocks = 148 * 2;
  const double gathers = double(threads) * blocks * kIters;
  auto run = [&](const char* name, auto launch) {
    launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 10;
    printf("%-14s %8.3f ms  %7.1f Ggathers/s  %5.2f per SM-cycle@1.9GHz  err=%s\n", name, ms,
           gathers / ms / 1e6, gathers / (ms * 1e-3) / 148 / 1.9e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  run("global(L2)", [&] { k_global<<<blocks, threads>>>(x, nx - 1, out); });
  cudaFuncSetAttribute(k_local, cudaFuncAttributeMaxDynamicSharedMemorySize, kWords * 8);
  run("local smem", [&] { k_local<<<blocks, threads, kWords * 8>>>(out); });
  cudaFuncSetAttribute(k_dsmem<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWords * 8);
  cudaFuncSetAttribute(k_dsmem<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWords * 8);
  cudaFuncSetAttribute(k_dsmem<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWords * 8);
  run("dsmem c=2", [&] { k_dsmem<2><<<blocks, threads, kWords * 8>>>(out); });
  run("dsmem c=4", [&] { k_dsmem<4><<<blocks, threads, kWords * 8>>>(out); });
  run("dsmem c=8", [&] { k_dsmem<8><<<blocks, threads, kWords * 8>>>(out); });
  return 0;
}
