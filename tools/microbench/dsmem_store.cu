// Coalesced distributed-shared-memory STORES inside a cluster (records moved
// in bulk between the shared memories of a cluster's CTAs): aggregate rate,
// for the fused refine+sort idea of the CRS->CCS pipeline.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int C>
__global__ void __cluster_dims__(C, 1, 1) __launch_bounds__(512) k_dsmem_store(int rounds, int* sink) {
  extern __shared__ int4 buf[];  // 64 KB
  cg::cluster_group cl = cg::this_cluster();
  const unsigned me = cl.block_rank();
  const int t = threadIdx.x, w = t >> 5;
  int4 v = make_int4(t, me, 1, 2);
  for (int r = 0; r < rounds; ++r) {
    // each warp stores 512 contiguous bytes into another CTA's buffer
    const unsigned dst = (me + 1 + ((w + r) % (C - 1))) % C;
    int4* remote = cl.map_shared_rank(buf, dst);
    const int slot = ((r * 16 + w) % 128) * 32 + (t & 31);  // 4096 int4 = 64 KB
    remote[slot] = v;
    v.z += 1;
    if ((r & 15) == 15) cl.sync();
  }
  cl.sync();
  if (t == 0) sink[blockIdx.x] = buf[t].x;
}

template <int C>
__global__ void __launch_bounds__(512) k_local_store(int rounds, int* sink) {
  extern __shared__ int4 buf[];
  const int t = threadIdx.x, w = t >> 5;
  int4 v = make_int4(t, 0, 1, 2);
  for (int r = 0; r < rounds; ++r) {
    const int slot = ((r * 16 + w) % 128) * 32 + (t & 31);
    buf[slot] = v;
    v.z += 1;
    if ((r & 15) == 15) __syncthreads();
  }
  __syncthreads();
  if (t == 0) sink[blockIdx.x] = buf[t].x;
}

template <typename K>
void run(const char* name, K kern, int grid, int rounds) {
  int* sink;
  cudaMalloc(&sink, 4096 * 4);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  kern<<<grid, 512, 65536>>>(rounds, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<grid, 512, 65536>>>(rounds, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = double(grid) * 512 * 16 * rounds;
  printf("%-22s grid %4d: %8.3f ms  %8.1f GB/s aggregate  %6.1f B/SM-cycle@1.9GHz  err=%s\n", name, grid,
         ms, bytes / ms / 1e6, bytes / (ms * 1e-3) / 148 / 1.9e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink);
}

int main() {
  const int rounds = 4096;
  run("local smem", k_local_store<1>, 296, rounds);
  run("dsmem cluster 2", k_dsmem_store<2>, 296, rounds);
  run("dsmem cluster 4", k_dsmem_store<4>, 296, rounds);
  run("dsmem cluster 8", k_dsmem_store<8>, 296, rounds);
  return 0;
}
