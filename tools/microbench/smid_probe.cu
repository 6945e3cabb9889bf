// Which SM does each CTA of a grid land on?  (Block placement for the
// SM-local row regions of the banded SpMV mapping.)
#include <cstdio>
#include <vector>
__global__ void k_smid(int* out, int spin) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = static_cast<int>(s);
  // keep the CTA resident a while so later CTAs cannot reuse its slot
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
}
int main() {
  int* d;
  cudaMalloc(&d, 4096 * sizeof(int));
  const int cfgs[][2] = {{148, 1024}, {296, 1024}, {296, 512}, {592, 256}, {1184, 256}};
  for (auto& c : cfgs) {
    const int g = c[0], b = c[1];
    k_smid<<<g, b>>>(d, 2000000);
    cudaDeviceSynchronize();
    std::vector<int> h(g);
    cudaMemcpy(h.data(), d, g * sizeof(int), cudaMemcpyDeviceToHost);
    int same = 0, per_sm[256] = {0};
    for (int i = 0; i < g; ++i) {
      per_sm[h[i]]++;
      if (i >= 148 && h[i] == h[i % 148]) ++same;
    }
    int mx = 0, mn = 1 << 30, used = 0;
    for (int s = 0; s < 256; ++s) if (per_sm[s]) { ++used; mx = per_sm[s] > mx ? per_sm[s] : mx; mn = per_sm[s] < mn ? per_sm[s] : mn; }
    printf("grid %4d x %4d: SMs used %d, CTAs/SM %d..%d, CTA b (b>=148) on the SM of CTA b%%148: %d of %d;"
           " first 16 smids:", g, b, used, mn, mx, same, g > 148 ? g - 148 : 0);
    for (int i = 0; i < 16; ++i) printf(" %d", h[i]);
    printf("\n");
  }
  return 0;
}
