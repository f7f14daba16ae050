// Probe: are cvta.to.shared addresses cluster-window addresses carrying the CTA rank?
#include <cstdio>
#include "../paper_2601_02609_b200/csrc/sm100.cuh"
using namespace cce;
__global__ void __cluster_dims__(4, 1, 1) probe(unsigned* out) {
  __shared__ uint64_t bar;
  const uint32_t r = cluster_ctarank();
  if (threadIdx.x == 0) {
    const uint32_t local = smem_u32(&bar);
    out[r * 6 + 0] = local;
    for (int k = 0; k < 4; ++k) out[r * 6 + 1 + k] = mapa_shared(local, k);
    out[r * 6 + 5] = r;
  }
}
int main() {
  unsigned* d;
  cudaMalloc(&d, 4 * 6 * 4);
  probe<<<4, 32>>>(d);
  unsigned h[24];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int r = 0; r < 4; ++r)
    printf("rank %u: cvta=0x%08x mapa0=0x%08x mapa1=0x%08x mapa2=0x%08x mapa3=0x%08x\n", h[r * 6 + 5], h[r * 6],
           h[r * 6 + 1], h[r * 6 + 2], h[r * 6 + 3], h[r * 6 + 4]);
  return 0;
}
