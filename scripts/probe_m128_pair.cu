// Probe: where does tcgen05.mma.cta_group::2 with M = 128 put its accumulator rows in each
// CTA's TMEM?  A[m][0] = m + 1 (64 rows per CTA), B[n][0] = 1 -> D[m][n] = m + 1.  Every
// CTA reads column 0 and column 200 of all 128 lanes and prints which row each lane holds.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/pm scripts/probe_m128_pair.cu
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "../paper_2601_02609_b200/csrc/sm100.cuh"
using namespace cce;

__global__ void __launch_bounds__(128, 1) kprobe(float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  // zero A (64 rows x 128 B) and B (128 rows x 128 B)
  for (int i = threadIdx.x; i < (64 + 128) * 128 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  __syncthreads();
  __nv_bfloat16* A = reinterpret_cast<__nv_bfloat16*>(smem);
  __nv_bfloat16* B = reinterpret_cast<__nv_bfloat16*>(smem + 64 * 128);
  if (threadIdx.x < 64) {
    const int r = threadIdx.x;
    A[(r * 128 + (r & 7) * 16) / 2] = __float2bfloat16((float)(64 * rank + r + 1));
  }
  for (int r = threadIdx.x; r < 128; r += 128) B[(r * 128 + (r & 7) * 16) / 2] = __float2bfloat16(1.f);
  fence_proxy_async_shared();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 1) tmem_alloc_pair(&slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0 && rank == 0) {
    if (elect_one()) {
      const uint64_t ad = sdesc_sw128(smem_u32(A), 16, 1024);
      const uint64_t bd = sdesc_sw128(smem_u32(B), 16, 1024);
      umma_bf16_pair(tmem, ad, bd, idesc_bf16_f32(128, 256, 0, 0), 0u);
      umma_commit_pair(&bar);
    }
    __syncwarp();
  }
  mbar_wait_cluster(&bar, 0);
  tc_fence_after();
  float v[32];
  tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
  out[(rank * 128 + warp * 32 + lane) * 2 + 0] = v[0];
  tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 192, v);
  out[(rank * 128 + warp * 32 + lane) * 2 + 1] = v[8];
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair(tmem, 512);
}

int main() {
  float* d;
  cudaMalloc(&d, 2 * 128 * 2 * 4);
  cudaMemset(d, 0xff, 2 * 128 * 2 * 4);
  cudaFuncSetAttribute(kprobe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 64 * 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kprobe, d);
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  float h[512];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int c = 0; c < 2; ++c) {
    printf("CTA %d lane: row+1 (col 0) / (col 200)\n", c);
    for (int l = 0; l < 128; ++l) printf("%d:%g/%g%s", l, h[(c * 128 + l) * 2], h[(c * 128 + l) * 2 + 1], (l % 8 == 7) ? "\n" : "  ");
  }
  return 0;
}
