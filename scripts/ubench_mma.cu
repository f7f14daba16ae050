// Microbenchmark: raw tcgen05.mma throughput from shared memory (no TMA, no epilogue).
//   one-CTA : M=128, N=256, K=16 per instruction, cta_group::1
//   pair    : M=256, N=256, K=16 per instruction, cta_group::2 (leader issues)
// Each CTA issues `iters` k-blocks of 4 MMAs, committing every k-block to an mbarrier
// and waiting for completion every `depth` k-blocks (like a pipelined mainloop).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ubench scripts/ubench_mma.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2601_02609_b200/csrc/sm100.cuh"
using namespace cce;

template <int PAIR, int AMN = 0, int BMN = 0>
__global__ void __launch_bounds__(128, 1) kmma(int iters, unsigned long long* out, int n_k_major) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[8];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint32_t rank = 0;
  if (PAIR) rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    if (PAIR) tmem_alloc_pair(&slot, 512); else tmem_alloc(&slot, 512);
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  unsigned long long t0 = 0, t1 = 0;
  if (warp == 0 && lane == 0 && rank == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint32_t idesc = idesc_bf16_f32(PAIR ? 256 : 128, 256, AMN, BMN);
    uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int s = it & 7;
      if (it >= 8) { mbar_wait(&bar[s], ph[s]); ph[s] ^= 1; }
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = AMN ? sdesc_sw128(a + k * 2048, 8192, 1024) : sdesc_sw128(a + k * 32, 16, 1024);
        const uint64_t bd = BMN ? sdesc_sw128(b + k * 2048, 8192, 1024) : sdesc_sw128(b + k * 32, 16, 1024);
        if (PAIR) umma_bf16_pair(tmem + (it & 1) * 256, ad, bd, idesc, k > 0 ? 1u : 0u);
        else umma_bf16(tmem + (it & 1) * 256, ad, bd, idesc, k > 0 ? 1u : 0u);
      }
      if (PAIR) umma_commit_pair(&bar[s]); else umma_commit(&bar[s]);
    }
    for (int s = 0; s < 8; ++s) { mbar_wait(&bar[s], ph[s]); }
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  __syncwarp();
  tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    if (PAIR) tmem_dealloc_pair(tmem, 512); else tmem_dealloc(tmem, 512);
  }
}

template <int PAIR, int AMN = 0, int BMN = 0>
void run(int grid, int iters) {
  unsigned long long* d;
  cudaMalloc(&d, grid * 8);
  cudaMemset(d, 0, grid * 8);
  auto k = kmma<PAIR, AMN, BMN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 80 * 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = PAIR ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k, iters, d, 0);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, iters, d, 0);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[256];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  const double flops = (double)grid * iters * 4 * 128.0 * 256 * 16 * 2;  // per CTA share
  printf("amn=%d bmn=%d %s grid=%d iters=%d err=%s: %.3f ms, %.1f TFLOP/s, max cycles/kblock %.1f (ideal 512)\n",
         AMN, BMN, PAIR ? "pair M=256" : "1cta M=128", grid, iters, cudaGetErrorString(err), ms, flops / ms / 1e9,
         (double)mx / iters);
  cudaFree(d);
}

int main() {
  run<1>(148, 20000);
  run<1, 0, 1>(148, 20000);
  run<1, 1, 1>(148, 20000);
  run<1, 1, 0>(148, 20000);
  return 0;
}
