// Microbenchmark (design-B feasibility): tcgen05.mma.cta_group::2 throughput
// from shared memory as a function of the tile width N (M = 256 per pair, K = 16 per
// instruction), operands resident (no TMA): does a narrow-N tile (N = 64..128, the widths a
// [D x N] fp32 accumulator of 896 rows leaves in TMEM) still reach the tensor floor
// max(M,128) N / 512 cycles per instruction, or does the SMEM operand read bound it?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ubn scripts/ubench_narrow_n.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2601_02609_b200/csrc/sm100.cuh"
using namespace cce;

template <int N, int AMN, int M = 256, int PAIR = 1, int KB = 1>
__global__ void __launch_bounds__(128, 1) knarrow(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[8];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) { if (PAIR) tmem_alloc_pair(&slot, 512); else tmem_alloc(&slot, 512); }
  tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0 && lane == 0 && rank == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    const uint32_t idesc = idesc_bf16_f32(M, N, AMN, 0);
    uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int s = it & 7;
      if (it >= 8) { mbar_wait(&bar[s], ph[s]); ph[s] ^= 1; }
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < 4 * KB; ++k) {
        const uint64_t ad = AMN ? sdesc_sw128(a + (s & 1) * 32768 + (k & 3) * 2048, 8192, 1024)
                                : sdesc_sw128(a + (s & 1) * 16384 + (k & 3) * 32, 16, 1024);
        const uint64_t bd = sdesc_sw128(b + (s & 1) * 8192 + (k & 3) * 32, 16, 1024);
        if (PAIR) umma_bf16_pair(tmem + (it & 1) * 256, ad, bd, idesc, k > 0 ? 1u : 0u);
        else umma_bf16(tmem + (it & 1) * 256, ad, bd, idesc, k > 0 ? 1u : 0u);
      }
      if (PAIR) umma_commit_pair(&bar[s]); else umma_commit(&bar[s]);
    }
    for (int s = 0; s < 8; ++s) mbar_wait(&bar[s], ph[s]);
    out[blockIdx.x] = clock64() - t0;
  }
  __syncwarp();
  tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  if (warp == 1) { if (PAIR) tmem_dealloc_pair(tmem, 512); else tmem_dealloc(tmem, 512); }
}

template <int N, int AMN, int M = 256, int PAIR = 1, int KB = 1>
void run(int grid, int iters) {
  unsigned long long* d;
  cudaMalloc(&d, grid * 8);
  auto k = knarrow<N, AMN, M, PAIR, KB>;
  const int sm = 100 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = sm;
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
  cudaLaunchKernelEx(&cfg, k, iters, d);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[256];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < grid; i += (PAIR ? 2 : 1)) mx = h[i] > mx ? h[i] : mx;
  const double flops = (double)(PAIR ? grid / 2 : grid) * iters * 4 * KB * (double)M * N * 16 * 2;
  const int floor = (M > 128 ? M : 128) * N / (256 * (PAIR ? 2 : 1)) * 4;
  printf("KB=%d %s M=%3d N=%3d A_%s err=%s: %.3f ms, %.1f TFLOP/s, cycles per 64-k-block %.1f (tensor floor %d)\n",
         KB, PAIR ? "cta_group::2" : "cta_group::1", M, N, AMN ? "MN" : "K ", cudaGetErrorString(err), ms,
         flops / ms / 1e9, (double)mx / iters / KB, floor);
  cudaFree(d);
}

int main() {
  const int it = 10000;
  // KB = 2: 8 MMAs per commit, as the pair kernel issues them (two 64-wide k-blocks per stage)
  run<256, 0, 256, 1, 2>(148, it); run<240, 0, 256, 1, 2>(148, it); run<224, 0, 256, 1, 2>(148, it);
  run<208, 0, 256, 1, 2>(148, it); run<192, 0, 256, 1, 2>(148, it); run<160, 0, 256, 1, 2>(148, it);
  run<128, 0, 256, 1, 2>(148, it);
  run<224, 1, 256, 1, 2>(148, it); run<128, 1, 256, 1, 2>(148, it);
  // narrow N with many MMAs per commit (design B's shapes: N = 64..96)
  run<256, 0, 256, 1, 4>(148, it); run<128, 0, 256, 1, 4>(148, it); run<96, 0, 256, 1, 4>(148, it);
  run<64, 0, 256, 1, 4>(148, it);
  return 0;
}
