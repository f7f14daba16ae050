// Microbenchmark (design-B feasibility): L2 -> SMEM bandwidth through TMA, per SM, with every
// SM streaming the SAME L2-resident operand tiles in lockstep (as the pair kernels do: all
// CTAs sweep one W / Hc tile sequence, so after the first touch every load hits L2).
// One producer thread per CTA, `stages` x 32 KB ring (two 64-column x 128-row bf16 boxes
// per stage), a consumer thread releasing each stage as soon as it has landed.
// Reports bytes per SM clock and aggregate TB/s for a few ring depths.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ubl2 scripts/ubench_l2_tma.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_2601_02609_b200/csrc/sm100.cuh"
using namespace cce;

__global__ void __launch_bounds__(64, 1) kl2(const __grid_constant__ CUtensorMap tm, int iters, int stages,
                                             int rows_total, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[8], empty[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      if (it >= stages) mbar_wait(&empty[s], ((it / stages) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], 32768);
      const int row = (it * 128) % rows_total;
      tma_load_2d(&tm, &full[s], smem + s * 32768, 0, row);
      tma_load_2d(&tm, &full[s], smem + s * 32768 + 16384, 64, row);
    }
    (void)ph;
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      mbar_wait(&full[s], (it / stages) & 1);
      mbar_arrive(&empty[s]);
    }
    out[blockIdx.x] = clock64() - t0;
  }
}

typedef CUresult (*PFN_encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  PFN_encode enc = (PFN_encode)fn;
  for (int mb : {16, 64, 512}) {
    const int D = 896;
    const int rows = (int)((size_t)mb * 1024 * 1024 / (D * 2)) / 128 * 128;
    void* buf;
    cudaMalloc(&buf, (size_t)rows * D * 2);
    cudaMemset(buf, 0, (size_t)rows * D * 2);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)D * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    cudaFuncSetAttribute(kl2, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768 + 1024);
    for (int stages : {2, 3, 4, 6}) {
      const int iters = 20000;
      kl2<<<148, 64, 6 * 32768 + 1024>>>(tm, 200, stages, rows, d);
      if (cudaGetLastError() != cudaSuccess) { printf("launch failed\n"); return 1; }
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      kl2<<<148, 64, 6 * 32768 + 1024>>>(tm, iters, stages, rows, d);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long h[148], mx = 0;
      cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      const double bytes = 148.0 * iters * 32768;
      printf("footprint %3d MB stages %d err=%s: %.2f TB/s aggregate, %.1f B/clk/SM (slowest SM)\n", mb, stages,
             cudaGetErrorString(err), bytes / ms / 1e9, (double)iters * 32768 / mx);
    }
    cudaFree(buf);
    cudaFree(d);
  }
  return 0;
}
