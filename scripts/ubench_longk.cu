// Microbenchmark: long-K pair GEMM shaped like the backward's dW items (K = n_valid rows,
// A = one vocabulary tile of G^T streamed from HBM, B = hidden tiles of Hc), with a real
// epilogue (TMEM -> bf16 -> global), to compare
//   pair  : 256 x 256 tile per CTA pair, 6-stage ring (32 KB / stage / CTA), 2 accumulators
//   wide  : 256 x 512 tile per CTA pair (A shared by two N = 256 MMAs), 4-stage ring
//           (48 KB / stage / CTA), one 512-column accumulator (epilogue not overlapped)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/ubench_longk scripts/ubench_longk.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <vector>
#include "../paper_2601_02609_b200/csrc/sm100.cuh"
using namespace cce;

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled enc;
static uint64_t g_ldb = 0;
static int g_rot = 0;       // rotate each pair's k-loop start (desynchronises operand sharing)  // row stride (elements) override for the MN-major B map
static void mk(CUtensorMap* m, void* p, uint64_t cols, uint64_t rows, uint32_t box_rows, uint64_t ld = 0) {
  cuuint64_t d[2] = {cols, rows}, s[1] = {(ld ? ld : cols) * 2};
  cuuint32_t b[2] = {64, box_rows}, e[2] = {1, 1};
  enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

// WIDE = 0: pair tile 256x256, ST = 6, 2 accumulators.  WIDE = 1: 256x512, ST = 4, 1 acc.
// MN = 1: both operands MN-major (stored [K][rows]; two 64 x 64 boxes per 128 rows), as
// the dW items load G^T and Hc.
template <int WIDE, int MN = 0>
__global__ void __launch_bounds__(256, 1) klk(const __grid_constant__ CUtensorMap ta,
                                              const __grid_constant__ CUtensorMap tb, int K, int tiles_v,
                                              int tiles_d, __nv_bfloat16* C, int ldc, unsigned long long* out,
                                              int epi_mode, const __grid_constant__ CUtensorMap tc, int rot) {
  constexpr int ST = WIDE ? 4 : 6;
  constexpr int NB = WIDE ? 2 : 1;                 // B boxes (N = 256 halves) per stage
  constexpr int STAGE = 16384 * (1 + NB);
  constexpr int NACC = WIDE ? 1 : 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[ST], empty[ST], tfull[2], tempty[2];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const int unit = blockIdx.x / 2, nunits = gridDim.x / 2;
  const int num_kb = K / 64;
  const int dt_per = WIDE ? 2 : 1;
  const int items = tiles_v * (tiles_d / dt_per);
  if (threadIdx.x == 0) {
    for (int i = 0; i < ST; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 8); }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(&slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0 && lane == 0) {
    uint32_t st = 0, ph = 0;
    const uint32_t fb0 = mapa_shared(smem_u32(&full[0]), 0);
    for (int x = unit; x < items; x += nunits) {
      const int vt = x / (tiles_d / dt_per), d0 = (x % (tiles_d / dt_per)) * dt_per;
      for (int kb_ = 0; kb_ < num_kb; ++kb_) {
        const int kb = rot ? (kb_ + unit * 13) % num_kb : kb_;
        mbar_wait(&empty[st], ph ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(&full[st], 2 * STAGE);
        uint8_t* s = smem + st * STAGE;
        if (MN) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            tma_load_2d_pair(&ta, fb0 + st * 8, s + h * 8192, vt * 256 + rank * 128 + h * 64, kb * 64);
#pragma unroll
            for (int j = 0; j < NB; ++j)
              tma_load_2d_pair(&tb, fb0 + st * 8, s + 16384 * (1 + j) + h * 8192, (d0 + j) * 256 + rank * 128 + h * 64,
                               kb * 64);
          }
        } else {
          tma_load_2d_pair(&ta, fb0 + st * 8, s, kb * 64, vt * 256 + rank * 128);
#pragma unroll
          for (int j = 0; j < NB; ++j)
            tma_load_2d_pair(&tb, fb0 + st * 8, s + 16384 * (1 + j), kb * 64, (d0 + j) * 256 + rank * 128);
        }
        if (++st == ST) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1 && rank == 0) {
    uint32_t st = 0, ph = 0;
    const uint32_t idesc = idesc_bf16_f32(256, 256, MN, MN);
    const unsigned long long t0 = clock64();
    int it = 0;
    for (int x = unit; x < items; x += nunits, ++it) {
      const int acc = it % NACC;
      const uint32_t aph = (it / NACC) & 1;
      mbar_wait(&tempty[acc], aph ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full[st], ph);
        tc_fence_after();
        const uint32_t a = smem_u32(smem + st * STAGE);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = MN ? sdesc_sw128(a + k * 2048, 8192, 1024) : sdesc_sw128(a + k * 32, 16, 1024);
#pragma unroll
            for (int j = 0; j < NB; ++j) {
              const uint64_t bd = MN ? sdesc_sw128(a + 16384 * (1 + j) + k * 2048, 8192, 1024)
                                     : sdesc_sw128(a + 16384 * (1 + j) + k * 32, 16, 1024);
              umma_bf16_pair(tmem + acc * 256 + j * 256, ad, bd, idesc, (kb | k) ? 1u : 0u);
            }
          }
          umma_commit_pair(&empty[st]);
        }
        __syncwarp();
        if (++st == ST) { st = 0; ph ^= 1; }
      }
      if (elect_one()) umma_commit_pair(&tfull[acc]);
      __syncwarp();
    }
    if (lane == 0) out[blockIdx.x] = (clock64() - t0) / (unsigned long long)(it * num_kb * NB > 0 ? it * num_kb * NB : 1);
  } else if (warp >= 4) {
    const int q = warp - 4;
    const uint32_t tl0 = mapa_shared(smem_u32(&tempty[0]), 0);
    int it = 0;
    for (int x = unit; x < items; x += nunits, ++it) {
      const int vt = x / (tiles_d / dt_per), d0 = (x % (tiles_d / dt_per)) * dt_per;
      const int acc = it % NACC;
      mbar_wait(&tfull[acc], (it / NACC) & 1);
      tc_fence_after();
      const int row = vt * 256 + rank * 128 + q * 32 + lane;
      if (epi_mode >= 2) {  // G-like: bf16 tile staged in SMEM (128B swizzle), then TMA store (2) or coalesced STG (3)
        uint4* stg = reinterpret_cast<uint4*>(smem + ST * STAGE + q * 4096);
#pragma unroll 1
        for (int j2 = 0; j2 < 4 * NB; ++j2) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            float v[32];
            tmem_ld32(tmem + acc * 256 + ((uint32_t)(q * 32) << 16) + j2 * 64 + hh * 32, v);
            if (hh == 0 && epi_mode == 2 && j2 > 0) {
              if (lane == 0) bulk_wait_read<0>();
              __syncwarp();
            }
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const int chunk = hh * 4 + q4;
              stg[lane * 8 + (chunk ^ (lane & 7))] =
                  make_uint4(pack_bf16(ex2(v[8 * q4]), ex2(v[8 * q4 + 1])), pack_bf16(ex2(v[8 * q4 + 2]), ex2(v[8 * q4 + 3])),
                             pack_bf16(ex2(v[8 * q4 + 4]), ex2(v[8 * q4 + 5])), pack_bf16(ex2(v[8 * q4 + 6]), ex2(v[8 * q4 + 7])));
            }
          }
          const int row0 = vt * 256 + rank * 128 + q * 32;
          const int col0 = d0 * 256 + j2 * 64;
          if (epi_mode == 2) {
            fence_proxy_async_shared();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tc, stg, col0, row0);
              bulk_commit();
            }
          } else {
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int r = i * 4 + (lane >> 3), c = lane & 7;
              *reinterpret_cast<uint4*>(C + (size_t)(row0 + r) * ldc + col0 + c * 8) = stg[r * 8 + (c ^ (r & 7))];
            }
            __syncwarp();
          }
        }
        if (epi_mode == 2) {
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (rank == 0) mbar_arrive(&tempty[acc]);
          else mbar_arrive_cluster_relaxed(tl0 + acc * 8);
        }
        continue;
      }
      if (epi_mode == 1) {  // forward-like: online (max, sum-exp) over the row, no stores
        float m = -1e30f, dsum = 0.f;
#pragma unroll 1
        for (int j = 0; j < 8 * NB; ++j) {
          float v[32];
          tmem_ld32(tmem + acc * 256 + ((uint32_t)(q * 32) << 16) + j * 32, v);
          float cm = v[0];
#pragma unroll
          for (int i = 1; i < 32; ++i) cm = fmaxf(cm, v[i]);
          const float mn = fmaxf(m, cm);
          float s0 = 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i) s0 += ex2(v[i] - mn);
          dsum = dsum * ex2(m - mn) + s0;
          m = mn;
        }
        if (dsum == 12345.f) C[row] = __float2bfloat16(m);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (rank == 0) mbar_arrive(&tempty[acc]);
          else mbar_arrive_cluster_relaxed(tl0 + acc * 8);
        }
        continue;
      }
#pragma unroll 1
      for (int j = 0; j < 8 * NB; ++j) {
        float v[32];
        tmem_ld32(tmem + acc * 256 + ((uint32_t)(q * 32) << 16) + j * 32, v);
        uint4* dst = reinterpret_cast<uint4*>(C + (size_t)row * ldc + d0 * 256 + j * 32);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          dst[q4] = make_uint4(pack_bf16(v[8 * q4], v[8 * q4 + 1]), pack_bf16(v[8 * q4 + 2], v[8 * q4 + 3]),
                               pack_bf16(v[8 * q4 + 4], v[8 * q4 + 5]), pack_bf16(v[8 * q4 + 6], v[8 * q4 + 7]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(&tempty[acc]);
        else mbar_arrive_cluster_relaxed(tl0 + acc * 8);
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair(tmem, 512);
}

__global__ void fill_random(uint16_t* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed * 0x9E3779B9u;
    x ^= x >> 15; x *= 0x2c1b3c6dU; x ^= x >> 12; x *= 0x297a2d39U; x ^= x >> 15;
    p[i] = (uint16_t)(((x & 1) << 15) | ((0x79 + ((x >> 1) & 1)) << 7) | ((x >> 8) & 0x7F));
  }
}

template <int WIDE, int MN = 0>
void run(void* A, void* B, __nv_bfloat16* C, int MV, int ND, int K, int epi_mode = 0) {
  CUtensorMap ta, tb;
  if (MN) {
    mk(&ta, A, MV, K, 64);
    mk(&tb, B, ND, K, 64, g_ldb);
  } else {
    mk(&ta, A, K, MV, 128);
    mk(&tb, B, K, ND, 128);
  }
  constexpr int ST = WIDE ? 4 : 6, STAGE = 16384 * (1 + (WIDE ? 2 : 1));
  const int smem = ST * STAGE + 1024 + 4 * 4096;
  CUtensorMap tcm;
  {
    cuuint64_t d[2] = {(cuuint64_t)ND, (cuuint64_t)MV}, st[1] = {(cuuint64_t)ND * 2};
    cuuint32_t b[2] = {64, 32}, e[2] = {1, 1};
    enc(&tcm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, C, d, st, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  auto k = klk<WIDE, MN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaMemset(d, 0, 148 * 8);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k, ta, tb, K, MV / 256, ND / 256, C, ND, d, epi_mode, tcm, g_rot);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(148);
    cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    int n = 0;
    for (int i = 0; i < 148; ++i)
      if (h[i]) { avg += h[i]; ++n; }
    const double flops = 2.0 * MV * ND * (double)K;
    printf("%s epi%d MV=%d ND=%d K=%d err=%s: %.3f ms  %.0f TFLOP/s  avg cycles per 256x256x64 pair MMA block %.0f\n",
           WIDE ? (MN ? "wide-mn" : "wide") : (MN ? "pair-mn" : "pair"), epi_mode, MV, ND, K, cudaGetErrorString(err), ms, flops / ms / 1e9, avg / (n ? n : 1));
  }
  cudaFree(d);
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  enc = (PFN_encodeTiled)p;
  const int MV = 4 * 8192, ND = 1024, K = 4928;  // 4 backward chunks of G^T, Hc^T (hidden padded to 1024)
  void *A, *B;
  __nv_bfloat16* C;
  cudaMalloc(&A, (size_t)MV * K * 2);
  cudaMalloc(&B, (size_t)ND * K * 2);
  cudaMalloc(&C, (size_t)151552 * 5120 * 2);
  fill_random<<<1024, 256>>>((uint16_t*)A, (size_t)MV * K, 1);
  fill_random<<<1024, 256>>>((uint16_t*)B, (size_t)ND * K, 2);
  cudaDeviceSynchronize();
  // desynchronised operand sharing: each pair starts its k-loop at a different k-block
  g_rot = 1;
  run<0, 1>(A, B, C, MV, 1024, K, 0);
  run<1, 1>(A, B, C, MV, 1024, K, 0);
  run<0>(A, B, C, MV, 1024, K, 0);
  run<1>(A, B, C, MV, 1024, K, 0);
  g_rot = 0;
  return 0;
}
