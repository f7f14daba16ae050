// Microbenchmark: does shared-memory traffic from other warps slow tcgen05.mma?  And do
// MN-major operands cost more than K-major ones?
//   pair (cta_group::2) M = 256, N = 256, K = 16, 8 MMAs per commit (the pair kernel's stage),
//   operands resident in shared memory; while the leader issues MMAs, `nw` other warps per CTA
//   stream 16-byte st.shared (and optionally ld.shared) over a separate 32 KB region, as the
//   dlogits epilogue stages its tiles.  Prints cycles per 64-wide k-block (tensor floor 512) and
//   the shared-memory bytes per cycle the other warps moved.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/ubench_smem_contention scripts/ubench_smem_contention.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2601_02609_b200/csrc/sm100.cuh"
using namespace cce;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

template <int AMN, int BMN>
__global__ void __launch_bounds__(384, 1) kc(int iters, int nw, int mode, unsigned long long* out,
                                           unsigned long long* bytes_out, const uint8_t* gsrc, int fill) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[8];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(&slot, 512);
  tc_fence_before();
  cluster_sync_all();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  __shared__ uint64_t fbar[2];
  if (fill && warp == 3 && lane == 0) {
    // TMA-like operand fills: 32 KB bulk copies from L2-resident global memory into a 64 KB
    // region (two alternating halves), as the pair kernel's producer loads 32 KB per k-block
    mbar_init(&fbar[0], 1);
    mbar_init(&fbar[1], 1);
    fence_barrier_init();
    uint32_t ph[2] = {0, 0};
    unsigned long long nb = 0;
    const unsigned long long t0 = clock64();
    const uint32_t dst0 = smem_u32(smem + 131072 + 32768);  // beyond the noise region
    while (clock64() - t0 < (unsigned long long)iters * 980ull) {  // two 32 KB copies in flight
      const int hb = (int)(nb & 1);
      if (nb >= 2) { mbar_wait(&fbar[hb], ph[hb]); ph[hb] ^= 1; }
      mbar_arrive_expect_tx(&fbar[hb], 32768);
      bulk_g2s(dst0 + (uint32_t)(hb * 32768), gsrc + ((blockIdx.x * 7 + nb) & 63) * 32768, 32768, smem_u32(&fbar[hb]));
      ++nb;
    }
    for (int hb = 0; hb < 2; ++hb) if (nb > (unsigned long long)hb) mbar_wait(&fbar[hb], ph[hb]);
    atomicAdd(bytes_out + 296 + blockIdx.x, nb * 32768);
    atomicAdd(bytes_out + 444 + blockIdx.x, clock64() - t0);
  }
  if (warp == 0) {
    if (lane == 0 && rank == 0) {
      const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
      const uint32_t idesc = idesc_bf16_f32(256, 256, AMN, BMN);
      uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      const unsigned long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        const int s = it & 7;
        if (it >= 8) { mbar_wait(&bar[s], ph[s]); ph[s] ^= 1; }
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t ad = AMN ? sdesc_sw128(a + (s & 1) * 32768 + (k & 3) * 2048, 8192, 1024)
                                  : sdesc_sw128(a + (s & 1) * 16384 + (k & 3) * 32, 16, 1024);
          const uint64_t bd = BMN ? sdesc_sw128(b + (s & 1) * 32768 + (k & 3) * 2048, 8192, 1024)
                                  : sdesc_sw128(b + (s & 1) * 16384 + (k & 3) * 32, 16, 1024);
          umma_bf16_pair(tmem + (it & 1) * 256, ad, bd, idesc, k > 0 ? 1u : 0u);
        }
        umma_commit_pair(&bar[s]);
      }
      for (int s = 0; s < 8; ++s) mbar_wait(&bar[s], ph[s]);
      out[blockIdx.x] = clock64() - t0;
    }
    __syncwarp();
  } else if (mode >= 3 && warp == nw) {
    // one noise warp on warp `nw` (SMSP nw % 4): mode 3 = independent FFMA chains (ALU issue
    // pressure, no memory), mode 4 = ex2 (MUFU), mode 5 = 16-byte st.shared bursts
    float x0 = lane, x1 = lane + 1, x2 = lane + 2, x3 = lane + 3;
    uint4* reg = reinterpret_cast<uint4*>(smem + 131072) + 256;
    unsigned long long n = 0;
    const unsigned long long t0 = clock64();
    while (true) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (mode == 3) {
          x0 = fmaf(x0, 1.0001f, 0.5f); x1 = fmaf(x1, 1.0001f, 0.5f); x2 = fmaf(x2, 1.0001f, 0.5f); x3 = fmaf(x3, 1.0001f, 0.5f);
        } else if (mode == 4) {
          x0 = ex2(x0 * 1e-3f); x1 = ex2(x1 * 1e-3f); x2 = ex2(x2 * 1e-3f); x3 = ex2(x3 * 1e-3f);
        } else {
          reg[(r * 32 + lane) & 255] = make_uint4(__float_as_uint(x0), r, lane, 0);
        }
      }
      n += 16;
      if ((n & 255) == 0 && clock64() - t0 > (unsigned long long)iters * 980ull) break;
    }
    if (lane == 0) atomicAdd(bytes_out + 148 + blockIdx.x, clock64() - t0);
    if (x0 + x1 + x2 + x3 == 12345.f) reg[0] = make_uint4(1, 2, 3, 4);
  } else if (mode < 3 && warp >= 4 && warp < 4 + nw) {
    // shared-memory traffic: 16-byte stores (mode 1), stores + loads (mode 2), to a 32 KB region
    uint4* reg = reinterpret_cast<uint4*>(smem + 131072) + (warp - 4) * 256;  // 4 KB per warp
    unsigned long long n = 0;
    uint4 acc = make_uint4(lane, 0, 0, 0);
    const unsigned long long t0 = clock64();
    while (true) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int i = (r * 32 + lane) ^ (lane & 7);
        reg[i] = acc;
        if (mode == 2) {
          const uint4 v = reg[(i + 32) & 255];
          acc.x += v.x;
        }
      }
      n += 8;
      if ((n & 255) == 0 && clock64() - t0 > (unsigned long long)iters * 980ull) break;  // ~ the MMA loop's length
    }
    if (lane == 0) atomicAdd(bytes_out + blockIdx.x, n * 32 * 16 * (mode == 2 ? 2 : 1));
    if (lane == 0 && warp == 4) atomicAdd(bytes_out + 148 + blockIdx.x, clock64() - t0);
    if (acc.x == 0xdeadbeef) reg[0] = acc;
  }
  __syncthreads();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair(tmem, 512);
}

static uint8_t* g_src = nullptr;
template <int AMN, int BMN>
void run(int nw, int mode, int iters, int fill = 0) {
  const int grid = 148;
  unsigned long long *d, *bts;
  if (!g_src) { cudaMalloc(&g_src, 64 * 32768); cudaMemset(g_src, 1, 64 * 32768); }
  cudaMalloc(&d, grid * 8);
  cudaMalloc(&bts, 4 * grid * 8);
  cudaMemset(bts, 0, 4 * grid * 8);
  auto k = kc<AMN, BMN>;
  const int sm = 228 * 1024 - 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = sm;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, iters, nw, mode, d, bts, (const uint8_t*)g_src, fill);
  cudaMemset(bts, 0, 4 * grid * 8);
  cudaLaunchKernelEx(&cfg, k, iters, nw, mode, d, bts, (const uint8_t*)g_src, fill);
  cudaError_t err = cudaDeviceSynchronize();
  unsigned long long h[256], hb[1024];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hb, bts, 4 * grid * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < grid; i += 2) mx = h[i] > mx ? h[i] : mx;
  const double per_kb = (double)mx / iters / 2;
  static const char* names[6] = {"", "st   ", "st+ld", "ffma ", "ex2  ", "sts  "};
  printf("A_%s B_%s other warps %d mode %s fill %d err=%s: cycles per 64-k-block %.1f (floor 512); other-warp smem traffic %.1f B/clk/SM; fills %.1f B/clk/SM\n",
         AMN ? "MN" : "K ", BMN ? "MN" : "K ", nw, names[mode], fill, cudaGetErrorString(err), per_kb,
         nw && hb[148] ? (double)hb[0] / (double)hb[148] : 0.0, fill && hb[444] ? (double)hb[296] / (double)hb[444] : 0.0);
  cudaFree(d);
  cudaFree(bts);
}

int main() {
  const int it = 20000;
  run<0, 0>(0, 1, it); run<1, 0>(0, 1, it); run<0, 1>(0, 1, it); run<1, 1>(0, 1, it);
  for (int nw : {1, 2, 4, 8}) run<0, 0>(nw, 1, it);
  for (int nw : {1, 2, 4, 8}) run<0, 0>(nw, 2, it);
  run<1, 1>(4, 1, it);
  // one noise warp on each SMSP (warp 4..7; the MMA issuer is warp 0 = SMSP 0): ALU, MUFU, st.shared
  for (int mode : {3, 4, 5})
    for (int w : {4, 5, 6, 7}) run<0, 0>(w, mode, it);
  // with TMA-like operand fills streaming into shared memory (warp 3): alone, and with st.shared
  // bursts from warps on the OTHER SMSPs (not the issuer's)
  run<0, 0>(0, 1, it, 1);
  for (int w : {5, 6, 7}) run<0, 0>(w, 5, it, 1);
  return 0;
}
