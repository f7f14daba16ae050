// cce_designb.cuh -- SURVEY 7.3 "design B" (rows a3, a6): the dH numerator accumulated in the
// FORWARD and dlogits kept ON CHIP in the backward.  Opt-in (CCE_FLAG_DESIGN_B); measured
// slower than the default chunked path on B200, kept as the built and
// parity-tested alternative.
//
// Forward (mode 0), one CTA per SM, a unit = (token tile of NX = 64 valid rows, a contiguous
// range of 128-row vocabulary steps).  The token tile Hc_t [64 x D] stays in shared memory;
// per step j (vocabulary rows v0 .. v0 + 127):
//   GEMM1  S^T = W_j Hc_t^T        M = 128 vocabulary rows (TMEM lanes), N = 64 tokens, K = D
//   epilogue: per token t (column): running reference m_t (log2 units, shared by the whole
//          tile), P'[v][t] = 2^(S log2e - m_t) with the TARGET EXCLUDED (P' = 0 at v = y_t,
//          whose logit z_y is captured instead), d_nt[t] += sum_v P' (fp32, per thread),
//          P' -> bf16 into shared memory as the MN-major B operand of
//   GEMM2  O'^T[d][t] += W_j^T P'^T M = D in 128-row blocks (TMEM lanes), N = 64, K = 128
//   This is the FlashAttention-2 output accumulator (Alg. FA2 forward) with
//   K = V = W.  Lazy rescale (FA4 style): m_t moves only when a logit exceeds it by 2^16,
//   then O' columns (TMEM) and d_nt are multiplied by 2^(m_old - m_new) before GEMM2_j.
// At the end of a unit the partial (m, d_nt, z_y, O') of the tile's 64 rows goes to the
// workspace; k_merge_designb combines a row's partials in a fixed order into
//   U_n = (O'_n - d_nt,n W_{y_n}) / d_n,   d_n = d_nt,n + e^{z_y - m}      (SURVEY H5 fix)
// i.e. U = E_p[W] - W_y = dH_n / s, with no cancellation for confident tokens (p_y -> 1).
//
// Backward (mode 1), a unit = a vocabulary tile of NX = 64 rows W_u [64 x D] (shared memory),
// swept over the valid rows in steps of 128:
//   GEMM1  S = Hc_j W_u^T          M = 128 rows (lanes), N = 64 vocabulary, K = D
//   epilogue: G = s (2^(S log2e - lse log2e) - 1[v = y]), bf16 into shared memory
//          only -- dlogits never reach HBM (row a6) --
//   GEMM2  dW_u^T[d][v] += Hc_j^T G  M = D (128-row blocks), N = 64, K = 128
//   and dH = s U is a row scaling of the forward's U (k_scale_rows), no second sweep.
// Executed work: forward 2 + 2 NVD, backward 2 + 2 NVD (the same 8 NVD as the default path);
// no [N x C] dlogits buffer and no fp32 dH reductions.  Why it is slower on B200: both GEMMs
// are N = 64 wide (TMEM holds the [D x 64] fp32 accumulator: 7 x 64 + 64 = 512 columns at
// D = 896), and a tcgen05.mma costs a fixed ~100-145 issue cycles below N = 256
// (scripts/ubench_narrow_n.cu), and W (forward) / Hc (backward) is streamed twice per step.
#pragma once
#include "cce_common.cuh"

namespace cce {
namespace dsb {

constexpr int NX = 64;                 // stationary rows per CTA (tokens / vocabulary rows)
constexpr int YM = 128;                // streamed rows per step
constexpr int NB_MAX = 7;              // D <= 896: 7 blocks of 128 hidden rows
constexpr int D_MAX = NB_MAX * 128;
// ring stage: 128 streamed rows x two 64-wide hidden blocks (32 KB, one 3-D TMA box): two
// K-major k-blocks of GEMM1 or one 128-row hidden block of GEMM2 -- 8 MMAs per commit (a
// commit per 4 MMAs cost ~145 cycles per MMA at N = 64, ~100 at 8; scripts/ubench_narrow_n.cu)
constexpr int STG = 32768;
constexpr int NSTG = 3;
constexpr int XBYTES = NX * D_MAX * 2;         // 112 KB
constexpr int B2BYTES = YM * NX * 2;           // 16 KB, single buffer (GEMM2_{j-1} reads it
                                               // while GEMM1_{j+1} runs; P'_j is written after)
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 128 + 32 * EPI_WARPS;
constexpr int SCRATCH = 128 /*barriers*/ + 3 * 64 * 4 /*m2, fsc, ytile*/ + 4 * 64 * 4 /*wmax / dsum*/;
constexpr int SMEM = XBYTES + B2BYTES + NSTG * STG + SCRATCH + 1024 /*align*/;
static_assert(SMEM <= 232448, "design-B shared memory");
constexpr float THRESH = 16.f;         // log2 headroom before the reference max moves (P' <= 2^16)

struct Params {
  int mode;            // 0 forward, 1 backward
  int D, V_local, vocab_offset, Npad;
  const int* n_valid;
  const int* labels_c;
  float* opart;        // forward: [unit][NX][D] fp32 O' partials (unit = k tiles + t)
  float4* spart;       // forward: [unit][NX] (m natural, d_nt, z_y, -)
  // backward
  const float* lse_c;
  const float* dloss;  // device scalar
  const float* dloss_c;  // reduction "none": per compact row, else nullptr
  int reduction;
  void* dW;
  int dw_fp32, dw_accumulate;
};

// Forward work split: every token tile's vocabulary sweep is cut into K segments of L steps;
// units u = k * tiles + t are handed out round-robin (CTA p: u = p, p + G, ...), so in any
// round the CTAs work on one or two vocabulary segments together and read W through the L2
// (a contiguous per-CTA split scattered the CTAs over the whole vocabulary: 28.8 GB of DRAM
// reads per forward, ncu).  K balances the rounds: the smallest K with the best
// units / (rounds x G) ratio among K tiles <= 6 G.
constexpr int MAX_ROUNDS = 6;
__host__ __device__ __forceinline__ int fwd_splits(int tiles, int ns, int G) {
  if (tiles <= 0) return 1;
  int best = 1;
  float best_eff = -1.f;
  for (int k = 1; k <= ns && (long long)k * tiles <= (long long)MAX_ROUNDS * G; ++k) {
    const int u = k * tiles;
    const int rounds = (u + G - 1) / G;
    const float eff = (float)u / (float)(rounds * G);
    if (eff > best_eff + 1e-3f) { best_eff = eff; best = k; }
  }
  return best;
}
// forward partial slots the workspace must hold for up to `tiles_max` token tiles
__host__ __forceinline__ long long fwd_slots_max(long long tiles_max, int G) {
  return (long long)MAX_ROUNDS * G + tiles_max;
}

__device__ __forceinline__ int fkey(float f) {  // order-preserving float -> int
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float fkey_inv(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }

__global__ void __launch_bounds__(THREADS, 1)
    cce_designb_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmY1,
                       const __grid_constant__ CUtensorMap tmY2, const Params P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sX = smem;
  uint8_t* sB2 = smem + XBYTES;
  uint8_t* sR = sB2 + B2BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sR + NSTG * STG);
  uint64_t* full = bar;                 // [NSTG]
  uint64_t* empty = bar + NSTG;         // [NSTG]
  uint64_t* x_full = bar + 2 * NSTG;
  uint64_t* x_empty = x_full + 1;
  uint64_t* s_full = x_full + 2;
  uint64_t* s_empty = x_full + 3;
  uint64_t* b2_full = x_full + 4;
  uint64_t* b2_empty = x_full + 5;
  uint64_t* a2_full = x_full + 6;
  uint64_t* a2_empty = x_full + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(x_full + 8);
  float* m2 = reinterpret_cast<float*>(sR + NSTG * STG + 128);   // [NX] running reference (log2)
  float* fsc = m2 + NX;                 // [NX] rescale factors of the current step
  int* ytile = reinterpret_cast<int*>(fsc + NX);   // [NX] local target ids of the unit's tokens
  int* wmax = ytile + NX;               // [4][NX] per-quarter column maxima (fkey), rescale path
  float* dsum = reinterpret_cast<float*>(wmax);  // [4][NX] per-quarter d_nt sums, unit end (same space)

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int D = P.D;
  const int nkb = D / BK;               // k-blocks of GEMM1 (two per stage)
  const int ns1 = (nkb + 1) / 2;        // GEMM1 stages
  const int nb = (D + 127) / 128;       // hidden blocks of GEMM2 (2 stages each)
  const int nv = *P.n_valid;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmX); tma_prefetch_desc(&tmY1); tma_prefetch_desc(&tmY2);
    for (int s = 0; s < NSTG; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(x_full, 1); mbar_init(x_empty, 1);
    mbar_init(s_full, 1); mbar_init(s_empty, EPI_WARPS);
    mbar_init(b2_full, EPI_WARPS);
    mbar_init(b2_empty, 1);
    mbar_init(a2_full, 1); mbar_init(a2_empty, EPI_WARPS);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;   // S: columns [0, 64); O' / dW^T block b: [64 + 64 b, 128 + 64 b)

  // ---- the unit sequence (identical in every role) ----
  // forward: units u = k * tiles + t (segment k of token tile t), round-robin over the CTAs
  const int ns_f = (P.V_local + YM - 1) / YM;
  const int tiles = (nv + NX - 1) / NX;
  const int Kf = fwd_splits(tiles, ns_f, gridDim.x);
  const int Lf = (ns_f + Kf - 1) / Kf;
  const int uf = tiles * Kf;
  // backward: vocabulary tiles u = blockIdx.x, blockIdx.x + grid, ...; steps over the valid rows
  const int n_vt = (P.V_local + NX - 1) / NX;
  const int ns_b = (nv + YM - 1) / YM;
  const int n_all = P.mode == 0 ? uf : n_vt;
  const int n_units = n_all > (int)blockIdx.x ? (n_all - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  // backward with no valid rows: no pipeline; the epilogue writes dW = 0 (kept when accumulating)
  const bool empty_bwd = P.mode == 1 && ns_b == 0;
  const int n_pipe = empty_bwd ? 0 : n_units;
  // unit i of this CTA (global unit u = blockIdx.x + i G): stationary rows x0 (token tile /
  // vocabulary tile), steps [s0, s1) (step s covers streamed rows [s YM, s YM + YM)); a forward
  // segment past the vocabulary (K L > ns) is empty and skipped by every role
  auto unit = [&](int i, int& x0, int& s0, int& s1) {
    const int u = (int)blockIdx.x + i * (int)gridDim.x;
    if (P.mode == 0) {
      const int t = u % tiles, k = u / tiles;
      x0 = t * NX;
      s0 = min(k * Lf, ns_f);
      s1 = min(s0 + Lf, ns_f);
    } else {
      x0 = u * NX;
      s0 = 0;
      s1 = ns_b;
    }
  };

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer: the stationary tile, then the ring in MMA order
      uint32_t st = 0, ph = 0;
      auto ring = [&](const CUtensorMap* m, int c1, int c2) {
        mbar_wait(&empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&full[st], STG);
        tma_load_3d(m, &full[st], sR + st * STG, 0, c1, c2);
        if (++st == NSTG) { st = 0; ph ^= 1; }
      };
      int xu = 0;   // units loaded so far
      for (int u = 0; u < n_pipe; ++u) {
        int x0, s0, s1;
        unit(u, x0, s0, s1);
        if (s1 == s0) continue;
        if (xu > 0) mbar_wait(x_empty, (xu - 1) & 1);
        ++xu;
        mbar_arrive_expect_tx(x_full, NX * D * 2);
        tma_load_3d(&tmX, x_full, sX, 0, x0, 0);
        for (int j = s0; j <= s1; ++j) {
          if (j < s1)
            for (int k2 = 0; k2 < ns1; ++k2) ring(&tmY1, j * YM, 2 * k2);          // GEMM1_j: k-blocks 2 k2, 2 k2 + 1
          if (j > s0)
            for (int b = 0; b < nb; ++b) ring(&tmY2, (j - 1) * YM, 2 * b);     // GEMM2_{j-1}: hidden block b
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (whole warp, one elected lane issues)
    uint32_t st = 0, ph = 0;
    int g1 = 0, g2 = 0;   // GEMM1 / GEMM2 steps issued so far (all units)
    const uint32_t idesc1 = idesc_bf16_f32(128, NX, 0, 0);   // A K-major (Y), B K-major (X)
    const uint32_t idesc2 = idesc_bf16_f32(128, NX, 1, 1);   // A MN-major (Y^T), B MN-major (B2)
    const uint32_t xa = smem_u32(sX), ra = smem_u32(sR), b2a = smem_u32(sB2);
    int xu = 0;
    for (int u = 0; u < n_pipe; ++u) {
      int x0, s0, s1;
      unit(u, x0, s0, s1);
      if (s1 == s0) continue;
      const int uu = xu++;
      mbar_wait(x_full, uu & 1);
      for (int j = s0; j <= s1; ++j) {
        if (j < s1) {
          mbar_wait(s_empty, (g1 & 1) ^ 1);   // the epilogue has read S of the previous step
          tc_fence_after();
          for (int k2 = 0; k2 < ns1; ++k2) {
            mbar_wait(&full[st], ph);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
              for (int kh = 0; kh < 2; ++kh) {
                const int k = 2 * k2 + kh;
                if (k < nkb) {
#pragma unroll
                  for (int kk = 0; kk < BK / 16; ++kk)
                    umma_bf16(tmem, sdesc_sw128(ra + st * STG + kh * (YM * 128) + kk * 32, 16, 1024),
                              sdesc_sw128(xa + k * (NX * 128) + kk * 32, 16, 1024), idesc1, (k | kk) ? 1u : 0u);
                }
              }
              umma_commit(&empty[st]);
              if (k2 == ns1 - 1) {
                if (j == s1 - 1) umma_commit(x_empty);
                umma_commit(s_full);
              }
            }
            __syncwarp();
            if (++st == NSTG) { st = 0; ph ^= 1; }
          }
          ++g1;
        }
        if (j > s0) {
          mbar_wait(b2_full, g2 & 1);
          if (j - 1 == s0) mbar_wait(a2_empty, (uu & 1) ^ 1);   // previous unit's accumulator drained
          tc_fence_after();
          for (int b = 0; b < nb; ++b) {
            mbar_wait(&full[st], ph);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < YM / 16; ++kk) {
                // A: 128 hidden rows (two 64-wide MN atoms, 16 KB apart) x 16 streamed rows;
                // B: 16 K-rows of the [128 x 64] interleaved P' / G tile
                const uint64_t ad = sdesc_sw128(ra + st * STG + kk * 2048, YM * 128, 1024);
                const uint64_t bd = sdesc_none(b2a + kk * 2 * 128, 128, 2048);
                umma_bf16(tmem + 64 + 64 * b, ad, bd, idesc2, (j - 1 > s0 || kk) ? 1u : 0u);
              }
              umma_commit(&empty[st]);
              if (b == nb - 1) {
                umma_commit(b2_empty);
                if (j == s1) umma_commit(a2_full);
              }
            }
            __syncwarp();
            if (++st == NSTG) { st = 0; ph ^= 1; }
          }
          ++g2;
        }
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue: warp w reads TMEM lane quarter q (32 lanes) and column half h (32 cols)
    const int q = warp & 3, h = (warp - 4) >> 2;
    const int r = q * 32 + lane;                      // TMEM lane
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int ebar_n = 32 * EPI_WARPS;
    int g1 = 0, g2 = 0;
    float scale_all = 0.f;
    if (P.mode == 1 && nv > 0 && P.reduction != 2) scale_all = P.reduction == 1 ? *P.dloss : (*P.dloss) / (float)nv;
    if (empty_bwd && !P.dw_accumulate) {
      for (int u = 0; u < n_units; ++u) {
        int x0, s0, s1;
        unit(u, x0, s0, s1);
        for (int i = threadIdx.x - 128; i < NX * D; i += ebar_n) {
          const int v = x0 + i / D;
          if (v >= P.V_local) break;
          if (P.dw_fp32) static_cast<float*>(P.dW)[(size_t)v * D + i % D] = 0.f;
          else static_cast<__nv_bfloat16*>(P.dW)[(size_t)v * D + i % D] = __float2bfloat16_rn(0.f);
        }
      }
    }
    int xu = 0;
    for (int u = 0; u < n_pipe; ++u) {
      int x0, s0, s1;
      unit(u, x0, s0, s1);
      if (s1 == s0) continue;
      const int uu = xu++;
      float dpart[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) dpart[c] = 0.f;
      if (P.mode == 0) {
        // unit start: reference maxima unknown (-inf: the first step takes the rescale path),
        // the tile's local target ids
        for (int t = threadIdx.x - 128; t < NX; t += ebar_n) {
          m2[t] = -INFINITY;
          const int row = x0 + t;
          const int yl = row < nv ? P.labels_c[row] - P.vocab_offset : -1;
          ytile[t] = ((unsigned)yl < (unsigned)P.V_local) ? yl : -1;
        }
        named_bar_sync(1, ebar_n);
      }
      const int slot = (int)blockIdx.x + u * (int)gridDim.x;   // the global unit index
      for (int j = s0; j < s1; ++j) {
        mbar_wait(s_full, g1 & 1);
        tc_fence_after();
        uint32_t sv[32];
        {
          uint32_t (&a)[8] = *reinterpret_cast<uint32_t(*)[8]>(&sv[0]);
          uint32_t (&b)[8] = *reinterpret_cast<uint32_t(*)[8]>(&sv[8]);
          uint32_t (&c)[8] = *reinterpret_cast<uint32_t(*)[8]>(&sv[16]);
          uint32_t (&d)[8] = *reinterpret_cast<uint32_t(*)[8]>(&sv[24]);
          tmem_ld8_nowait(tmem + lane_off + 32 * h, a);
          tmem_ld8_nowait(tmem + lane_off + 32 * h + 8, b);
          tmem_ld8_nowait(tmem + lane_off + 32 * h + 16, c);
          tmem_ld8_nowait(tmem + lane_off + 32 * h + 24, d);
          tmem_wait_ld();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_empty);
        ++g1;
        float pv[32];
        if (P.mode == 0) {
          const int v = j * YM + r;                   // local vocabulary row of this lane
          bool viol = false;
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const int t = 32 * h + c;
            float x = __uint_as_float(sv[c]) * LOG2E;
            if (v >= P.V_local) x = -INFINITY;
            if (v == ytile[t]) {                      // the target: captured, excluded from P'
              P.spart[(size_t)slot * NX + t].z = __uint_as_float(sv[c]);
              x = -INFINITY;
            }
            viol |= x > m2[t] + THRESH;
            pv[c] = x;
          }
          if (bar_red_or(1, ebar_n, viol)) {
            // rare path (always at a unit's first step): exact column maxima of this step,
            // new references, rescale of the accumulated O' and d_nt
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const int k = __reduce_max_sync(0xffffffffu, fkey(pv[c]));
              if (lane == 0) wmax[q * NX + 32 * h + c] = k;
            }
            named_bar_sync(1, ebar_n);
            for (int t = threadIdx.x - 128; t < NX; t += ebar_n) {
              int k = wmax[t];
              for (int qq = 1; qq < 4; ++qq) k = max(k, wmax[qq * NX + t]);
              const float cm = fkey_inv(k);
              const float mo = m2[t];
              const float mn = fmaxf(mo, cm);
              fsc[t] = (mo == -INFINITY) ? 0.f : ex2(mo - mn);
              m2[t] = mn;
            }
            named_bar_sync(1, ebar_n);
            if (j > s0) {
              // O' holds GEMM2 of steps s0 .. j-1: wait for the last of them, scale in place
              mbar_wait(b2_empty, (g2 - 1) & 1);
              tc_fence_after();
              for (int b = 0; b < nb; ++b) {
#pragma unroll
                for (int c8 = 0; c8 < 4; ++c8) {
                  uint32_t o[8];
                  const uint32_t ta = tmem + lane_off + 64 + 64 * b + 32 * h + 8 * c8;
                  tmem_ld8_nowait(ta, o);
                  tmem_wait_ld();
#pragma unroll
                  for (int i = 0; i < 8; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * fsc[32 * h + 8 * c8 + i]);
                  tmem_st8(ta, o);
                }
              }
              tmem_wait_st();
              tc_fence_before();
            }
#pragma unroll
            for (int c = 0; c < 32; ++c) dpart[c] *= fsc[32 * h + c];
          }
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const float x = pv[c];
            const float p = (x == -INFINITY) ? 0.f : ex2(x - m2[32 * h + c]);
            dpart[c] += p;
            pv[c] = p;
          }
        } else {
          // backward: lane = valid row, columns = vocabulary rows x0 + 32 h + c
          const int row = j * YM + r;
          const bool rv = row < nv;
          const int yl = rv ? P.labels_c[row] - P.vocab_offset : -1;
          const float lse2 = rv ? P.lse_c[row] * LOG2E : 0.f;
          const float sc = rv ? (P.dloss_c ? P.dloss_c[row] : scale_all) : 0.f;
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const int v = x0 + 32 * h + c;
            float gv = sc * ex2(fmaf(__uint_as_float(sv[c]), LOG2E, -lse2));
            if (v == yl) gv -= sc;
            pv[c] = (rv && v < P.V_local) ? gv : 0.f;
          }
        }
        // P' / G -> the interleaved MN-major B tile: element (k = r, n = 32 h + c) at
        // (n / 8) * 2048 + (r / 8) * 128 + (r % 8) * 16 + (n % 8) * 2
        mbar_wait(b2_empty, (g2 & 1) ^ 1);   // GEMM2 of the previous step is done with the tile
        uint8_t* dst = sB2 + (r >> 3) * 128 + (r & 7) * 16;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          *reinterpret_cast<uint4*>(dst + (4 * h + i) * 2048) =
              make_uint4(pack_bf16(pv[8 * i], pv[8 * i + 1]), pack_bf16(pv[8 * i + 2], pv[8 * i + 3]),
                         pack_bf16(pv[8 * i + 4], pv[8 * i + 5]), pack_bf16(pv[8 * i + 6], pv[8 * i + 7]));
        fence_proxy_async_shared();
        tc_fence_before();   // orders this thread's earlier TMEM stores (rescale) before the arrive
        __syncwarp();
        if (lane == 0) mbar_arrive(b2_full);
        ++g2;
      }
      // ---- unit end: drain the O' / dW^T accumulator
      mbar_wait(a2_full, uu & 1);
      tc_fence_after();
      if (P.mode == 0) {
        // per-token d_nt of this CTA: warp sums, then the 4 quarters in order
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          float s = dpart[c];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == 0) dsum[q * NX + 32 * h + c] = s;
        }
        named_bar_sync(1, ebar_n);
        for (int t = threadIdx.x - 128; t < NX; t += ebar_n) {
          const float dn = ((dsum[t] + dsum[NX + t]) + dsum[2 * NX + t]) + dsum[3 * NX + t];
          float4* sp = P.spart + (size_t)slot * NX + t;
          sp->x = m2[t] * (1.f / LOG2E);   // natural units (the merge uses e^{m_s - m})
          sp->y = dn;
        }
        // O' partial rows: [slot][t][d], d = 128 b + r
        for (int b = 0; b < nb; ++b) {
          const int d = 128 * b + r;
#pragma unroll
          for (int c8 = 0; c8 < 4; ++c8) {
            uint32_t o[8];
            tmem_ld8_nowait(tmem + lane_off + 64 + 64 * b + 32 * h + 8 * c8, o);
            tmem_wait_ld();
            if (d < D) {
#pragma unroll
              for (int i = 0; i < 8; ++i)
                P.opart[((size_t)slot * NX + 32 * h + 8 * c8 + i) * D + d] = __uint_as_float(o[i]);
            }
          }
        }
        named_bar_sync(1, ebar_n);   // dsum / m2 / ytile are rewritten by the next unit
      } else {
        // dW rows x0 + n (n = 32 h + c), hidden d = 128 b + r: lanes are consecutive d
        for (int b = 0; b < nb; ++b) {
          const int d = 128 * b + r;
#pragma unroll
          for (int c8 = 0; c8 < 4; ++c8) {
            uint32_t o[8];
            if (s1 > s0) {
              tmem_ld8_nowait(tmem + lane_off + 64 + 64 * b + 32 * h + 8 * c8, o);
              tmem_wait_ld();
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i) o[i] = 0u;   // no valid rows: dW = 0
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int v = x0 + 32 * h + 8 * c8 + i;
              if (v < P.V_local && d < D) {
                const size_t off = (size_t)v * D + d;
                float g = __uint_as_float(o[i]);
                if (P.dw_fp32) {
                  float* p = static_cast<float*>(P.dW) + off;
                  *p = P.dw_accumulate ? *p + g : g;
                } else {
                  __nv_bfloat16* p = static_cast<__nv_bfloat16*>(P.dW) + off;
                  if (P.dw_accumulate) g += __bfloat162float(*p);
                  *p = __float2bfloat16_rn(g);
                }
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a2_empty);
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, TMEM_COLS);
}

// a4 for design B: one warp per valid row; the row's K partials (units k tiles + t) in
// segment order (fixed -> deterministic), the online-softmax merge of
// (m, d_nt, O'), then
//   stats = (m_f, d, z_y, 0) with d = d_nt e^{m - m_f} + e^{z_y - m_f}   (forward_tail's input)
//   U     = (O' e^{m - m_f} - d_nt e^{m - m_f} W_y) / d
__global__ void __launch_bounds__(256) k_merge_designb(const float* __restrict__ opart, const float4* __restrict__ spart,
                                                       int grid, int V_local, int vocab_offset, int D,
                                                       const int* __restrict__ n_valid,
                                                       const int* __restrict__ labels_c,
                                                       const __nv_bfloat16* __restrict__ W, long long ldw,
                                                       float4* __restrict__ stats, float* __restrict__ U) {
  const int nv = *n_valid;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= nv) return;
  const int ns = (V_local + YM - 1) / YM;
  const int tiles = (nv + NX - 1) / NX;
  const int K = fwd_splits(tiles, ns, grid);
  const int L = (ns + K - 1) / K;
  const int t = row / NX, col = row % NX;
  const int yl = labels_c[row] - vocab_offset;
  // pass 1: the partials' maxima; the target's logit from the segment covering its row
  float m = -INFINITY, zy = 0.f;
  bool have_y = false;
  for (int k = 0; k < K && k * L < ns; ++k) {
    const float4 sp = spart[((size_t)k * tiles + t) * NX + col];
    m = fmaxf(m, sp.x);
    if (yl >= k * L * YM && yl < min((k + 1) * L, ns) * YM) { zy = sp.z; have_y = true; }
  }
  const float mf = have_y ? fmaxf(m, zy) : m;
  // pass 2: d_nt and O' in segment order
  constexpr int PER = D_MAX / 32;  // hidden elements per lane
  float o[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) o[i] = 0.f;
  float dn = 0.f;
  for (int k = 0; k < K && k * L < ns; ++k) {
    const size_t s = (size_t)k * tiles + t;
    const float4 sp = spart[s * NX + col];
    if (sp.x == -INFINITY) continue;   // only masked / target entries in this segment
    const float f = __expf(sp.x - mf);
    dn += sp.y * f;
    const float* orow = opart + (s * NX + col) * (size_t)D;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int d = lane + 32 * i;
      if (d < D) o[i] += orow[d] * f;
    }
  }
  const float dd = dn + (have_y ? __expf(zy - mf) : 0.f);
  if (lane == 0) stats[row] = make_float4(mf, dd, have_y ? zy : 0.f, 0.f);
  const float inv = dd > 0.f ? 1.f / dd : 0.f;
  const __nv_bfloat16* wy = (have_y && (unsigned)yl < (unsigned)V_local) ? W + (size_t)yl * ldw : nullptr;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int d = lane + 32 * i;
    if (d < D) {
      const float w = wy ? __bfloat162float(wy[d]) : 0.f;
      U[(size_t)row * D + d] = (o[i] - dn * w) * inv;
    }
  }
}

// dH32 = s_n U_n for the valid rows (s = dloss / n_valid, dloss, or the per-row upstream
// gradient for reduction "none"); the existing scatter / RMSNorm tail then consumes dH32.
// U is left as the forward wrote it (a second backward of the same forward is valid).
__global__ void k_scale_rows(const float* __restrict__ U, float* __restrict__ dH32, int D,
                             const int* __restrict__ n_valid, const float* __restrict__ dloss,
                             const float* __restrict__ dloss_c, int reduction) {
  const int nv = *n_valid;
  const float s_all = nv > 0 ? (reduction == 1 ? *dloss : (reduction == 0 ? *dloss / (float)nv : 0.f)) : 0.f;
  const long long total = (long long)nv * D;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(i / D);
    dH32[i] = U[i] * (dloss_c ? dloss_c[row] : s_all);
  }
}

}  // namespace dsb
}  // namespace cce
