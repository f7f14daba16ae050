// cce_gemm.cuh -- the tcgen05/TMEM/TMA tile engine behind every contraction of
// the fused linear cross-entropy (arxiv 2601.02609, section "Cut Cross-Entropy",
// P:470-687), with the four epilogues that make it the CCE hot path.
//
// One persistent, warp-specialised kernel per launch (one CTA per SM):
//   warp 0        TMA producer      (one elected lane; 4-stage smem ring, mbarriers)
//   warp 1        MMA issuer        (one lane; tcgen05.mma cta_group::1, M=128 N=256 K=16)
//   warp 2        TMEM allocator    (512 columns = 2 x 256-column fp32 accumulators)
//   warps 4..7    epilogue          (tcgen05.ld 32x32b: thread = one TMEM lane = one tile row)
// Accumulators are double-buffered in TMEM so the epilogue of tile i overlaps the
// MMAs of tile i+1.
//
// Modes (D = A * B^T over a 128 x 256 tile, K in 64-wide blocks):
//   FWD  S = Hc W^T        A = Hc [rows][D]  K-major, B = W [V][D] K-major.
//        Epilogue: per-row online softmax (running max m, sum-exp d over the tile's
//        256 logits, Def. "Online Softmax" P:511-519) and the target logit
//        (Alg. P:545-565 lines 10-11).  Writes (m, d) per (vocab tile, row) and z_y.
//   G    S recomputed for one vocabulary chunk ("compute_chunk_logits"); the
//        epilogue forms G = (dloss/n_valid)(exp(S - lse) - 1[v = y]) in place
//         and stores it as bf16 into the chunk buffer Gbuf [rows][C].
//   DW   dW^T = Hc^T Gbuf    (P:667 grad_W[chunk] += probs^T @ h): M = D (A = Hc,
//        MN-major), N = vocab in chunk (B = Gbuf, MN-major), K = valid rows.
//   DH   dH^T += W_c^T Gbuf^T (P:666 grad_h += probs @ W[chunk]): M = D (A = W chunk,
//        MN-major), N = valid rows (B = Gbuf, K-major), K = vocab in chunk; the
//        epilogue accumulates into the fp32 buffer dH32 across chunks in chunk order.
// Rows are the compacted valid rows (ignored rows are never read).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "sm100.cuh"

namespace cce {

enum GemmMode : int { MODE_FWD = 0, MODE_G = 1, MODE_DW = 2, MODE_DH = 3 };

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_BYTES = BN * BK * 2;  // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int GEMM_THREADS = 128 + 8 * 32;  // 4 control warps + 8 epilogue warps
constexpr int TMEM_COLS = 512;
constexpr int GEMM_SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align slack*/ + 256 /*barriers*/ + 1024 /*xchg*/;
constexpr float LOG2E = 1.4426950408889634f;

struct GemmParams {
  int D;              // hidden size (multiple of 64)
  int V_local;        // vocabulary rows held by this rank
  int Npad;           // rows of the compact buffers
  int c0;             // first local vocabulary row of the chunk (G / DW / DH); 0 for FWD
  int width;          // vocabulary rows covered (V_local for FWD, chunk width otherwise)
  int C;              // row stride (elements) of Gbuf
  int vocab_offset;   // global id of local vocabulary row 0
  const int* n_valid;   // device scalar
  const int* labels_c;  // [Npad] compact labels (global ids)
  float2* part;         // FWD: [ceil(V_local/BN)][Npad] per-tile (m, d)
  float* zy_c;          // FWD: [Npad] target logit (written by the tile that owns y)
  const float* lse_c;   // G: [Npad]
  const float* dloss;   // G: device scalar
  __nv_bfloat16* gbuf;  // G: [Npad][C]
  void* dW;             // DW: [V_local][D] bf16 (or float32 with dw_fp32)
  float* dH32;          // DH: [Npad][D]
  int dh_accumulate;    // DH: 0 = overwrite (first chunk), 1 = add
  // regularised loss (pair / quad kernels only; cce.h cce_config)
  float ls_eps;         // label smoothing eps
  float z_loss;         // z-loss weight lambda
  float inv_vtotal;     // 1 / vocab_total (the mean of the logits runs over the global vocabulary)
  float* zs_part;       // FWD: [ceil(V_local/256)][Npad] per-tile logit sums, or nullptr (eps == 0)
  // reduction / gradient modes (pair / quad kernels only; cce.h CCE_REDUCTION_*, CCE_FLAG_GRAD_*)
  int reduction;        // 0 mean (dloss / n_valid), 1 sum (dloss), 2 none (dloss_c per row)
  const float* dloss_c; // G: reduction "none": per-row upstream gradients (compact rows), else nullptr
  int dw_fp32;          // DW: dW is float32 (else bf16)
  int dw_accumulate;    // DW: dW += gradient (else overwrite)
  // fused AdamW in the dW epilogue (pair kernel only; cce.h cce_backward_adamw,
  // Alg. Fused AdamW P:2003-2046): dW is consumed in registers, W / master / m / v updated
  int adamw;
  float lr, beta1, beta2, eps, wd, bc1, bc2;
  const float* clip_coef;  // device scalar or nullptr (1)
  float* master;           // [V_local][D] fp32 or nullptr (theta = the bf16 W)
  float* am;               // [V_local][D] fp32 first moment
  float* av;               // [V_local][D] fp32 second moment
  const float* grad_in;    // [V_local][D] fp32 earlier micro-batches' gradient or nullptr
  const __nv_bfloat16* Win;  // the forward's W (theta when master == nullptr), row stride ldw
  __nv_bfloat16* Wout;       // bf16(theta_new), row stride ldw: == Win (in place) or a second buffer
  int ldw;
  int adamw_inplace;
  int dbg;                   // debug (env CCE_DBG_G; garbage results): bit 0 skip the dlogits stores,
                             // bit 1 skip the exponentials -- isolates the epilogue's energy cost         // Wout == Win: the chunk's dW epilogue waits for its dH items
};


struct TileGeom {
  int tiles_m, tiles_n, num_kb;
};

template <int MODE>
__device__ __forceinline__ TileGeom tile_geom(const GemmParams& p, int nv) {
  TileGeom g;
  if (MODE == MODE_FWD || MODE == MODE_G) {
    g.tiles_m = (nv + BM - 1) / BM;
    g.tiles_n = (p.width + BN - 1) / BN;
    g.num_kb = p.D / BK;
  } else if (MODE == MODE_DW) {
    g.tiles_m = (p.D + BM - 1) / BM;
    g.tiles_n = (p.width + BN - 1) / BN;
    g.num_kb = (nv + BK - 1) / BK;
  } else {
    g.tiles_m = (p.D + BM - 1) / BM;
    g.tiles_n = (nv + BN - 1) / BN;
    g.num_kb = (p.width + BK - 1) / BK;
  }
  return g;
}

// ------------------------------------------------------------------ epilogues
// 8 epilogue warps: warp w (4..11) reads TMEM lane quarter q = w % 4 (rows
// 32q..32q+31 of the tile) and column half h = (w - 4) / 4 (columns 128h..128h+127).
// Each thread owns one accumulator row of its half.
constexpr int EPI_WARPS = 8;
constexpr int EPI_THREADS = EPI_WARPS * 32;
constexpr int HALF = BN / 2;          // columns per epilogue warp
constexpr int JCH = HALF / 32;        // 32-column chunks per warp

struct EpiCtx {
  int row_in_tile;  // TMEM lane == tile row
  int q, half;
  float* xchg;      // smem scratch [2][128] float2 for the FWD half merge
};

template <int MODE>
__device__ __forceinline__ void epilogue_tile(const GemmParams& p, uint32_t taddr, const EpiCtx& e, int mt, int nt,
                                              int nv, float scale, bool have_acc) {
  const int cbase = e.half * HALF;  // first column of this warp's half
  if (MODE == MODE_FWD) {
    // Per-row online softmax over this half's 128 logits: running max m and sum-exp d
    // (Def. "Online Softmax"), target logit captured when y falls here.
    const int row = mt * BM + e.row_in_tile;
    const bool rv = row < nv;
    // the target only counts on the rank that owns it: a label of the NEXT shard can fall in
    // this shard's padded tail tile (local id in [V_local, 256-aligned)), where the logits are masked
    const int yl = rv ? (p.labels_c[row] - p.vocab_offset) : -1;
    const int y = ((unsigned)yl < (unsigned)p.V_local) ? yl : -1;
    float m = -INFINITY, d = 0.f;
#pragma unroll 1
    for (int j = 0; j < JCH; ++j) {
      float v[32];
      tmem_ld32(taddr + cbase + j * 32, v);
      const int col0 = nt * BN + cbase + j * 32;
      if (col0 >= p.V_local) break;  // warp-uniform: rest of the half is past the vocabulary
      if (col0 + 32 > p.V_local) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (col0 + i >= p.V_local) v[i] = -INFINITY;
      }
      float cmax = v[0];
#pragma unroll
      for (int i = 1; i < 32; ++i) cmax = fmaxf(cmax, v[i]);
      const float mn = fmaxf(m, cmax);
      const float ms = mn * LOG2E;
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        s0 += ex2(fmaf(v[i], LOG2E, -ms));
        s1 += ex2(fmaf(v[i + 1], LOG2E, -ms));
      }
      d = d * ex2((m - mn) * LOG2E) + (s0 + s1);  // first chunk: m = -inf -> ex2(-inf) = 0
      m = mn;
      const unsigned off = (unsigned)(y - col0);
      if (off < 32u) {
        float zy = 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (off == (unsigned)i) zy = v[i];
        p.zy_c[row] = zy;  // exactly one (tile, half, chunk) owns y
      }
    }
    // merge the two halves of the row: half 1 hands (m, d) to half 0 through smem
    float2* x = reinterpret_cast<float2*>(e.xchg);
    if (e.half == 1) x[e.row_in_tile] = make_float2(m, d);
    named_bar_sync(3 + e.q, 64);
    if (e.half == 0) {
      const float2 o = x[e.row_in_tile];
      const float mn = fmaxf(m, o.x);
      const float dd = (d > 0.f ? d * ex2((m - mn) * LOG2E) : 0.f) + (o.y > 0.f ? o.y * ex2((o.x - mn) * LOG2E) : 0.f);
      if (rv) p.part[(size_t)nt * p.Npad + row] = make_float2(mn, dd);
    }
    named_bar_sync(3 + e.q, 64);  // xchg reusable for the next tile
  } else if (MODE == MODE_G) {
    // G = s (exp(S - lse) - 1[v = y]) with s = dloss / n_valid folded into
    // the exponent: s exp(S - lse) = 2^(S log2e - lse log2e + log2 s).  Rows past
    // n_valid use an exponent offset of +inf (-> 0); the vocab tail is masked per chunk.
    const int row = mt * BM + e.row_in_tile;
    const bool rv = row < nv;
    // the target only counts on the rank that owns it: a label of the NEXT shard can fall in
    // this shard's padded tail tile (local id in [V_local, 256-aligned)), where the logits are masked
    const int yl = rv ? (p.labels_c[row] - p.vocab_offset) : -1;
    const int y = ((unsigned)yl < (unsigned)p.V_local) ? yl : -1;
    const float off2 = rv ? (p.lse_c[row] * LOG2E - __log2f(fabsf(scale))) : INFINITY;
    __nv_bfloat16* out = p.gbuf + (size_t)row * p.C + nt * BN + cbase;
#pragma unroll 1
    for (int j = 0; j < JCH; ++j) {
      float v[32];
      tmem_ld32(taddr + cbase + j * 32, v);
      const int lcol0 = nt * BN + cbase + j * 32;  // column within the chunk
      const int col0 = p.c0 + lcol0;               // local vocabulary row
      float g[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) g[i] = ex2(fmaf(v[i], LOG2E, -off2));
      const unsigned toff = (unsigned)(y - col0);
      if (scale < 0.f) {  // warp-uniform: negative upstream gradient
#pragma unroll
        for (int i = 0; i < 32; ++i) g[i] = -g[i];
      }
      if (toff < 32u) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (toff == (unsigned)i) g[i] -= scale;
      }
      if (lcol0 + 32 > p.width) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (lcol0 + i >= p.width) g[i] = 0.f;
      }
      uint4* dst = reinterpret_cast<uint4*>(out + j * 32);
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4)
        dst[q4] = make_uint4(pack_bf16(g[8 * q4], g[8 * q4 + 1]), pack_bf16(g[8 * q4 + 2], g[8 * q4 + 3]),
                             pack_bf16(g[8 * q4 + 4], g[8 * q4 + 5]), pack_bf16(g[8 * q4 + 6], g[8 * q4 + 7]));
    }
  } else if (MODE == MODE_DW) {
    const int dcol = mt * BM + e.row_in_tile;  // hidden index
#pragma unroll 1
    for (int j = 0; j < JCH; ++j) {
      float v[32];
      if (have_acc) {
        tmem_ld32(taddr + cbase + j * 32, v);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
      const int lcol0 = nt * BN + cbase + j * 32;
      if (dcol < p.D) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (lcol0 + i < p.width)
            static_cast<__nv_bfloat16*>(p.dW)[(size_t)(p.c0 + lcol0 + i) * p.D + dcol] = __float2bfloat16_rn(v[i]);
        }
      }
    }
  } else {  // MODE_DH
    // fp32 accumulation across vocabulary chunks in chunk order: load the 32 old
    // values first (independent L2 loads, .cg: another SM wrote them), then store.
    const int dcol = mt * BM + e.row_in_tile;
#pragma unroll 1
    for (int j = 0; j < JCH; ++j) {
      float v[32];
      tmem_ld32(taddr + cbase + j * 32, v);
      const int t0 = nt * BN + cbase + j * 32;
      if (dcol < p.D) {
        float* base = p.dH32 + (size_t)t0 * p.D + dcol;
        if (p.dh_accumulate) {
          float old[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) old[i] = (t0 + i < nv) ? __ldcg(base + (size_t)i * p.D) : 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += old[i];
        }
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (t0 + i < nv) __stcg(base + (size_t)i * p.D, v[i]);
      }
    }
  }
}

// ------------------------------------------------------------------ kernel
template <int MODE>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    cce_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const GemmParams p) {
  constexpr bool A_MN = (MODE == MODE_DW || MODE == MODE_DH);
  constexpr bool B_MN = (MODE == MODE_DW);
  constexpr uint32_t IDESC = idesc_bf16_f32(BM, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  float* xchg = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], EPI_THREADS);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int nv = *p.n_valid;
  const TileGeom g = tile_geom<MODE>(p, nv);
  const int total = g.tiles_m * g.tiles_n;

  if (warp == 0) {
    if (lane == 0 && g.num_kb > 0) {
      // ===== TMA producer =====
      uint32_t stage = 0, phase = 0;
      for (int x = blockIdx.x; x < total; x += gridDim.x) {
        const int mt = x % g.tiles_m, nt = x / g.tiles_m;
        for (int kb = 0; kb < g.num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* a = sA + stage * A_BYTES;
          uint8_t* b = sB + stage * B_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);
          if (MODE == MODE_FWD || MODE == MODE_G) {
            tma_load_2d(&tmA, &full_bar[stage], a, kb * BK, mt * BM);
            tma_load_2d(&tmB, &full_bar[stage], b, kb * BK, p.c0 + nt * BN);
          } else if (MODE == MODE_DW) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d(&tmA, &full_bar[stage], a + j * 8192, mt * BM + j * 64, kb * BK);
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_2d(&tmB, &full_bar[stage], b + j * 8192, nt * BN + j * 64, kb * BK);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_2d(&tmA, &full_bar[stage], a + j * 8192, mt * BM + j * 64, p.c0 + kb * BK);
            tma_load_2d(&tmB, &full_bar[stage], b, kb * BK, nt * BN);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && g.num_kb > 0) {
      // ===== MMA issuer =====
      uint32_t stage = 0, phase = 0;
      int it = 0;
      for (int x = blockIdx.x; x < total; x += gridDim.x, ++it) {
        const uint32_t acc = it & 1, acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < g.num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a = smem_u32(sA + stage * A_BYTES);
          const uint32_t b = smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? sdesc_sw128(a + k * 2048, 8192, 1024) : sdesc_sw128(a + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? sdesc_sw128(b + k * 2048, 8192, 1024) : sdesc_sw128(b + k * 32, 16, 1024);
            umma_bf16(tmem_d, ad, bd, IDESC, (kb > 0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty_bar[stage]);  // frees the smem slot once these MMAs retire
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull_bar[acc]);  // accumulator ready for the epilogue
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue =====
    EpiCtx e;
    e.q = warp & 3;  // TMEM lane quarter accessible to this warp
    e.half = (warp - 4) >> 2;
    e.row_in_tile = e.q * 32 + lane;
    e.xchg = xchg;
    float scale = 0.f;
    if (MODE == MODE_G) scale = nv > 0 ? (*p.dloss) / (float)nv : 0.f;
    int it = 0;
    for (int x = blockIdx.x; x < total; x += gridDim.x, ++it) {
      const int mt = x % g.tiles_m, nt = x / g.tiles_m;
      const uint32_t acc = it & 1, acc_phase = (it >> 1) & 1;
      const bool have_acc = g.num_kb > 0;
      if (have_acc) {
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
      }
      const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)(e.q * 32) << 16);
      epilogue_tile<MODE>(p, taddr, e, mt, nt, nv, scale, have_acc);
      if (have_acc) {
        tc_fence_before();
        mbar_arrive(&tempty_bar[acc]);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, TMEM_COLS);
}

}  // namespace cce
