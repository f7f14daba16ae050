// cce_common.cuh -- parameters and small device helpers shared by the CCE kernels
// (arxiv 2601.02609, section "Cut Cross-Entropy").
//
// The contractions of the hot path:
//   FWD  S = Hc W^T over (row tile, vocabulary tile); epilogue: per-row online softmax
//        (running max m, sum-exp d, Def. "Online Softmax" P:511-519) and the target
//        logit (Alg. P:545-565 lines 10-11) -> per-(vocabulary tile, row) partials.
//   G    S recomputed for one vocabulary chunk ("compute_chunk_logits"); the
//        epilogue forms G = (dloss/n_valid)(exp(S - lse) - 1[v = y]), bf16.
//   DW   dW_c = G_c^T Hc   (P:667 grad_W[chunk] += probs^T @ h).
//   DH   dH  += G_c W_c    (P:666 grad_h += probs @ W[chunk]), fp32 in chunk order.
// Rows are the compacted valid rows (ignored rows are never read).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "sm100.cuh"

namespace cce {

constexpr int BN = 256;          // vocabulary tile of the forward partials (Tv = ceil(V / BN))
constexpr int BK = 64;           // k-block (one 128-byte swizzle atom of bf16)
constexpr int TMEM_COLS = 512;
#ifndef CCE_SLOTS
#define CCE_SLOTS 3
#endif
constexpr int GBUF_SLOTS = CCE_SLOTS;  // ring of chunk dlogits buffers: G(c) reuses the slot of chunk c-SLOTS
constexpr float LOG2E = 1.4426950408889634f;

struct GemmParams {
  int D;              // hidden size (multiple of 64)
  int V_local;        // vocabulary rows held by this rank
  int Npad;           // rows of the compact buffers
  int C;              // vocabulary rows per backward chunk
  int vocab_offset;   // global id of local vocabulary row 0
  const int* n_valid;   // device scalar
  const int* labels_c;  // [Npad] compact labels (global ids)
  float2* part;         // FWD: [ceil(V_local/BN)][Npad] per-tile (m, d)
  float* zy_c;          // FWD: [Npad] target logit (written by the tile that owns y)
  const float* lse_c;   // G: [Npad]
  const float* dloss;   // G: device scalar
  __nv_bfloat16* gbuf;  // G: dlogits ring [slot][C/64][Npad][64]
  void* dW;             // DW: [V_local][D] bf16 (or float32 with dw_fp32)
  float* dH32;          // DH: [Npad][D]
  // regularised loss (cce.h cce_config)
  float ls_eps;         // label smoothing eps
  float z_loss;         // z-loss weight lambda
  float inv_vtotal;     // 1 / vocab_total (the mean of the logits runs over the global vocabulary)
  float* zs_part;       // FWD: [ceil(V_local/256)][Npad] per-tile logit sums, or nullptr (eps == 0)
  // reduction / gradient modes (cce.h CCE_REDUCTION_*, CCE_FLAG_GRAD_*)
  int reduction;        // 0 mean (dloss / n_valid), 1 sum (dloss), 2 none (dloss_c per row)
  const float* dloss_c; // G: reduction "none": per-row upstream gradients (compact rows), else nullptr
  int dw_fp32;          // DW: dW is float32 (else bf16)
  int dw_accumulate;    // DW: dW += gradient (else overwrite)
  // fused AdamW in the dW epilogue (cce.h cce_backward_adamw, Alg. Fused AdamW P:2003-2046):
  // dW is consumed in registers, W / master / m / v updated
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
  int adamw_inplace;         // Wout == Win: the chunk's dW epilogue waits for its dH items
};

// Optional per-item trace record (cce_debug_trace; measurement only, off unless a buffer
// is registered): 16 x u64 per queue position.
struct TraceRec {
  unsigned long long q_type_c, smid, t_deq, t_ready, t_epi0, t_epi1, tile, pad;
  unsigned long long t_load0, t_load1, t_mma0, t_mma1, t_full_wait, r0, r1, r2;
};
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_ge(const int* p, int target) {
  while (ld_acquire(p) < target) __nanosleep(100);
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

}  // namespace cce
