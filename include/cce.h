/*
 * cce.h -- C ABI of the B200-native fused linear cross-entropy library
 * ("Cut Cross-Entropy", arxiv 2601.02609 "Chronicals", section "Cut
 * Cross-Entropy: Memory-Efficient Loss Computation").
 *
 * The library computes, for hidden states H[N,D] (bf16), an LM-head weight
 * (shard) W[V_local,D] (bf16) and labels y[N] (int32, ignore_index allowed):
 *
 *   z[n,v] = H[n,:] . W[v,:]                       (Alg. "Chunked Cross-Entropy
 *                                                   Forward Pass")
 *   lse_n  = log sum_v exp(z[n,v])                  (Def. Online Softmax / Theorem,
 *                                                   P:511-541; stable form P:3528-3543)
 *   loss   = (1/n_valid) sum_{y_n != ignore} (lse_n - z[n,y_n])
 *                                                  (Def. Cross-Entropy Loss P:243-248;
 *                                                   mean over non-ignored rows P:899)
 *   G[n,v] = (dloss/n_valid) (softmax(z_n)_v - 1[v = y_n])
 *                                                  (Prop. CE Gradient P:254-258;
 *                                                   Thm. CCE Backward P:645-650)
 *   dH = G W,  dW = G^T H                           (Alg. "CCE Triton Backward Kernel",
 *                                                   P:652-670, lines 666-667)
 *
 * without ever allocating an [N x V] buffer (Def. Memory Bottleneck).
 * Readings where the paper is silent or garbled are listed in DESIGN.md.
 *
 * Conventions (all functions):
 *  - Pointers are DEVICE pointers unless the parameter name ends in _host.
 *    bf16 tensors are passed as `void*` to raw 2-byte IEEE bfloat16 storage;
 *    `stream` is a cudaStream_t passed as `void*` (NULL = legacy default stream).
 *  - Layout: H is row-major with row stride `ldh` elements (ldh >= D), W is
 *    row-major with row stride `ldw` (ldw >= D).  dH [N,D] and dW [V_local,D]
 *    outputs are dense row-major (row stride D).  H, W must be 16-byte aligned
 *    and ldh*2, ldw*2 multiples of 16 bytes.  D must be a multiple of 64.
 *  - Ownership: the caller owns every buffer, including `workspace`.  The
 *    handle owns only host-side state (the pointers saved between forward and
 *    backward).  H, W, labels and workspace must stay alive and unmodified
 *    from cce_forward until the matching cce_backward has been enqueued.
 *    The library never allocates device memory on the hot path.
 *  - Errors: host-detectable errors return a status immediately and enqueue
 *    nothing.  Device-detected label errors (a label that is neither
 *    ignore_index nor in [0, vocab_total)) set a device flag in the workspace
 *    and make `loss` NaN; cce_get_error reports the flag of the most recent
 *    forward (it is the only synchronising call besides cce_step_host).
 *  - No host synchronisation inside cce_forward / cce_backward.
 *  - Determinism: outputs are bit-reproducible run to run (no atomics on
 *    outputs, fixed-order reductions).
 *  - Threading: a handle is single-stream and not thread-safe; one
 *    forward/backward pair in flight per handle.  Handles are independent.
 */
#ifndef CCE_H_
#define CCE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cce_handle cce_handle;

typedef enum {
  CCE_OK = 0,
  CCE_ERR_INVALID_VALUE = 1,  /* NULL pointer, N < 0, D <= 0, V_local < 0, ld < D, bad rank/world */
  CCE_ERR_UNSUPPORTED = 2,    /* D % 64 != 0, misaligned pointer/stride, no sm_100 device */
  CCE_ERR_LABEL_RANGE = 3,    /* device-detected, sticky; reported by cce_get_error */
  CCE_ERR_NO_FORWARD = 4,     /* cce_backward without a matching cce_forward on this handle */
  CCE_ERR_WORKSPACE = 5,      /* workspace NULL or smaller than cce_workspace_bytes() */
  CCE_ERR_CUDA = 6,           /* a CUDA runtime/driver call failed */
  CCE_ERR_NCCL = 7            /* NCCL unavailable or an NCCL call failed */
} cce_status;

/* flags */
#define CCE_FLAG_NONE 0u
/* Flag bits 2, 4, 8, 16 and 32 named round-1 A/B kernel variants (per-chunk launches,
 * 1-CTA tiles, 4-CTA multicast clusters), all measured slower than the default CTA-pair
 * kernel and removed; cce_create rejects them (CCE_ERR_INVALID_VALUE), like any unknown bit. */
/* Gradient modes: CCE_FLAG_GRAD_FP32 = dH and dW are float32 arrays;
 * CCE_FLAG_ACCUMULATE = dH += gradient and dW += gradient (micro-batch accumulation
 * into .grad, the paper's 4-8 step accumulation) instead of overwrite.
 * Accumulation adds in fp32 and rounds once (bf16 outputs); ignored rows of dH are
 * left untouched. */
#define CCE_FLAG_GRAD_FP32 64u
#define CCE_FLAG_ACCUMULATE 128u
/* Split-phase combine for vocabulary sharding with the caller's own collectives (world > 1
 * without an NCCL communicator, e.g. torch.distributed or a single process driving several
 * shards): see cce_combine_offsets / cce_forward_finish / cce_backward_finish.  Not with
 * cce_backward_rmsnorm, cce_backward_adamw or cce_step_host (CCE_ERR_UNSUPPORTED). */
#define CCE_FLAG_EXTERNAL_COMBINE 256u
/* Sequence-sharded dH (for sequence-parallel callers): with world P,
 * cce_backward writes only this rank's slice of dH, the original rows
 * [rank S, min(N, (rank + 1) S)) with S = ceil(N / P), as a dense [n_r, D] array; the
 * partial dH of the ranks is reduce-scattered (ncclReduceScatter, half the bytes of the
 * all-reduce) instead of all-reduced.  World 1: the full dH.  Not with
 * cce_backward_rmsnorm (CCE_ERR_UNSUPPORTED). */
#define CCE_FLAG_DH_SEQ_SHARD 512u
/* The sharded exchange over peer memory instead of NCCL: this rank's
 * per-row stats are pushed into every rank's all-ranks array right after the merge (stores
 * over NVLink / to peer memory), and inside the backward kernel, as soon as every rank's
 * dH tile is final, the tile's owner sums it over the ranks (loads from peer memory, rank
 * order) and stores the sum into every rank's reduced array, overlapping the remaining
 * tensor-core work tile by tile; release / acquire flags per step, waits bounded
 * (a peer that never signals makes cce_get_error return CCE_ERR_NCCL and loss NaN instead
 * of hanging).  Needs cce_p2p_attach; world <= 8; not with a communicator,
 * CCE_FLAG_EXTERNAL_COMBINE or CCE_FLAG_DH_SEQ_SHARD.  One backward per forward.  Every rank must
 * own a non-empty shard at world > 1 (cce_forward returns CCE_ERR_UNSUPPORTED for V_local == 0:
 * an empty shard runs no backward kernel, so it could neither flag nor reduce its dH tiles).
 * Forward-only loops are safe: the stats exchange is double-buffered by step parity. */
#define CCE_FLAG_P2P_COMBINE 1024u
/* Design B (rows a3 / a6): the forward also accumulates the dH numerator
 * U_n = E_p[W] - W_{y_n} (online-rescaled like the FlashAttention output accumulator,
 * P:1220-1226, target excluded: (O' - d_nt W_y) / d) and the backward recomputes the logits,
 * keeps the dlogits in shared memory only and contracts them into dW; dH = s U.  Same
 * results as the default path within the stated tolerances; measured 1.58x SLOWER on B200
 * (its GEMMs are N = 64 wide).  D <= 896 (else CCE_ERR_UNSUPPORTED from
 * cce_forward), world 1, no label smoothing / z-loss, not with cce_backward_adamw
 * (CCE_ERR_UNSUPPORTED). */
#define CCE_FLAG_DESIGN_B 2048u

/* Reduction of the per-token losses (cce_config.reduction). */
#define CCE_REDUCTION_MEAN 0  /* loss = sum_valid l_n / n_valid (default) */
#define CCE_REDUCTION_SUM 1   /* loss = sum_valid l_n */
#define CCE_REDUCTION_NONE 2  /* loss[n] = l_n per token (0 for ignored rows); dloss is [N] */

typedef struct {
  int32_t ignore_index;   /* label value that marks a skipped row; -100 in the paper */
  int64_t vocab_total;    /* global vocabulary size V, for the label range check */
  int64_t vocab_offset;   /* first global vocabulary id owned by this rank (0 if unsharded) */
  int32_t rank;           /* this rank, 0 if unsharded */
  int32_t world;          /* number of vocabulary shards (ranks), 1 if unsharded */
  void *nccl_comm;        /* ncclComm_t from cce_nccl_comm_init: required when world > 1; optional with
                           * world == 1 (the collectives then run on one rank: a test of that path) */
  uint32_t flags;         /* CCE_FLAG_* */
  /* Regularised loss, both 0 by default (the paper's CCE kernels
   * apply neither):
   *   label_smoothing eps in [0, 1): Def. Smoothed CE,
   *     l_n = (1-eps)(lse_n - z_y) + eps (lse_n - mean_v z_v)
   *   z_loss lambda >= 0: Def. Z-Loss, added: l_n += lambda lse_n^2
   * and their gradients.  mean_v runs over the GLOBAL
   * vocabulary (vocab_total). */
  float label_smoothing;
  float z_loss;
  /* CCE_REDUCTION_MEAN (default) / SUM / NONE.  With NONE, cce_forward's `loss` is an
   * [N] float32 array and cce_backward's `dloss` an [N] float32 array (the upstream
   * gradient of each token's loss); cce_step_host supports MEAN and SUM only. */
  int32_t reduction;
} cce_config;

/* Fill `cfg` with defaults: ignore_index=-100, vocab_total=0 (must be set),
 * offset 0, rank 0, world 1, no comm, no flags. */
void cce_config_default(cce_config *cfg);

/* Create / destroy a handle.  cce_create validates cfg (vocab_total > 0,
 * 0 <= rank < world, comm present iff world > 1) and queries the current
 * device (must be compute capability 10.x for the sm_100a kernels). */
cce_status cce_create(cce_handle **out, const cce_config *cfg);
cce_status cce_destroy(cce_handle *h);

/* Bytes of device workspace needed for a problem of N rows, D hidden, V_local
 * vocabulary rows on this rank.  O(N*D + N*ceil(V_local/256) + N*chunk); never
 * O(N*V).  Returns 0 for invalid arguments. */
size_t cce_workspace_bytes(const cce_handle *h, int64_t N, int64_t D, int64_t V_local);

/*
 * Forward: mean loss over non-ignored rows, per-row global log-sum-exp.
 *   H      [N, D] bf16, row stride ldh          (hidden states)
 *   W      [V_local, D] bf16, row stride ldw     (this rank's LM-head rows [off, off+V_local))
 *   labels [N] int32, global ids or ignore_index
 *   loss   device float scalar                   (mean over valid rows; 0 if none; NaN on label error;
 *                                                 the sum with CCE_REDUCTION_SUM; with CCE_REDUCTION_NONE
 *                                                 an [N] array of per-token losses, 0 for ignored rows)
 *   lse    [N] device float, may be NULL         (global LSE; 0.0f for ignored rows)
 *   n_valid device int32 scalar, may be NULL     (number of non-ignored rows)
 * World > 1: every rank passes the same H/labels and its own W shard; loss
 * and lse come out identical on every rank (NCCL allgather of per-row
 * (max, sum-exp, target-logit) partials, merged in rank order).
 */
cce_status cce_forward(cce_handle *h,
                       const void *H, int64_t N, int64_t D, int64_t ldh,
                       const void *W, int64_t V_local, int64_t ldw,
                       const int32_t *labels,
                       float *loss, float *lse, int32_t *n_valid,
                       void *workspace, size_t workspace_bytes, void *stream);

/*
 * Backward of the mean loss w.r.t. H and this rank's W shard.
 *   dloss  device float scalar, the upstream gradient of `loss` ([N] array with
 *          CCE_REDUCTION_NONE: the gradient of each token's loss)
 *   dH     [N, D] bf16 output (float32 with CCE_FLAG_GRAD_FP32), overwritten; ignored
 *          rows are written as 0 (with CCE_FLAG_ACCUMULATE: dH += gradient, ignored rows
 *          untouched) (world > 1: the full dH, summed over ranks by NCCL all-reduce)
 *   dW     [V_local, D] bf16 output (float32 with CCE_FLAG_GRAD_FP32), overwritten or,
 *          with CCE_FLAG_ACCUMULATE, accumulated (stays local to the rank)
 * Uses the inputs and workspace saved by the last cce_forward on `h`.
 */
cce_status cce_backward(cce_handle *h, const float *dloss, void *dH, void *dW, void *stream);

/*
 * RMSNorm prologue (the step before the path).  The forward takes
 * the un-normalised final hidden states X [N, D] (bf16, row stride ldx) and the scale
 * gamma [D] (bf16) and runs the path on H = bf16(RMSNorm(X)), Def. RMSNorm:
 *   rstd_n = 1 / sqrt((1/D) sum_i X[n,i]^2 + eps),  H[n,i] = (X[n,i] rstd_n) gamma_i
 * in fp32 (Alg. Fused RMSNorm Forward), fused into the gather of the valid
 * rows (ignored rows are never read) with rstd cached in the workspace ("Cache rstd for
 * backward").  eps > 0 (else CCE_ERR_INVALID_VALUE: an all-zero row would give rstd = inf); D <= 8192; gamma 16-byte aligned.  Other arguments and
 * outputs as cce_forward.  X and gamma must stay alive and unmodified until the matching
 * backward has been enqueued.
 */
cce_status cce_forward_rmsnorm(cce_handle *h,
                               const void *X, int64_t N, int64_t D, int64_t ldx,
                               const void *gamma, float eps,
                               const void *W, int64_t V_local, int64_t ldw,
                               const int32_t *labels,
                               float *loss, float *lse, int32_t *n_valid,
                               void *workspace, size_t workspace_bytes, void *stream);

/*
 * Backward through the loss AND the RMSNorm prologue, from the unrounded fp32 dH
 * (never rounded to bf16 in between).  With xbar = X rstd and g = dL/dH (DESIGN.md
 * reading R18: the exact gradient of Def. RMSNorm; the paper's Prop. P:227-233 and
 * Alg. P:737-746 are garbled):
 *   dX[n,k]   = rstd_n (gamma_k g[n,k] - xbar[n,k] (1/D) sum_i g[n,i] gamma_i xbar[n,i])
 *   dgamma[k] = sum_{valid n} g[n,k] xbar[n,k]                        (Alg. P:745)
 *   dX     [N, D] bf16 (float32 with CCE_FLAG_GRAD_FP32), dense; ignored rows 0
 *   dgamma [D] bf16 (float32 with CCE_FLAG_GRAD_FP32)
 *   dW     as cce_backward
 * CCE_FLAG_ACCUMULATE adds into dX / dgamma / dW (ignored rows of dX untouched).
 * Deterministic (fixed-order reductions).  Requires that the last forward on `h` was
 * cce_forward_rmsnorm (else CCE_ERR_NO_FORWARD).
 */
cce_status cce_backward_rmsnorm(cce_handle *h, const float *dloss, void *dX, void *dgamma, void *dW, void *stream);

/*
 * Fused AdamW.  The update is the paper's fused kernel,
 * Alg. "Fused AdamW Triton Kernel (Complete)", which is Def. AdamW
 * with a pre-computed clipping coefficient, per element:
 *   g  = (grad_in + grad) * clip_coef
 *   th = th * (1 - lr * weight_decay)              decoupled weight decay
 *   m  = beta1 m + (1 - beta1) g ;  v = beta2 v + (1 - beta2) g^2
 *   th = th - lr * (m / bias_correction1) / (sqrt(v / bias_correction2) + eps)
 * in float32.  bias_correction_i = 1 - beta_i^t is computed by the caller from its
 * host step counter (no device sync).
 *   master  [n] float32 master weights (row stride D for the fused backward), or NULL:
 *           then the bf16 weights themselves are theta (read, updated, rounded back)
 *   m, v    [n] float32 moments (same layout as master), updated in place; required
 *   grad_in [n] float32 gradient accumulated over earlier micro-batches,
 *           added to this step's gradient; NULL = none
 *   clip_coef device float scalar min(1, max_norm / global_norm), or NULL = 1.
 *           Global-norm clipping needs the norm of the whole gradient before any update,
 *           so a fused step takes the coefficient as an input (the caller's norm pass)
 * All pointers are device pointers owned by the caller.
 */
typedef struct {
  float lr, beta1, beta2, eps, weight_decay;
  float bias_correction1, bias_correction2;
  const float *clip_coef;
  float *master;
  float *m;
  float *v;
  const float *grad_in;
  void *W_out;  /* bf16 [V_local, D] with W's row stride: receives bf16(theta_new); NULL = W itself
                 * (in place).  A second buffer (weights double-buffered across steps) lets the
                 * fused backward skip the wait described below */
} cce_adamw_params;

/*
 * Backward with the optimizer step fused into the dW epilogue: when a
 * vocabulary-stationary tile of dW = G^T H is complete in TMEM, the epilogue
 * applies AdamW to those rows of W (and master / m / v) directly, so dW never
 * goes to HBM (saves the dW write and re-read, and the optimizer launch).  dH as
 * in cce_backward.  W is the buffer passed to the last cce_forward on `h`.  With
 * opt->W_out == NULL it is UPDATED IN PLACE (bf16(theta_new)) and must be writable:
 * the epilogue of a chunk's dW tiles then waits until that chunk's dH tiles (which
 * read W) are complete, so the update never races the backward's own reads.  With
 * opt->W_out a distinct buffer (same shape and row stride as W), W is only read.
 * CCE_FLAG_ACCUMULATE returns CCE_ERR_UNSUPPORTED.  opt->m / opt->v NULL -> CCE_ERR_INVALID_VALUE.
 *
 * MEASURED SLOWER than the unfused pair on B200: at the Qwen2.5-0.5B head the fused step adds
 * +1.54 ms (in place) / +1.64 ms (W_out) to forward + backward, cce_backward (fp32 dW) +
 * cce_adamw_step adds +0.84 ms (the DW epilogues cannot keep the optimizer's
 * 26 B per element in flight while the backward runs).  Kept as a correct, parity-tested
 * entry point; the recommended optimizer path is cce_backward + cce_adamw_step.
 */
cce_status cce_backward_adamw(cce_handle *h, const float *dloss, void *dH, const cce_adamw_params *opt,
                              void *stream);

/*
 * Standalone fused AdamW over n elements (the paper's one-kernel optimizer step,
 * P:2003-2046; also the unfused baseline for cce_backward_adamw): grad is [n]
 * bf16 (grad_fp32 = 0) or float32 (grad_fp32 = 1), may be NULL (zero gradient:
 * decay and moment decay only); W_bf16 [n] bf16 receives bf16(theta_new) and is
 * theta itself when opt->master is NULL (W_bf16 may be NULL only if master is set).
 * HBM-bound: one read and one write of each state array.
 */
cce_status cce_adamw_step(const cce_adamw_params *opt, const void *grad, int32_t grad_fp32, int64_t n,
                          void *W_bf16, void *stream);

/*
 * Split-phase combine (CCE_FLAG_EXTERNAL_COMBINE; SURVEY 8(e) rows a9 / a10 done by the
 * caller).  cce_forward then stops after this rank's per-row partial statistics; the
 * caller gathers them from every rank into the all-ranks array (rank-major) and calls
 * cce_forward_finish, which merges them in rank order into the global LSE / loss exactly
 * like the NCCL path.  cce_backward stops with this rank's partial dH (fp32, compact valid
 * rows); the caller replaces it with the sum over ranks and calls cce_backward_finish,
 * which writes dH.  dW is complete after cce_backward.
 * cce_combine_offsets: byte offsets inside the workspace for a problem (N, D, V_local):
 *   out4[0] this rank's stats   float [Npad][4]          (m, d, z_y, sum of logits)
 *   out4[1] all ranks' stats    float [world][Npad][4]
 *   out4[2] partial dH          float [Npad][D] compact valid rows; with
 *                               CCE_FLAG_DH_SEQ_SHARD float [P S][D] in original row order,
 *                               to be reduce-scattered: rank r's summed slice (S rows) goes
 *                               at row r S of its own array before cce_backward_finish
 *   out4[3] Npad (rows of those arrays; rows >= n_valid are ignored)
 * The finish calls return CCE_ERR_NO_FORWARD without a pending phase.
 */
cce_status cce_combine_offsets(const cce_handle *h, int64_t N, int64_t D, int64_t V_local, int64_t *out4);
cce_status cce_forward_finish(cce_handle *h, void *stream);
cce_status cce_backward_finish(cce_handle *h, void *stream);

/* Synchronises `stream` and returns CCE_ERR_LABEL_RANGE if the most recent
 * cce_forward on this handle saw an out-of-range label (the offending rows are
 * treated as ignored and loss is NaN), else CCE_OK.  Clears the flag. */
cce_status cce_get_error(cce_handle *h, void *stream);

/*
 * End-to-end step with HOST inputs: copies H_host [N,D] (dense, pinned
 * recommended) and labels_host [N] to the device, runs forward + backward
 * with dloss = 1, copies the loss back to *loss_host and synchronises
 * `stream`.  W, dH, dW, the device staging buffer `dev_inputs` (at least
 * cce_host_staging_bytes(N, D) bytes) and workspace are device memory.
 */
size_t cce_host_staging_bytes(int64_t N, int64_t D);
cce_status cce_step_host(cce_handle *h,
                         const void *H_host, int64_t N, int64_t D,
                         const int32_t *labels_host,
                         const void *W, int64_t V_local, int64_t ldw,
                         float *loss_host, void *dH, void *dW,
                         void *dev_inputs, size_t dev_inputs_bytes,
                         void *workspace, size_t workspace_bytes, void *stream);

/*
 * cce_step_host without the final synchronisation, for a training loop that keeps the
 * next batch's upload in flight (the paper's zero-sync principle): the
 * H2D copies run on `copy_stream` (NULL or equal to `stream`: no overlap) after the
 * previous step that used the same `dev_inputs` buffer has finished with it, the compute
 * waits for them on `stream`, and the loss is copied to `loss_host` (pinned memory) at
 * the end of the step on `stream`.  Rotate two (at most four) staging buffers so step i+1's
 * copy overlaps step i's compute; synchronise `stream` before reading loss_host.
 */
cce_status cce_step_host_async(cce_handle *h,
                               const void *H_host, int64_t N, int64_t D,
                               const int32_t *labels_host,
                               const void *W, int64_t V_local, int64_t ldw,
                               float *loss_host, void *dH, void *dW,
                               void *dev_inputs, size_t dev_inputs_bytes,
                               void *workspace, size_t workspace_bytes, void *stream, void *copy_stream);

/*
 * Peer-memory setup for CCE_FLAG_P2P_COMBINE.  cce_p2p_export: the CUDA IPC handle
 * (CCE_P2P_HANDLE_BYTES bytes, written to host memory) of the allocation holding
 * `dev_ptr`, and dev_ptr's byte offset inside it.  Each rank exports its workspace, the
 * caller all-gathers (handle, offset) (e.g. torch.distributed), and every rank calls
 * cce_p2p_attach with the arrays indexed by rank (its own entry is ignored), the
 * workspace it will pass to cce_forward and the problem's N, D (later steps must use the
 * same N, D: the flag arrays are laid out for them); attach zeroes this rank's flags, so all ranks
 * must attach before any rank's first step (a barrier).  The workspace must stay the same
 * buffer afterwards (cce_forward returns CCE_ERR_INVALID_VALUE otherwise); the mappings
 * are closed by cce_destroy.
 */
#define CCE_P2P_HANDLE_BYTES 64
cce_status cce_p2p_export(const void *dev_ptr, void *handle_out, int64_t *offset_out);
cce_status cce_p2p_attach(cce_handle *h, void *workspace, int64_t N, int64_t D, const void *handles,
                          const int64_t *offsets);

/*
 * One-GPU emulation of the peer-memory exchange, for testing where there are fewer GPUs than
 * ranks: `world` handles (CCE_FLAG_P2P_COMBINE, cfg.rank == index, cfg.world == world) in ONE
 * process on ONE device, hs[r] using workspaces[r] (device pointers; no IPC).  Ranks whose
 * kernels wait on one another must not be separate launches time-sliced on one GPU (nothing
 * makes them run at the same time; B200_PROFILING.md reports Xid 109 for such processes), so
 * the group defers: cce_forward on ranks 0 .. world-2 pushes and signals only, and the last
 * rank's cce_forward runs every rank's wait + finalize; cce_backward on ranks 0 .. world-2
 * prepares the launch only, and the last rank's cce_backward issues ONE backward launch in
 * which CTA pairs [r p, (r + 1) p) run rank r's queue (p = (SMs / 2) / world; the RED items
 * reduce across the co-resident rank groups), then every rank's tail.  So call the forwards of
 * ranks 0 .. world-1 in order on one stream, then the backwards in order on the same stream
 * (CCE_ERR_NO_FORWARD otherwise).  Same kernels and arithmetic as cce_p2p_attach.  Destroy the
 * handles together: once one member is destroyed, the others return CCE_ERR_INVALID_VALUE from
 * cce_forward / cce_backward.
 */
cce_status cce_p2p_attach_group(cce_handle *const *hs, void *const *workspaces, int32_t world, int64_t N, int64_t D);

/* NCCL plumbing for world > 1 (NCCL is resolved at run time with dlopen; the
 * library does not link it).  The 128-byte unique id is produced on rank 0 and
 * broadcast by the caller (e.g. over torch.distributed). */
cce_status cce_nccl_unique_id(void *id_out_128_bytes_host);
cce_status cce_nccl_comm_init(void **comm_out, int32_t world, const void *id_128_bytes_host, int32_t rank);
cce_status cce_nccl_comm_destroy(void *comm);

/* Human-readable status. */
const char *cce_status_string(cce_status s);

/* Optional per-kernel-class timing for roofline reporting.  When enabled, every
 * kernel the handle launches is bracketed by CUDA events on its stream (no host
 * sync).  cce_profile_read synchronises on the recorded events and returns, per
 * class, the summed device milliseconds and launch counts, then (if reset != 0)
 * clears the record.  Classes: 0 forward logit GEMM (a1+a2), 1 backward
 * recompute + dlogits GEMM (a5+a6), 2 dW GEMM (a7), 3 dH GEMM (a8), 4 all
 * other (label scan, gather, merges, loss, scatter). */
#define CCE_PROF_CLASSES 5
cce_status cce_profile_enable(cce_handle *h, int32_t on);
cce_status cce_profile_read(cce_handle *h, double *ms_out, int64_t *launches_out, int32_t reset);

/* Debug: record a per-work-item timeline of the persistent kernels into the
 * device buffer `dev_buf`: the first half holds backward items, the second half
 * forward items, 128 bytes per queue entry: {queue<<32|type<<16|chunk, smid,
 * t_dequeue, t_deps_ready, t_epilogue_begin, t_epilogue_end, m0<<32|n0,
 * num_kblocks, t_first_tma, t_last_tma, t_first_mma, t_last_mma,
 * ns_waiting_on_full_barriers, 0, 0, 0} (globaltimer ns; pair kernels fill all
 * fields).  bytes = 0 disables.  Caller owns the buffer. */
cce_status cce_debug_trace(cce_handle *h, void *dev_buf, size_t bytes);

/* Library introspection: number of kernels launched by this handle so far
 * (forward + backward), for the bench's launch count; build string. */
int64_t cce_kernel_launches(const cce_handle *h);
const char *cce_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* CCE_H_ */
