// cce_aux.cuh -- the non-GEMM steps of the CCE hot path (SURVEY 8a rows a0, a4,
// a8-scatter): label scan + compaction, row gather, the online-softmax merge of
// per-tile partials, the deterministic mean loss and the dH scatter.
// All are O(N*D) or O(N*V/256) HBM-bound helpers around the tensor-core engine.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace cce {

__device__ __forceinline__ int ld_acquire_sys_i(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// a0: range check + stable compaction of the non-ignored rows (P:2076-2079:
// rows with y == ignore_index are skipped; the mean divides by their count,
// P:899).  One block of 1024 threads; per pass over 8192 labels each warp owns a contiguous
// block of 256 (lane-strided: coalesced), ranks its valid labels with 8 ballots, and one
// block-wide scan of the 32 warp counts gives every warp its offset, so the compact order
// equals the original row order.  (The round-1 form scanned 8 tiles of 1024 one after
// another: 16 block barriers per 8192 labels.)
// Out-of-range labels set err and are treated as ignored.
// The same launch also resets the per-forward state the later kernels accumulate into
// (saves three memsets): the target logits zy_c [Npad] (written only by the tile that owns
// the label), the forward work-queue head / done counters and the finalize block counter.
__global__ void __launch_bounds__(1024) k_label_scan(const int32_t* __restrict__ labels, int N, int ignore_index,
                                                     long long vocab_total, int* __restrict__ pos,
                                                     int* __restrict__ idx, int* __restrict__ labels_c,
                                                     int* __restrict__ n_valid_out, int* __restrict__ err_out,
                                                     float* __restrict__ zy_c, int Npad, int* __restrict__ sched2,
                                                     int* __restrict__ fin_counter) {
  __shared__ int warp_tot[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  for (int i = t; i < Npad; i += 1024) zy_c[i] = 0.f;
  if (t == 0) {
    sched2[0] = 0;
    sched2[1] = 0;
    fin_counter[0] = 0;  // the finalize's last-block counter
    fin_counter[1] = 0;  // the merge kernel's (peer-memory signal)
  }
  // per pass of 8192 labels: warp w owns the contiguous block [s0 + 256 w, s0 + 256 (w + 1)),
  // lane l its labels l + 32 j (j = 0..7: coalesced loads and stores); the compact position of
  // (j, l) is the warp's offset + the valid labels of sub-blocks j' < j + those of lanes < l
  constexpr int PT = 8;
  int base = 0, bad = 0;
  for (int s0 = 0; s0 < N; s0 += PT * 1024) {
    const int b0 = s0 + 256 * w;
    int ys[PT];
    unsigned mk[PT];
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < PT; ++j) {
      const int n = b0 + 32 * j + lane;
      ys[j] = n < N ? labels[n] : ignore_index;
      bool v = false;
      if (n < N && ys[j] != ignore_index) {
        if (ys[j] < 0 || (long long)ys[j] >= vocab_total) bad = 1;
        else v = true;
      }
      mk[j] = __ballot_sync(0xffffffffu, v);
      cnt += __popc(mk[j]);
    }
    if (lane == 0) warp_tot[w] = cnt;
    __syncthreads();
    if (w == 0) {
      int v = warp_tot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      warp_tot[lane] = v;  // inclusive over warps
    }
    __syncthreads();
    int off = base + (w > 0 ? warp_tot[w - 1] : 0);
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < PT; ++j) {
      const int n = b0 + 32 * j + lane;
      if (n < N) {
        if (mk[j] >> lane & 1u) {
          const int o = off + __popc(mk[j] & lt);
          pos[n] = o;
          idx[o] = n;
          labels_c[o] = ys[j];
        } else {
          pos[n] = -1;
        }
      }
      off += __popc(mk[j]);
    }
    base += warp_tot[31];
    __syncthreads();  // warp_tot is rewritten by the next pass
  }
  const int any_bad = __syncthreads_or(bad);
  if (t == 0) {
    *n_valid_out = base;
    *err_out = any_bad ? 1 : 0;  // the flag of THIS forward (cce_get_error)
  }
}

// Gather the valid rows of H into the compact, dense, 16-byte aligned Hc so TMA
// tiles are contiguous; rows [n_valid, round_up(n_valid,128)) are zeroed (they
// are read as K-padding by the dW contraction).  Ignored rows of H are never read.
__global__ void k_gather_rows(const __nv_bfloat16* __restrict__ H, long long ldh, int D, int Npad,
                              const int* __restrict__ idx, const int* __restrict__ n_valid,
                              __nv_bfloat16* __restrict__ Hc) {
  const int nv = *n_valid;
  const int rows = min(Npad, ((nv + 127) / 128) * 128);
  const int vec_per_row = D / 8;
  const long long total = (long long)rows * vec_per_row;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // four 16-byte copies per thread in flight (the row-index loads first, then the data loads,
  // then the stores): the kernel is latency-bound at this size otherwise
  constexpr int U = 4;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < total; i0 += U * stride) {
    int src[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + u * stride;
      const int r = (int)(i / vec_per_row);
      src[u] = (i < total && r < nv) ? idx[r] : -1;
    }
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + u * stride;
      const int c = (int)(i % vec_per_row);
      v[u] = src[u] >= 0 ? *reinterpret_cast<const uint4*>(H + (long long)src[u] * ldh + c * 8) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + u * stride;
      if (i < total) {
        const int r = (int)(i / vec_per_row), c = (int)(i % vec_per_row);
        *reinterpret_cast<uint4*>(Hc + (long long)r * D + c * 8) = v[u];
      }
    }
  }
}

// The last block to arrive (threadfence + counter) sums loss_rows[0, nv) in a fixed order:
// threads 0-255 each keep eight independent partial sums (loads in flight), then a fixed
// shuffle tree and warp order -- the same order whatever the launch's block size, so the
// loss is bit-identical between the kernels that end with it.  Resets the counter.
__device__ __forceinline__ void loss_reduce_last_block(const float* __restrict__ loss_rows,
                                                       const int* __restrict__ n_valid, const int* __restrict__ err,
                                                       float* __restrict__ loss, int32_t* __restrict__ n_valid_out,
                                                       int sum, int* __restrict__ counter) {
  constexpr int RT = 256;  // reducing threads
  __shared__ int am_last;
  __shared__ float red[RT / 32];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = atomicAdd(counter, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  const int nv = *n_valid;
  if (threadIdx.x < RT) {
    float a8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int i0 = threadIdx.x; i0 < nv; i0 += 8 * RT) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * RT;
        if (i < nv) a8[u] += __ldcg(loss_rows + i);
      }
    }
    float acc = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int k = 0; k < RT / 32; ++k) t += red[k];
    float l = sum ? t : (nv > 0 ? t / (float)nv : 0.f);
    if (*err) l = __int_as_float(0x7fc00000);
    if (loss) *loss = l;
    if (n_valid_out) *n_valid_out = nv;
    *counter = 0;
  }
}

// Per-row loss from the row's global (lse, z_y, sum z):, with label smoothing eps /
// z-loss lambda (1 - eps)(lse - z_y) + eps (lse - sum_v z_v / V_total) + lambda lse^2.
__device__ __forceinline__ float row_loss(float lse, float zy, float zs, float ls_eps, float z_loss, float inv_vtotal) {
  float l = lse - zy;
  if (ls_eps != 0.f || z_loss != 0.f) l = (1.f - ls_eps) * l + ls_eps * (lse - zs * inv_vtotal) + z_loss * lse * lse;
  return l;
}

// world == 1 (no exchange): the finalize fused into the merge kernel (one launch less).
struct MergeFinalize {
  int on;
  const int* pos;    // [N] original -> compact (-1: ignored)
  const int* idx;    // [Npad] compact -> original
  int N;
  float* lse_out;    // [N] or nullptr
  float* lse_c;      // [Npad]
  float* loss_rows;  // [Npad]
  float* loss_tok;   // [N] (reduction "none") or nullptr
  float ls_eps, z_loss, inv_vtotal;
  const int* err;
  float* loss;       // scalar or nullptr
  int32_t* n_valid_out;
  int sum;
  int* counter;
};

// CCE_FLAG_P2P_COMBINE: the merged stats also go straight into every rank's all-ranks array
// (slot of this rank, peer memory), so the exchange needs no separate kernel (a9 fused).
struct StatsPush {
  float4* dst[8];  // every rank's stats_all + rank * Npad (peer memory), or unused
  int n;           // number of destinations (0: no push)
  // the flag (kind P2P_STATS, this rank) in every rank, raised to `epoch` by the last block to
  // finish (counter: last-block pattern) after a system-scope fence -- the signal fused into
  // the kernel that produced the stats
  int* flag[8];
  int epoch;
  int* counter;
};

constexpr int MERGE_SL = 16;  // tile slices per merge block (512 threads: two blocks per SM, one wave)
// a4 (local part): merge the per-vocabulary-tile (m, d) partials of each valid
// row with the online-softmax merge:
// m = max_t m_t, d = sum_t d_t exp(m_t - m).  Block = 32 rows x MERGE_SL tile-slices
// (512 threads): thread (lane, w) folds tiles t = w, w+16,
// ... of row i0+lane (coalesced: part is [tile][row]), then warp 0 folds the slices in order.
// Fixed order -> deterministic.  Out: (m, d, z_y) per compact row.
// With label smoothing the per-tile logit sums (zs_part, may be nullptr) are summed in
// the same fixed order into the 4th stat (sum_v z_v of the row over this shard).
__global__ void __launch_bounds__(32 * MERGE_SL) k_merge_tiles(const float2* __restrict__ part, int Tv, int Npad,
                                                      const float* __restrict__ zy_c, const int* __restrict__ n_valid,
                                                      const float* __restrict__ zs_part, float4* __restrict__ stats,
                                                      const StatsPush push, const MergeFinalize fin) {
  __shared__ float2 red[MERGE_SL][33];
  __shared__ float redz[MERGE_SL][33];
  const int nv = *n_valid;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  float m = -INFINITY, d = 0.f, zs = 0.f;
  if (i < nv) {
    // batches of eight tiles' partials per thread, the next batch loaded before the current
    // one is merged (the loop is load-latency-bound otherwise); merged in tile order
    constexpr int NB = 8;
    float2 cur[NB], nxt[NB];
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const int t = w + MERGE_SL * u;
      cur[u] = t < Tv ? part[(size_t)t * Npad + i] : make_float2(-INFINITY, 0.f);
    }
    for (int t0 = w; t0 < Tv; t0 += NB * MERGE_SL) {
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        const int t = t0 + NB * MERGE_SL + MERGE_SL * u;
        nxt[u] = t < Tv ? part[(size_t)t * Npad + i] : make_float2(-INFINITY, 0.f);
      }
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        // one exponential per merge (the larger max keeps its partial unscaled); fast exp
        // (ex2.approx, reading R16): the kernel is instruction-bound, not memory-bound
        if (cur[u].y > 0.f) {
          if (cur[u].x > m) {
            d = d * __expf(m - cur[u].x) + cur[u].y;
            m = cur[u].x;
          } else {
            d += cur[u].y * __expf(cur[u].x - m);
          }
        }
      }
      if (zs_part) {
#pragma unroll
        for (int u = 0; u < NB; ++u)
          if (t0 + MERGE_SL * u < Tv) zs += zs_part[(size_t)(t0 + MERGE_SL * u) * Npad + i];
      }
#pragma unroll
      for (int u = 0; u < NB; ++u) cur[u] = nxt[u];
    }
  }
  red[w][lane] = make_float2(m, d);
  redz[w][lane] = zs;
  __syncthreads();
  if (w == 0 && i < nv) {
    float M = -INFINITY, S = 0.f, Z = 0.f;
    for (int k = 0; k < MERGE_SL; ++k) {
      const float2 pd = red[k][lane];
      if (pd.y > 0.f) {
        const float mn = fmaxf(M, pd.x);
        S = S * expf(M - mn) + pd.y * expf(pd.x - mn);
        M = mn;
      }
      Z += redz[k][lane];
    }
    const float4 st = make_float4(M, S, zy_c[i], Z);
    stats[i] = st;
    for (int k = 0; k < push.n; ++k) push.dst[k][i] = st;
    if (fin.on) {  // = k_finalize_loss at world 1: m = M, d = S exp(M - M) = S
      const float lse = M + logf(S);
      fin.lse_c[i] = lse;
      const float l = row_loss(lse, st.z, Z, fin.ls_eps, fin.z_loss, fin.inv_vtotal);
      fin.loss_rows[i] = l;
      const int n = fin.idx[i];
      if (fin.loss_tok) fin.loss_tok[n] = l;
      if (fin.lse_out) fin.lse_out[n] = lse;
    }
  }
  if (push.n) {
    __threadfence_system();  // this block's peer stores are visible before the flag
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(push.counter, 1) == (int)gridDim.x - 1) {
      *push.counter = 0;
      __threadfence_system();
      for (int r = 0; r < push.n; ++r)
        asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(push.flag[r]), "r"(push.epoch) : "memory");
    }
  }
  if (fin.on) {
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < fin.N; n += gridDim.x * blockDim.x)
      if (fin.pos[n] < 0) {  // ignored rows: lse = 0 (reading R4), per-token loss 0
        if (fin.lse_out) fin.lse_out[n] = 0.f;
        if (fin.loss_tok) fin.loss_tok[n] = 0.f;
      }
    loss_reduce_last_block(fin.loss_rows, n_valid, fin.err, fin.loss, fin.n_valid_out, fin.sum, fin.counter);
  }
}


// a4 (global part) + a9 combine: merge the per-rank stats in rank order (empty
// shards contribute m=-inf, d=0), lse = m + log d (Theorem), per-row loss
// lse - z_y.  Ignored rows get lse = 0 (reading R4).
// With label smoothing eps / z-loss lambda the row loss is
//   (1 - eps)(lse - z_y) + eps (lse - sum_v z_v / V_total) + lambda lse^2.
// The same launch then reduces the loss: every block publishes
// its rows (threadfence + counter), and the last block to finish sums loss_rows[0, nv)
// in a fixed order (thread-strided, then a fixed shuffle tree and warp order), so the
// result is deterministic; it resets the counter for the next forward.
__global__ void __launch_bounds__(256) k_finalize_loss(
    const float4* __restrict__ stats_all, int world, int Npad, const int* __restrict__ pos, int N,
    float* __restrict__ lse_out, float* __restrict__ lse_c, float* __restrict__ loss_rows, float ls_eps,
    float z_loss, float inv_vtotal, float* __restrict__ loss_tok, const int* __restrict__ n_valid,
    const int* __restrict__ err, float* __restrict__ loss, int32_t* __restrict__ n_valid_out, int sum,
    int* __restrict__ counter, const int* __restrict__ wait_flags, int epoch, int* __restrict__ err_w) {
  if (wait_flags) {
    // peer-memory exchange: every rank's stats flag (kind P2P_STATS) must show this step's epoch
    // before the rows are merged; bounded at 5 s (a missing peer sets err bit 4)
    if ((int)threadIdx.x < world) {
      const unsigned long long t0 = gtimer_ns();
      while (ld_acquire_sys_i(wait_flags + threadIdx.x) < epoch) {
        if (gtimer_ns() - t0 > 5000000000ull) { atomicOr(err_w, 4); break; }
        __nanosleep(256);
      }
    }
    __syncthreads();
  }
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    const int i = pos[n];
    if (i < 0) {
      if (lse_out) lse_out[n] = 0.f;
      if (loss_tok) loss_tok[n] = 0.f;
      continue;
    }
    float m = -INFINITY, zy = 0.f, zs = 0.f;
    for (int r = 0; r < world; ++r) {
      const float4 st = __ldcg(stats_all + (size_t)r * Npad + i);  // written by other kernels / GPUs: L2
      m = fmaxf(m, st.x);
      zy += st.z;
      zs += st.w;
    }
    float d = 0.f;
    for (int r = 0; r < world; ++r) {
      const float4 st = __ldcg(stats_all + (size_t)r * Npad + i);
      if (st.y > 0.f) d += st.y * expf(st.x - m);
    }
    const float lse = m + logf(d);
    lse_c[i] = lse;
    const float l = row_loss(lse, zy, zs, ls_eps, z_loss, inv_vtotal);
    loss_rows[i] = l;
    if (loss_tok) loss_tok[n] = l;
    if (lse_out) lse_out[n] = lse;
  }
  loss_reduce_last_block(loss_rows, n_valid, err, loss, n_valid_out, sum, counter);
}

// Mean loss over the valid rows in a fixed reduction order (deterministic).
// loss = 0 when n_valid == 0 (reading R2); NaN when a label was out of range.
// mean (default) or sum (sum = 1); loss may be nullptr (reduction "none": only n_valid).
__global__ void __launch_bounds__(1024) k_loss(const float* __restrict__ loss_rows, const int* __restrict__ n_valid,
                                               const int* __restrict__ err, float* __restrict__ loss,
                                               int32_t* __restrict__ n_valid_out, int sum) {
  __shared__ float red[32];
  const int nv = *n_valid;
  float s = 0.f;
  for (int i = threadIdx.x; i < nv; i += 1024) s += loss_rows[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = red[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) {
      float l = sum ? s : (nv > 0 ? s / (float)nv : 0.f);
      if (*err) l = __int_as_float(0x7fc00000);
      if (loss) *loss = l;
      if (n_valid_out) *n_valid_out = nv;
    }
  }
}

// a8: dH rows back to the original positions in bf16; ignored rows are bit-zero.
// fp32 = 1: dH is float32; accumulate = 1: dH += gradient (ignored rows untouched).
__global__ void k_scatter_dH(const float* __restrict__ dH32, const int* __restrict__ pos, int N, int D,
                             void* __restrict__ dH_out, int fp32, int accumulate, const int* __restrict__ done = nullptr,
                             const int* __restrict__ n_valid = nullptr, int epoch = 0, int* __restrict__ err = nullptr) {
  if (done) {
    // peer-memory exchange: every dH tile's reduced sum has arrived (the RED items raised
    // done[tile][cta] = epoch); bounded at 5 s like k_p2p_wait_tiles
    const int t256 = (*n_valid + 255) / 256, n_dt = (D + 255) / 256;
    const int n = 2 * t256 * n_dt;
    const unsigned long long t0 = gtimer_ns();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      while (ld_acquire_sys_i(done + i) < epoch) {
        if (gtimer_ns() - t0 > 5000000000ull) { atomicOr(err, 4); break; }
        __nanosleep(256);
      }
    }
    __syncthreads();
  }
  const int vec_per_row = D / 8;
  const long long total = (long long)N * vec_per_row;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(i / vec_per_row), c = (int)(i % vec_per_row);
    const int r = pos[n];
    if (fp32 || accumulate) {
      if (accumulate && r < 0) continue;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
      if (r >= 0) {
        a = __ldcg(reinterpret_cast<const float4*>(dH32 + (long long)r * D + c * 8));
        b = __ldcg(reinterpret_cast<const float4*>(dH32 + (long long)r * D + c * 8 + 4));
      }
      if (fp32) {
        float4* d = reinterpret_cast<float4*>(static_cast<float*>(dH_out) + (long long)n * D + c * 8);
        if (accumulate) {
          const float4 o0 = d[0], o1 = d[1];
          a.x += o0.x; a.y += o0.y; a.z += o0.z; a.w += o0.w;
          b.x += o1.x; b.y += o1.y; b.z += o1.z; b.w += o1.w;
        }
        d[0] = a;
        d[1] = b;
      } else {  // bf16 accumulate: add in fp32, round once
        uint4* d = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(dH_out) + (long long)n * D + c * 8);
        const uint4 o = *d;
        const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        const uint32_t w[4] = {o.x, o.y, o.z, o.w};
        uint32_t q[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float lo = f[2 * k] + __uint_as_float(w[k] << 16);
          const float hi = f[2 * k + 1] + __uint_as_float(w[k] & 0xffff0000u);
          __nv_bfloat162 p2 = __floats2bfloat162_rn(lo, hi);
          q[k] = *reinterpret_cast<uint32_t*>(&p2);
        }
        *d = make_uint4(q[0], q[1], q[2], q[3]);
      }
      continue;
    }
    __nv_bfloat16* dH = static_cast<__nv_bfloat16*>(dH_out);
    uint4 out = make_uint4(0, 0, 0, 0);
    if (r >= 0) {
      const float4 a = __ldcg(reinterpret_cast<const float4*>(dH32 + (long long)r * D + c * 8));
      const float4 b = __ldcg(reinterpret_cast<const float4*>(dH32 + (long long)r * D + c * 8 + 4));
      __nv_bfloat162 p0 = __floats2bfloat162_rn(a.x, a.y), p1 = __floats2bfloat162_rn(a.z, a.w);
      __nv_bfloat162 p2 = __floats2bfloat162_rn(b.x, b.y), p3 = __floats2bfloat162_rn(b.z, b.w);
      out.x = *reinterpret_cast<uint32_t*>(&p0);
      out.y = *reinterpret_cast<uint32_t*>(&p1);
      out.z = *reinterpret_cast<uint32_t*>(&p2);
      out.w = *reinterpret_cast<uint32_t*>(&p3);
    }
    *reinterpret_cast<uint4*>(dH + (long long)n * D + c * 8) = out;
  }
}

__global__ void k_set_scalar(float* p, float v) { *p = v; }

// CCE_FLAG_DH_SEQ_SHARD: rows of an fp32 dH slice -> the caller's dH (bf16 or fp32, overwrite or add).
__global__ void k_rows_out(const float* __restrict__ src, int rows, int D, void* __restrict__ dst, int fp32,
                           int accumulate) {
  const long long total = (long long)rows * D / 8;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    float4 a = reinterpret_cast<const float4*>(src)[2 * i], b = reinterpret_cast<const float4*>(src)[2 * i + 1];
    if (fp32) {
      float4* d = reinterpret_cast<float4*>(dst) + 2 * i;
      if (accumulate) {
        const float4 o0 = d[0], o1 = d[1];
        a.x += o0.x; a.y += o0.y; a.z += o0.z; a.w += o0.w;
        b.x += o1.x; b.y += o1.y; b.z += o1.z; b.w += o1.w;
      }
      d[0] = a;
      d[1] = b;
    } else {
      uint4* d = reinterpret_cast<uint4*>(dst) + i;
      float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      if (accumulate) {
        const uint4 o = *d;
        const uint32_t w[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          f[2 * k] += __uint_as_float(w[k] << 16);
          f[2 * k + 1] += __uint_as_float(w[k] & 0xffff0000u);
        }
      }
      __nv_bfloat162 q0 = __floats2bfloat162_rn(f[0], f[1]), q1 = __floats2bfloat162_rn(f[2], f[3]);
      __nv_bfloat162 q2 = __floats2bfloat162_rn(f[4], f[5]), q3 = __floats2bfloat162_rn(f[6], f[7]);
      *d = make_uint4(*reinterpret_cast<uint32_t*>(&q0), *reinterpret_cast<uint32_t*>(&q1),
                      *reinterpret_cast<uint32_t*>(&q2), *reinterpret_cast<uint32_t*>(&q3));
    }
  }
}

// reduction "none": the per-token upstream gradients of the valid rows in compact order.
__global__ void k_gather_dloss(const float* __restrict__ dloss, const int* __restrict__ idx,
                               const int* __restrict__ n_valid, int Npad, float* __restrict__ dloss_c) {
  const int nv = *n_valid;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < Npad; i += gridDim.x * blockDim.x)
    dloss_c[i] = i < nv ? dloss[idx[i]] : 0.f;
}

// One AdamW element update in the order of the paper's fused kernel.
__device__ __forceinline__ void adamw_elem(float g, float& th, float& m, float& v, float lr, float b1, float b2,
                                           float eps, float wd, float bc1, float bc2) {
  th = th * (1.f - lr * wd);
  m = b1 * m + (1.f - b1) * g;
  v = b2 * v + (1.f - b2) * g * g;
  const float mh = m / bc1;
  const float vh = v / bc2;
  th = th - lr * (mh / (sqrtf(vh) + eps));
}

// Standalone fused AdamW (Alg. Fused AdamW P:2003-2046; cce.h cce_adamw_step): one
// read and one write of each state array, 8 elements (32-byte vectors) per thread and
// iteration, grid-stride over n / 8 groups plus a scalar tail.  HBM-bound.
struct AdamwArgs {
  float lr, b1, b2, eps, wd, bc1, bc2;
  const float* clip;
  float* master;
  float* m;
  float* v;
  const float* grad_in;
  const void* grad;
  int grad_fp32;
  __nv_bfloat16* w;
  long long n;
};

__device__ __forceinline__ float adamw_grad_at(const AdamwArgs& a, long long i) {
  float g = 0.f;
  if (a.grad) g = a.grad_fp32 ? static_cast<const float*>(a.grad)[i]
                              : __bfloat162float(static_cast<const __nv_bfloat16*>(a.grad)[i]);
  if (a.grad_in) g += a.grad_in[i];
  return g;
}

__global__ void k_adamw(const AdamwArgs a) {
  const float clip = a.clip ? *a.clip : 1.f;
  const long long ngrp = a.n / 8;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < ngrp; gi += stride) {
    const long long i0 = gi * 8;
    float g[8], th[8], m[8], v[8];
    const float4* m4 = reinterpret_cast<const float4*>(a.m + i0);
    const float4* v4 = reinterpret_cast<const float4*>(a.v + i0);
    float4 t0 = m4[0], t1 = m4[1];
    m[0] = t0.x; m[1] = t0.y; m[2] = t0.z; m[3] = t0.w; m[4] = t1.x; m[5] = t1.y; m[6] = t1.z; m[7] = t1.w;
    t0 = v4[0]; t1 = v4[1];
    v[0] = t0.x; v[1] = t0.y; v[2] = t0.z; v[3] = t0.w; v[4] = t1.x; v[5] = t1.y; v[6] = t1.z; v[7] = t1.w;
    if (a.master) {
      const float4* th4 = reinterpret_cast<const float4*>(a.master + i0);
      t0 = th4[0]; t1 = th4[1];
      th[0] = t0.x; th[1] = t0.y; th[2] = t0.z; th[3] = t0.w; th[4] = t1.x; th[5] = t1.y; th[6] = t1.z; th[7] = t1.w;
    } else {
      const uint4 wb = *reinterpret_cast<const uint4*>(a.w + i0);
      const uint32_t w[4] = {wb.x, wb.y, wb.z, wb.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        th[2 * k] = __uint_as_float(w[k] << 16);
        th[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
      }
    }
    if (!a.grad) {
#pragma unroll
      for (int k = 0; k < 8; ++k) g[k] = 0.f;
    } else if (a.grad_fp32) {
      const float4* g4 = reinterpret_cast<const float4*>(static_cast<const float*>(a.grad) + i0);
      t0 = g4[0]; t1 = g4[1];
      g[0] = t0.x; g[1] = t0.y; g[2] = t0.z; g[3] = t0.w; g[4] = t1.x; g[5] = t1.y; g[6] = t1.z; g[7] = t1.w;
    } else {
      const uint4 gb = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.grad) + i0);
      const uint32_t w[4] = {gb.x, gb.y, gb.z, gb.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        g[2 * k] = __uint_as_float(w[k] << 16);
        g[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
      }
    }
    if (a.grad_in) {
      const float4* g4 = reinterpret_cast<const float4*>(a.grad_in + i0);
      t0 = g4[0]; t1 = g4[1];
      g[0] += t0.x; g[1] += t0.y; g[2] += t0.z; g[3] += t0.w; g[4] += t1.x; g[5] += t1.y; g[6] += t1.z; g[7] += t1.w;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) adamw_elem(g[k] * clip, th[k], m[k], v[k], a.lr, a.b1, a.b2, a.eps, a.wd, a.bc1, a.bc2);
    float4* mo = reinterpret_cast<float4*>(a.m + i0);
    float4* vo = reinterpret_cast<float4*>(a.v + i0);
    mo[0] = make_float4(m[0], m[1], m[2], m[3]); mo[1] = make_float4(m[4], m[5], m[6], m[7]);
    vo[0] = make_float4(v[0], v[1], v[2], v[3]); vo[1] = make_float4(v[4], v[5], v[6], v[7]);
    if (a.master) {
      float4* to = reinterpret_cast<float4*>(a.master + i0);
      to[0] = make_float4(th[0], th[1], th[2], th[3]); to[1] = make_float4(th[4], th[5], th[6], th[7]);
    }
    if (a.w) {
      __nv_bfloat162 p0 = __floats2bfloat162_rn(th[0], th[1]), p1 = __floats2bfloat162_rn(th[2], th[3]);
      __nv_bfloat162 p2 = __floats2bfloat162_rn(th[4], th[5]), p3 = __floats2bfloat162_rn(th[6], th[7]);
      *reinterpret_cast<uint4*>(a.w + i0) =
          make_uint4(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1),
                     *reinterpret_cast<uint32_t*>(&p2), *reinterpret_cast<uint32_t*>(&p3));
    }
  }
  // scalar tail (n % 8 elements)
  const long long tail = ngrp * 8 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (tail < a.n && tail < ngrp * 8 + 8) {
    const long long i = tail;
    float th = a.master ? a.master[i] : __bfloat162float(a.w[i]);
    float m = a.m[i], v = a.v[i];
    adamw_elem(adamw_grad_at(a, i) * clip, th, m, v, a.lr, a.b1, a.b2, a.eps, a.wd, a.bc1, a.bc2);
    a.m[i] = m;
    a.v[i] = v;
    if (a.master) a.master[i] = th;
    if (a.w) a.w[i] = __float2bfloat16_rn(th);
  }
}

}  // namespace cce

namespace cce {

// ------------------------------------------------------------------ RMSNorm prologue
// (Def. RMSNorm, Alg. Fused RMSNorm Forward P:712-731):
// the gather of the valid rows normalises them on the way, Hc[r] = bf16((x rstd) gamma)
// with rstd = 1 / sqrt(mean(x^2) + eps) in fp32, and caches rstd per compact row for the
// backward (Alg. "Cache rstd for backward").  One warp per row; 16-byte vectors; the
// warp's sum of squares is reduced in a fixed butterfly order (deterministic).  Rows
// [n_valid, round_up(n_valid, 128)) are zeroed like k_gather_rows; ignored rows are never read.
__global__ void k_gather_rmsnorm(const __nv_bfloat16* __restrict__ X, long long ldx, int D, int Npad,
                                 const int* __restrict__ idx, const int* __restrict__ n_valid,
                                 const __nv_bfloat16* __restrict__ gamma, float eps, __nv_bfloat16* __restrict__ Hc,
                                 float* __restrict__ rstd_c) {
  const int nv = *n_valid;
  const int rows = min(Npad, ((nv + 127) / 128) * 128);
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int nvec = D / 8;
  for (int r = blockIdx.x * wpb + (threadIdx.x >> 5); r < rows; r += gridDim.x * wpb) {
    uint4* dst = reinterpret_cast<uint4*>(Hc + (long long)r * D);
    if (r >= nv) {
      for (int c = lane; c < nvec; c += 32) dst[c] = make_uint4(0, 0, 0, 0);
      continue;
    }
    const uint4* src = reinterpret_cast<const uint4*>(X + (long long)idx[r] * ldx);
    float ss = 0.f;
    for (int c = lane; c < nvec; c += 32) {
      const uint4 v = src[c];
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float a = __uint_as_float(w[k] << 16), b = __uint_as_float(w[k] & 0xffff0000u);
        ss = fmaf(a, a, ss);
        ss = fmaf(b, b, ss);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float rstd = 1.f / sqrtf(ss / (float)D + eps);
    const uint4* g4 = reinterpret_cast<const uint4*>(gamma);
    for (int c = lane; c < nvec; c += 32) {
      const uint4 v = src[c], gv = g4[c];
      const uint32_t w[4] = {v.x, v.y, v.z, v.w}, gw[4] = {gv.x, gv.y, gv.z, gv.w};
      uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float y0 = (__uint_as_float(w[k] << 16) * rstd) * __uint_as_float(gw[k] << 16);
        const float y1 = (__uint_as_float(w[k] & 0xffff0000u) * rstd) * __uint_as_float(gw[k] & 0xffff0000u);
        __nv_bfloat162 p = __floats2bfloat162_rn(y0, y1);
        o[k] = *reinterpret_cast<uint32_t*>(&p);
      }
      dst[c] = make_uint4(o[0], o[1], o[2], o[3]);
    }
    if (lane == 0) rstd_c[r] = rstd;
  }
}

// RMSNorm backward (reading R18: the exact gradient of Def. RMSNorm), fed by the
// UNROUNDED fp32 dH of the CE path (dH32, compact rows):
//   xbar = x rstd,  c1 = (1/D) sum_i g_i gamma_i xbar_i,  dx = rstd (gamma g - xbar c1)
//   dgamma = sum_rows g xbar
// Block = 4 warps; warp w of block b takes compact rows b*4 + w, + 4*gridDim, ... in
// order and accumulates its dgamma contribution in its own shared-memory row [D];
// the block sums its 4 rows in fixed order into gpart[b][D] (k_dgamma_reduce then sums
// the blocks in fixed order): deterministic, no atomics.  dX rows of valid tokens are
// written here (scattered to the original positions); ignored rows by k_zero_ignored.
constexpr int RMS_BWD_WARPS = 4;
__global__ void __launch_bounds__(32 * RMS_BWD_WARPS)
    k_rmsnorm_bwd(const float* __restrict__ dH32, const __nv_bfloat16* __restrict__ X, long long ldx,
                  const int* __restrict__ idx, const int* __restrict__ n_valid,
                  const __nv_bfloat16* __restrict__ gamma, const float* __restrict__ rstd_c, int D, void* dX,
                  int grad_fp32, int accumulate, float* __restrict__ gpart) {
  extern __shared__ float sp[];  // [RMS_BWD_WARPS][D]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* part = sp + (size_t)w * D;
  for (int j = lane; j < D; j += 32) part[j] = 0.f;
  const int nv = *n_valid;
  const int nvec = D / 8;
  const uint4* g4 = reinterpret_cast<const uint4*>(gamma);
  for (int r = blockIdx.x * RMS_BWD_WARPS + w; r < nv; r += gridDim.x * RMS_BWD_WARPS) {
    const long long n = idx[r];
    const float rs = rstd_c[r];
    const uint4* xs = reinterpret_cast<const uint4*>(X + n * ldx);
    const float4* gs = reinterpret_cast<const float4*>(dH32 + (long long)r * D);
    float c1 = 0.f;
    for (int c = lane; c < nvec; c += 32) {
      const uint4 xv = xs[c], gv = g4[c];
      const float4 a = gs[2 * c], b = gs[2 * c + 1];
      const float gg[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w}, gw[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        c1 = fmaf(gg[2 * k] * __uint_as_float(gw[k] << 16), __uint_as_float(xw[k] << 16) * rs, c1);
        c1 = fmaf(gg[2 * k + 1] * __uint_as_float(gw[k] & 0xffff0000u), __uint_as_float(xw[k] & 0xffff0000u) * rs, c1);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c1 += __shfl_xor_sync(0xffffffffu, c1, o);
    c1 /= (float)D;
    for (int c = lane; c < nvec; c += 32) {
      const uint4 xv = xs[c], gv = g4[c];
      const float4 a = gs[2 * c], b = gs[2 * c + 1];
      const float gg[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w}, gw[4] = {gv.x, gv.y, gv.z, gv.w};
      float dx[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float xb0 = __uint_as_float(xw[k] << 16) * rs, xb1 = __uint_as_float(xw[k] & 0xffff0000u) * rs;
        dx[2 * k] = rs * (__uint_as_float(gw[k] << 16) * gg[2 * k] - xb0 * c1);
        dx[2 * k + 1] = rs * (__uint_as_float(gw[k] & 0xffff0000u) * gg[2 * k + 1] - xb1 * c1);
        part[c * 8 + 2 * k] = fmaf(gg[2 * k], xb0, part[c * 8 + 2 * k]);
        part[c * 8 + 2 * k + 1] = fmaf(gg[2 * k + 1], xb1, part[c * 8 + 2 * k + 1]);
      }
      if (grad_fp32) {
        float4* o = reinterpret_cast<float4*>(static_cast<float*>(dX) + n * D) + 2 * c;
        if (accumulate) {
          const float4 p0 = o[0], p1 = o[1];
          dx[0] += p0.x; dx[1] += p0.y; dx[2] += p0.z; dx[3] += p0.w;
          dx[4] += p1.x; dx[5] += p1.y; dx[6] += p1.z; dx[7] += p1.w;
        }
        o[0] = make_float4(dx[0], dx[1], dx[2], dx[3]);
        o[1] = make_float4(dx[4], dx[5], dx[6], dx[7]);
      } else {
        uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(dX) + n * D) + c;
        if (accumulate) {
          const uint4 p = *o;
          const uint32_t pw[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            dx[2 * k] += __uint_as_float(pw[k] << 16);
            dx[2 * k + 1] += __uint_as_float(pw[k] & 0xffff0000u);
          }
        }
        __nv_bfloat162 q0 = __floats2bfloat162_rn(dx[0], dx[1]), q1 = __floats2bfloat162_rn(dx[2], dx[3]);
        __nv_bfloat162 q2 = __floats2bfloat162_rn(dx[4], dx[5]), q3 = __floats2bfloat162_rn(dx[6], dx[7]);
        *o = make_uint4(*reinterpret_cast<uint32_t*>(&q0), *reinterpret_cast<uint32_t*>(&q1),
                        *reinterpret_cast<uint32_t*>(&q2), *reinterpret_cast<uint32_t*>(&q3));
      }
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < D; j += blockDim.x) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < RMS_BWD_WARPS; ++k) s += sp[(size_t)k * D + j];
    gpart[(size_t)blockIdx.x * D + j] = s;
  }
}

// dgamma = sum of the per-block partials in block order (deterministic).
__global__ void k_dgamma_reduce(const float* __restrict__ gpart, int nb, int D, void* dgamma, int grad_fp32,
                                int accumulate) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < D; j += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < nb; ++b) s += gpart[(size_t)b * D + j];
    if (grad_fp32) {
      float* o = static_cast<float*>(dgamma) + j;
      *o = accumulate ? *o + s : s;
    } else {
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(dgamma) + j;
      *o = __float2bfloat16_rn(accumulate ? __bfloat162float(*o) + s : s);
    }
  }
}

// dX rows of ignored tokens: 0 (overwrite mode only; they receive no gradient).
__global__ void k_zero_ignored(const int* __restrict__ pos, int N, int D, void* dX, int grad_fp32) {
  const int nvec = D / 8;
  const long long total = (long long)N * nvec;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(i / nvec), c = (int)(i % nvec);
    if (pos[n] >= 0) continue;
    if (grad_fp32) {
      float4* o = reinterpret_cast<float4*>(static_cast<float*>(dX) + (long long)n * D) + 2 * c;
      o[0] = make_float4(0.f, 0.f, 0.f, 0.f);
      o[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(dX) + (long long)n * D)[c] = make_uint4(0, 0, 0, 0);
    }
  }
}

}  // namespace cce
