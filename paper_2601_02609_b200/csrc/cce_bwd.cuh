// cce_bwd.cuh -- the whole CCE backward as ONE persistent,
// warp-specialised tcgen05 kernel driven by a device-side work queue.
//
// The paper's backward (Alg. "CCE Triton Backward Kernel") walks the
// vocabulary in chunks: recompute the chunk's logits, form softmax - onehot,
// then grad_h += probs @ W[chunk] and grad_W[chunk] += probs^T @ h.  Here each
// chunk c (CCE_CHUNK vocabulary rows) becomes three families of 128 x 256 tiles:
//   G(c)   recompute S = Hc W_c^T, epilogue G = s (exp(S - lse) - onehot) -> bf16
//          into the chunk's slot of a 3-slot ring buffer Gbuf (N x chunk, never N x V)
//   DW(c)  dW_c^T = Hc^T G_c      (tile: 128 hidden x 256 vocab, K = valid rows)
//   DH(c)  dH^T  += W_c^T G_c^T   (tile: 128 hidden x 256 rows, K = chunk), fp32
//          read-modify-write in chunk order (deterministic)
// All tiles of all chunks are handed out by one global atomic queue in the order
//   G0, G1, W0, G2, W1, ..., G_{n-1}, W_{n-2}, W_{n-1}      (W_c = DH(c) then DW(c))
// and each item's producer warp waits (acquire loads on global counters) only on
// items that precede it in the queue, so the schedule cannot deadlock:
//   G(c)        needs W(c-3) finished        (its Gbuf slot is free again; W(c-3) was
//               queued a whole phase before, so this wait is normally already satisfied)
//   DW(c),DH(c) need every G(c) tile finished (G_c complete in Gbuf)
//   DH(c,tile)  needs DH(c-1,tile) finished   (ordered fp32 accumulation)
// One launch replaces 3 x n_chunks launches: no wave-quantisation tail per chunk,
// and every epilogue (bf16 G store, dW store, dH RMW) overlaps later tiles' MMAs
// through the double-buffered TMEM accumulator.
#pragma once
#include "cce_gemm.cuh"

namespace cce {

enum ItemType : int { IT_G = 0, IT_DW = 1, IT_DH = 2, IT_END = 3 };

struct Item {
  int type, c, mt, nt, width, num_kb, tile_id, q;
  unsigned long long t_deq, t_ready;  // globaltimer stamps (trace only)
};

// Optional per-item trace record (cce_debug_trace): 8 x u64 per queue position.
struct TraceRec {
  unsigned long long q_type_c, smid, t_deq, t_ready, t_epi0, t_epi1, tile, pad;
  unsigned long long t_load0, t_load1, t_mma0, t_mma1, t_full_wait, r0, r1, r2;  // pair kernel only
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

struct BwdParams {
  GemmParams g;      // shared sizes/pointers (gbuf = slot 0 base)
  int n_chunks;
  int* sched;        // zeroed before launch: [0] queue head | [1] items done | g_done[n] | w_done[n] | dh_flag[tiles]
  TraceRec* trace;   // optional (nullptr): one record per queue position
  int trace_cap;
  int slots;         // Gbuf ring slots (>= 2)
  int strict;        // debug: every item waits for all earlier items to finish
};

constexpr int RING = 4;
constexpr int GBUF_SLOTS = 3;  // ring of chunk dlogits buffers: G(c) reuses the slot of chunk c-3

struct BwdCounts {
  int nv, tiles_tok, tiles_d, tiles_tok256, n_dh;
};

__device__ __forceinline__ int chunk_width(const GemmParams& g, int c) {
  const int rem = g.V_local - c * g.C;
  return rem < g.C ? rem : g.C;
}
__device__ __forceinline__ int n_g_items(const BwdCounts& k, int width) { return k.tiles_tok * ((width + BN - 1) / BN); }
__device__ __forceinline__ int n_dw_items(const BwdCounts& k, int width) { return k.tiles_d * ((width + BN - 1) / BN); }

// Decode queue position q into an item (walks the phase list; n_chunks <= ~40).
__device__ Item decode_item(const BwdParams& P, const BwdCounts& k, int q) {
  const GemmParams& g = P.g;
  const int n = P.n_chunks;
  // phase list: G0, then for c=1..n-1: G_c, W_{c-1}; then W_{n-1}
  for (int ph = 0; ph < 2 * n; ++ph) {
    int type, c;
    if (ph == 0) { type = IT_G; c = 0; }
    else if (ph == 2 * n - 1) { type = IT_DW; c = n - 1; }
    else if (ph & 1) { type = IT_G; c = (ph + 1) / 2; }
    else { type = IT_DW; c = ph / 2 - 1; }
    const int width = chunk_width(g, c);
    if (type == IT_G) {
      const int cnt = n_g_items(k, width);
      if (q < cnt) {
        Item it;
        it.type = IT_G; it.c = c; it.width = width;
        it.mt = q % k.tiles_tok; it.nt = q / k.tiles_tok;
        it.num_kb = g.D / BK; it.tile_id = 0;
        return it;
      }
      q -= cnt;
    } else {
      const int cnt = k.n_dh + n_dw_items(k, width);
      if (q < cnt) {
        Item it;
        it.c = c; it.width = width;
        if (q < k.n_dh) {
          it.type = IT_DH; it.mt = q % k.tiles_d; it.nt = q / k.tiles_d; it.tile_id = q;
          it.num_kb = (width + BK - 1) / BK;
        } else {
          const int r = q - k.n_dh;
          it.type = IT_DW; it.mt = r % k.tiles_d; it.nt = r / k.tiles_d; it.tile_id = 0;
          it.num_kb = (k.nv + BK - 1) / BK;
        }
        return it;
      }
      q -= cnt;
    }
  }
  Item e;
  e.type = IT_END; e.c = 0; e.mt = 0; e.nt = 0; e.width = 0; e.num_kb = 0; e.tile_id = 0;
  e.q = 0; e.t_deq = 0; e.t_ready = 0;
  return e;
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

__global__ void __launch_bounds__(GEMM_THREADS, 1)
    cce_bwd_kernel(const __grid_constant__ CUtensorMap tmHcK, const __grid_constant__ CUtensorMap tmWK,
                   const __grid_constant__ CUtensorMap tmHcMN, const __grid_constant__ CUtensorMap tmGMN,
                   const __grid_constant__ CUtensorMap tmWMN, const __grid_constant__ CUtensorMap tmGK,
                   const BwdParams P) {
  const GemmParams& g = P.g;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* rfull_bar = tempty_bar + 2;
  uint64_t* rempty_bar = rfull_bar + RING;
  Item* ring = reinterpret_cast<Item*>(rempty_bar + RING);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + RING);
  float* xchg = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 512);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  int* queue_head = P.sched;
  int* done_total = P.sched + 1;
  int* g_done = P.sched + 2;
  int* w_done = P.sched + 2 + P.n_chunks;
  int* dh_flag = P.sched + 2 + 2 * P.n_chunks;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmHcK); tma_prefetch_desc(&tmWK); tma_prefetch_desc(&tmHcMN);
    tma_prefetch_desc(&tmGMN); tma_prefetch_desc(&tmWMN); tma_prefetch_desc(&tmGK);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull_bar[b], 1); mbar_init(&tempty_bar[b], EPI_THREADS); }
    for (int r = 0; r < RING; ++r) { mbar_init(&rfull_bar[r], 1); mbar_init(&rempty_bar[r], 1 + EPI_THREADS); }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  BwdCounts k;
  k.nv = *g.n_valid;
  k.tiles_tok = (k.nv + BM - 1) / BM;
  k.tiles_d = (g.D + BM - 1) / BM;
  k.tiles_tok256 = (k.nv + BN - 1) / BN;
  k.n_dh = k.tiles_d * k.tiles_tok256;
  const int slot_rows = g.Npad;  // rows per Gbuf slot

  if (warp == 0) {
    if (lane == 0) {
      // ===== scheduler + TMA producer =====
      uint32_t stage = 0, phase = 0;
      uint32_t rslot = 0, rphase = 0;
      while (true) {
        const int q = atomicAdd(queue_head, 1);
        const unsigned long long t_deq = P.trace ? gtimer() : 0ull;
        Item it = decode_item(P, k, q);
        it.q = q;
        it.t_deq = t_deq;
        // dependencies (only on earlier queue entries)
        if (it.type == IT_G) {
          if (it.c >= P.slots) {
            const int wc = it.c - P.slots;
            wait_ge(&w_done[wc], k.n_dh + n_dw_items(k, chunk_width(g, wc)));
          }
        } else if (it.type == IT_DW || it.type == IT_DH) {
          wait_ge(&g_done[it.c], n_g_items(k, it.width));
          if (it.type == IT_DH) wait_ge(&dh_flag[it.tile_id], it.c);
        }
        if (P.strict && it.type != IT_END) wait_ge(done_total, q);  // debug: fully serialised dependencies
        fence_proxy_async_global();
        if (P.trace) it.t_ready = gtimer();
        mbar_wait(&rempty_bar[rslot], rphase ^ 1);
        ring[rslot] = it;
        mbar_arrive(&rfull_bar[rslot]);
        if (++rslot == RING) { rslot = 0; rphase ^= 1; }
        if (it.type == IT_END) break;
        const int slot_row0 = (it.c % P.slots) * slot_rows;
        const int c0 = it.c * g.C;
        for (int kb = 0; kb < it.num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* a = sA + stage * A_BYTES;
          uint8_t* b = sB + stage * B_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);
          if (it.type == IT_G) {
            tma_load_2d(&tmHcK, &full_bar[stage], a, kb * BK, it.mt * BM);
            tma_load_2d(&tmWK, &full_bar[stage], b, kb * BK, c0 + it.nt * BN);
          } else if (it.type == IT_DW) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_2d(&tmHcMN, &full_bar[stage], a + j * 8192, it.mt * BM + j * 64, kb * BK);
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(&tmGMN, &full_bar[stage], b + j * 8192, it.nt * BN + j * 64, slot_row0 + kb * BK);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_2d(&tmWMN, &full_bar[stage], a + j * 8192, it.mt * BM + j * 64, c0 + kb * BK);
            tma_load_2d(&tmGK, &full_bar[stage], b, kb * BK, slot_row0 + it.nt * BN);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      uint32_t stage = 0, phase = 0, rslot = 0, rphase = 0;
      int acc_it = 0;
      while (true) {
        mbar_wait(&rfull_bar[rslot], rphase);
        const Item it = ring[rslot];
        mbar_arrive(&rempty_bar[rslot]);
        if (++rslot == RING) { rslot = 0; rphase ^= 1; }
        if (it.type == IT_END) break;
        if (it.num_kb == 0) continue;
        const uint32_t acc = acc_it & 1, acc_phase = (acc_it >> 1) & 1;
        ++acc_it;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        const bool a_mn = it.type != IT_G;
        const bool b_mn = it.type == IT_DW;
        const uint32_t idesc = idesc_bf16_f32(BM, BN, a_mn ? 1 : 0, b_mn ? 1 : 0);
        for (int kb = 0; kb < it.num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a = smem_u32(sA + stage * A_BYTES);
          const uint32_t b = smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = a_mn ? sdesc_sw128(a + kk * 2048, 8192, 1024) : sdesc_sw128(a + kk * 32, 16, 1024);
            const uint64_t bd = b_mn ? sdesc_sw128(b + kk * 2048, 8192, 1024) : sdesc_sw128(b + kk * 32, 16, 1024);
            umma_bf16(tmem_d, ad, bd, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull_bar[acc]);
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue (128 threads) =====
    EpiCtx e;
    e.q = warp & 3;
    e.half = (warp - 4) >> 2;
    e.row_in_tile = e.q * 32 + lane;
    e.xchg = xchg;
    const bool leader = (threadIdx.x == 128);  // exactly one epilogue thread publishes
    const float scale = k.nv > 0 ? (*g.dloss) / (float)k.nv : 0.f;
    uint32_t rslot = 0, rphase = 0;
    int acc_it = 0;
    while (true) {
      mbar_wait(&rfull_bar[rslot], rphase);
      const Item it = ring[rslot];
      mbar_arrive(&rempty_bar[rslot]);
      if (++rslot == RING) { rslot = 0; rphase ^= 1; }
      if (it.type == IT_END) break;
      const bool have_acc = it.num_kb > 0;
      uint32_t acc = 0;
      if (have_acc) {
        acc = acc_it & 1;
        const uint32_t acc_phase = (acc_it >> 1) & 1;
        ++acc_it;
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
      }
      const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)(e.q * 32) << 16);
      const unsigned long long t_epi0 = P.trace ? gtimer() : 0ull;
      GemmParams gp = g;
      gp.c0 = it.c * g.C;
      gp.width = it.width;
      if (it.type == IT_G) {
        gp.gbuf = g.gbuf + (size_t)(it.c % P.slots) * slot_rows * g.C;
        epilogue_tile<MODE_G>(gp, taddr, e, it.mt, it.nt, k.nv, scale, true);
      } else if (it.type == IT_DW) {
        epilogue_tile<MODE_DW>(gp, taddr, e, it.mt, it.nt, k.nv, scale, have_acc);
      } else {
        gp.dh_accumulate = it.c > 0 ? 1 : 0;
        // DH(c-1, tile) has published (the producer already waited on it; re-acquire
        // here so these threads' .cg loads are ordered after that release)
        if (leader) wait_ge(&dh_flag[it.tile_id], it.c);
        named_bar_sync(2, EPI_THREADS);
        epilogue_tile<MODE_DH>(gp, taddr, e, it.mt, it.nt, k.nv, scale, true);
      }
      if (have_acc) {
        tc_fence_before();
        mbar_arrive(&tempty_bar[acc]);
      }
      // publish completion: all 128 threads' global stores, then one release
      fence_proxy_async_global();
      __threadfence();
      named_bar_sync(1, EPI_THREADS);
      if (leader && P.trace && it.q < P.trace_cap) {
        TraceRec r;
        r.q_type_c = ((unsigned long long)it.q << 32) | ((unsigned long long)it.type << 16) | (unsigned)it.c;
        r.smid = smid();
        r.t_deq = it.t_deq;
        r.t_ready = it.t_ready;
        r.t_epi0 = t_epi0;
        r.t_epi1 = gtimer();
        r.tile = ((unsigned long long)it.mt << 32) | (unsigned)it.nt;
        r.pad = it.num_kb;
        P.trace[it.q] = r;
      }
      if (leader) {
        if (it.type == IT_G) {
          atomicAdd(&g_done[it.c], 1);
        } else {
          if (it.type == IT_DH) atomicExch(&dh_flag[it.tile_id], it.c + 1);
          atomicAdd(&w_done[it.c], 1);
        }
        atomicAdd(done_total, 1);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, TMEM_COLS);
}

constexpr int BWD_SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 512 /*barriers, ring*/ + 1024 /*xchg*/;
static_assert(12 * 8 + 2 * RING * 8 + RING * sizeof(Item) + 4 <= 512, "bwd barrier area");

}  // namespace cce
