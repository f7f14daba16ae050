// cce_quad.cuh -- the CCE hot path on clusters of FOUR CTAs = two CTA pairs that share
// one operand through TMA multicast (SURVEY 8a rows a1-a2 forward, a5-a8 backward).
//
// Why: the pair kernel (cce_pair.cuh) runs the forward at the tensor floor but the
// backward at the L2 throughput ceiling (ncu: ~13 TB/s of L2 sectors in both).  Each
// quad work item gives the two pairs two tiles that share one operand:
//   FWD / G  two row tiles x one vocabulary tile   -> the W tile (B) is shared
//   DW       one vocabulary tile x two hidden tiles -> the G^T tile (A) is shared
//   DH       one row tile x two hidden tiles        -> the G tile (A) is shared
// Each CTA loads half of its share of the common operand and multicasts it to itself
// and to the matching CTA of the other pair, so per-CTA L2->SM traffic drops from 32 KB
// to 24 KB per 64-wide k-block (-25%), for the same tensor work.
//
// Everything else follows cce_pair.cuh: pair MMAs (cta_group::2, M = 256), 6-stage TMA
// ring, double-buffered TMEM accumulators, a scheduler warp (cluster rank 0) feeding a
// 4-deep item ring in all four CTAs, warp-specialised producer / MMA / epilogue.
// Differences: an SMEM stage is only refilled when BOTH pairs have consumed it (its
// empty barrier counts one tcgen05.commit from each pair leader; commits are
// multicast to all four CTAs); accumulator barriers stay per pair.
#pragma once
#include "cce_pair.cuh"

namespace cce {
namespace quadk {

using pairk::HM;
using pairk::PA_BYTES;
using pairk::PB_BYTES;
using pairk::PEPI_THREADS;
using pairk::PEPI_WARPS;
using pairk::PM;
using pairk::PN;
using pairk::PRING;
using pairk::PSTAGE_BYTES;
using pairk::PSTAGES;
using pairk::PT_DH;
using pairk::PT_DW;
using pairk::PT_END;
using pairk::PT_FWD;
using pairk::PT_G;

constexpr int QTHREADS = pairk::PTHREADS;
constexpr int QSMEM = pairk::PSMEM;

// One quad item: common fields + one sub-tile per pair.
struct QItem {
  int type, c, num_kb, q;
  int m0[2], n0[2], N[2], tile_id[2], active[2];
  int pad[2];
  unsigned long long t_deq, t_ready;
};
static_assert(sizeof(QItem) == 80, "QItem layout");
static_assert(24 * 8 + PRING * sizeof(QItem) + 4 <= 1024, "quad barrier + ring area");

struct QCounts {
  int nv, t256, tq, n_dt, n_dq, n_dh, tv;
};

__device__ __forceinline__ QItem q_make(int type, int c, int num_kb, int q) {
  QItem it;
  it.type = type; it.c = c; it.num_kb = num_kb; it.q = q;
#pragma unroll
  for (int p = 0; p < 2; ++p) { it.m0[p] = 0; it.n0[p] = 0; it.N[p] = 128; it.tile_id[p] = 0; it.active[p] = 0; }
  it.pad[0] = it.pad[1] = 0;
  it.t_deq = 0; it.t_ready = 0;
  return it;
}

__device__ __forceinline__ int q_n_g(const QCounts& k, int w) { return k.tq * ((w + PN - 1) / PN); }
__device__ __forceinline__ int q_n_dw(const QCounts& k, int w) { return ((w + PM - 1) / PM) * k.n_dq; }

// Forward: vocabulary tile outer, row-tile PAIR inner.  Backward: G0, G1, W0, G2, W1,
// ..., W_{n-1} (W_c = DH items then DW items), as in the pair kernel.
__device__ QItem q_decode(const pairk::PairParams& P, const QCounts& k, int q) {
  const GemmParams& g = P.g;
  if (P.mode == 0) {
    if (q >= k.tq * k.tv) return q_make(PT_END, 0, 0, q);
    QItem it = q_make(PT_FWD, 0, g.D / BK, q);
    const int tp = q % k.tq, v = q / k.tq;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int t = 2 * tp + p;
      it.m0[p] = t * PM; it.n0[p] = v * PN; it.N[p] = PN; it.active[p] = t < k.t256;
    }
    return it;
  }
  const int n = P.n_chunks;
  int r = q;
  for (int ph = 0; ph < 2 * n; ++ph) {
    int isG, c;
    if (ph == 0) { isG = 1; c = 0; }
    else if (ph == 2 * n - 1) { isG = 0; c = n - 1; }
    else if (ph & 1) { isG = 1; c = (ph + 1) / 2; }
    else { isG = 0; c = ph / 2 - 1; }
    const int w = pairk::p_chunk_width(g, c);
    const int c0 = c * g.C;
    if (isG) {
      const int cnt = q_n_g(k, w);
      if (r < cnt) {
        QItem it = q_make(PT_G, c, g.D / BK, q);
        const int tp = r % k.tq, vt = r / k.tq;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const int t = 2 * tp + p;
          it.m0[p] = t * PM; it.n0[p] = c0 + vt * PN; it.N[p] = PN; it.active[p] = t < k.t256;
        }
        return it;
      }
      r -= cnt;
    } else {
      if (r < k.n_dh) {
        QItem it = q_make(PT_DH, c, (w + BK - 1) / BK, q);
        const int t = r / k.n_dq, dq = r % k.n_dq;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const int dt = 2 * dq + p;
          it.active[p] = dt < k.n_dt;
          it.m0[p] = t * PM; it.n0[p] = dt * PN;
          it.N[p] = it.active[p] ? pairk::dtile_N(g.D, dt) : 128;
          it.tile_id[p] = t * k.n_dt + dt;
        }
        return it;
      }
      r -= k.n_dh;
      const int cnt = q_n_dw(k, w);
      if (r < cnt) {
        QItem it = q_make(PT_DW, c, (k.nv + BK - 1) / BK, q);
        const int vt = r / k.n_dq, dq = r % k.n_dq;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const int dt = 2 * dq + p;
          it.active[p] = dt < k.n_dt;
          it.m0[p] = vt * PM; it.n0[p] = dt * PN;
          it.N[p] = it.active[p] ? pairk::dtile_N(g.D, dt) : 128;
        }
        return it;
      }
      r -= cnt;
    }
  }
  return q_make(PT_END, 0, 0, q);
}

// The pair kernel's epilogues take a PItem; build the view of this pair's sub-tile.
__device__ __forceinline__ pairk::PItem sub_item(const QItem& it, int p) {
  pairk::PItem s = pairk::make_item(it.type, it.c, it.m0[p], it.n0[p], it.N[p], it.num_kb, it.tile_id[p], it.q);
  return s;
}

template <bool A_MN, bool B_MN, int NP>
__device__ __forceinline__ void q_mma_item(int N, int num_kb, uint64_t* full_bar, uint64_t* empty_bar,
                                           uint32_t a_base, uint32_t b_base, uint32_t tmem_d, uint32_t& stage,
                                           uint32_t& phase, unsigned long long* wait_ns) {
  const uint32_t idesc = idesc_bf16_f32(PM, N, A_MN ? 1 : 0, B_MN ? 1 : 0);
  for (int kb = 0; kb < num_kb; ++kb) {
    if (wait_ns) {
      const unsigned long long w0 = gtimer();
      mbar_wait(&full_bar[stage], phase);
      *wait_ns += gtimer() - w0;
    }
    mbar_wait(&full_bar[stage], phase);
    tc_fence_after();
    const uint64_t ad = sdesc_sw128(a_base + stage * PA_BYTES, A_MN ? 8192 : 16, 1024);
    const uint64_t bd = sdesc_sw128(b_base + stage * PB_BYTES, B_MN ? 8192 : 16, 1024);
    if (elect_one()) {
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk)
        umma_bf16_pair(tmem_d, ad + (uint64_t)(A_MN ? 128 * kk : 2 * kk), bd + (uint64_t)(B_MN ? 128 * kk : 2 * kk),
                       idesc, (kb | kk) ? 1u : 0u);
      // every pair of the cluster must release a stage (multicast slots)
      umma_commit_mask(&empty_bar[stage], NP == 2 ? 0xF : 0x3);
    }
    __syncwarp();
    if (++stage == PSTAGES) { stage = 0; phase ^= 1; }
  }
}

// NP = pairs per cluster.  NP = 2: the quad kernel proper (4-CTA clusters, shared
// operand multicast).  NP = 1: the same queue consumed by ONE CTA pair, which runs the
// item's two sub-tiles one after the other and loads the common operand itself.  A
// 4-CTA cluster cannot use every SM (GPCs hold 16-22 SMs: 33 clusters = 132 of 148
// SMs on B200), so the host co-launches NP = 1 clusters on the stranded SMs; both
// kernels pull from the one work queue and count 4 completions per item (NP = 2:
// 4 CTAs x 1; NP = 1: 2 CTAs x 2 sub-tiles), so the dependency protocol is unchanged.
template <int NP>
__global__ void __launch_bounds__(QTHREADS, 1)
    cce_quad_kernel(const __grid_constant__ CUtensorMap tmHcK, const __grid_constant__ CUtensorMap tmWK64,
                    const __grid_constant__ CUtensorMap tmGMN, const __grid_constant__ CUtensorMap tmHcMN,
                    const __grid_constant__ CUtensorMap tmGK64, const __grid_constant__ CUtensorMap tmWMN,
                    const __grid_constant__ CUtensorMap tmDH, const pairk::PairParams P) {
  static_assert(NP == 1 || NP == 2, "pairs per cluster");
  constexpr int NCTA = 2 * NP;
  constexpr int NSUB = NP == 2 ? 1 : 2;  // sub-tiles each pair runs per item
  const GemmParams& g = P.g;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + PSTAGES * PA_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + PSTAGES * PSTAGE_BYTES);
  uint64_t* empty_bar = full_bar + PSTAGES;
  uint64_t* tfull_bar = empty_bar + PSTAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* rfull_bar = tempty_bar + 2;
  uint64_t* rempty_bar = rfull_bar + PRING;  // rank 0 only: all consumers of all CTAs
  QItem* ring = reinterpret_cast<QItem*>(rempty_bar + PRING);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + PRING);
  float* xchg = reinterpret_cast<float*>(smem + PSTAGES * PSTAGE_BYTES + 1024);
  uint8_t* stage_base = smem + PSTAGES * PSTAGE_BYTES + 2048;

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int pr = rank & 1;          // rank within the pair
  const int pp = rank >> 1;         // which pair (sub-tile) this CTA works on (NP = 2)
  const uint32_t pair_leader = rank & ~1u;
  int* head = P.sched;
  int* done_total = P.sched + 1;
  int* g_done = P.sched + 2;
  int* w_done = P.sched + 2 + P.n_chunks;
  int* dh_flag = P.sched + 2 + 2 * P.n_chunks;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmHcK); tma_prefetch_desc(&tmWK64);
    if (P.mode == 1) {
      tma_prefetch_desc(&tmGMN); tma_prefetch_desc(&tmHcMN); tma_prefetch_desc(&tmGK64); tma_prefetch_desc(&tmWMN);
      tma_prefetch_desc(&tmDH);
    }
    for (int s = 0; s < PSTAGES; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], NP); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull_bar[b], 1); mbar_init(&tempty_bar[b], 2 * PEPI_WARPS); }
    for (int r = 0; r < PRING; ++r) {
      mbar_init(&rfull_bar[r], 1);
      // consumers per item: NCTA producers + NP MMA warps + NCTA x 8 epilogue warps
      mbar_init(&rempty_bar[r], NCTA + NP + NCTA * PEPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, TMEM_COLS);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  QCounts k;
  k.nv = *g.n_valid;
  k.t256 = (k.nv + PM - 1) / PM;
  k.tq = (k.t256 + 1) / 2;
  k.n_dt = (g.D + PN - 1) / PN;
  k.n_dq = (k.n_dt + 1) / 2;
  k.n_dh = k.t256 * k.n_dq;
  k.tv = (g.V_local + PN - 1) / PN;
  const int slot_rows = g.Npad;
  const uint32_t rempty0 = mapa_shared(smem_u32(&rempty_bar[0]), 0);

  if (warp == 3) {
    if (lane == 0 && rank == 0) {
      // ===== scheduler: dequeue quad items, publish them into every CTA's ring =====
      uint32_t rs = 0, rph = 0;
      while (true) {
        const int q = atomicAdd(head, 1);
        QItem it = q_decode(P, k, q);
        // debug bits 256 / 512 / 1024: run only the G / DW / DH items (no dependencies;
        // measures one item type's throughput in isolation, results are garbage)
        if ((P.strict & 1792) && it.type != PT_END && !((P.strict >> (8 + it.type - PT_G)) & 1)) continue;
        if (P.trace) it.t_deq = gtimer();
        mbar_wait(&rempty_bar[rs], rph ^ 1);
        ring[rs] = it;
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&it);
        for (int dst = 1; dst < NCTA; ++dst) {
          const uint32_t remote = mapa_shared(smem_u32(&ring[rs]), dst);
#pragma unroll
          for (int i = 0; i < (int)(sizeof(QItem) / 4); ++i) st_cluster_u32(remote + 4 * i, w[i]);
        }
        mbar_arrive(&rfull_bar[rs]);
        for (int dst = 1; dst < NCTA; ++dst) mbar_arrive_cluster(mapa_shared(smem_u32(&rfull_bar[rs]), dst));
        if (++rs == PRING) { rs = 0; rph ^= 1; }
        if (it.type == PT_END) break;
      }
    }
  } else if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (every CTA) =====
      uint32_t stage = 0, phase = 0, rs = 0, rph = 0;
      const uint32_t full_leader0 = mapa_shared(smem_u32(&full_bar[0]), pair_leader);
      const uint32_t full_local0 = smem_u32(&full_bar[0]);
      const uint16_t mc = (uint16_t)((1u << rank) | (1u << (rank ^ 2u)));  // me + my counterpart (NP = 2)
      while (true) {
        mbar_wait_cluster(&rfull_bar[rs], rph);
        const QItem it = ring[rs];
        mbar_arrive_cluster_relaxed(rempty0 + rs * 8);
        if (++rs == PRING) { rs = 0; rph ^= 1; }
        if (it.type == PT_END) break;
        if (P.mode == 1 && !(P.strict & 1792)) {
          if (P.strict & 1) wait_ge(done_total, 4 * it.q);
          if (it.type == PT_G) {
            if (it.c >= P.slots) {
              const int wc = it.c - P.slots;
              wait_ge(&w_done[wc], 4 * (k.n_dh + q_n_dw(k, pairk::p_chunk_width(g, wc))));
            }
          } else {
            wait_ge(&g_done[it.c], 4 * q_n_g(k, pairk::p_chunk_width(g, it.c)));
            // DH(c, tile) after DH(c-1, tile) is enforced at the epilogue's reduce only;
            // debug bit 8 also holds the operand loads back (the old RMW protocol)
            if (it.type == PT_DH && (P.strict & 8)) {
#pragma unroll
              for (int p = 0; p < 2; ++p)
                if (it.active[p]) wait_ge(&dh_flag[it.tile_id[p]], 2 * it.c);
            }
          }
          fence_proxy_async_global();
        }
        if (P.trace && rank == 0 && it.q < P.trace_cap) P.trace[it.q].t_ready = gtimer();
        const int hr = pr * HM;                 // this CTA's first tile row of its pair's tile
        const int slot_blk0 = (it.c % P.slots) * (g.C / 64);
        const int c0 = it.c * g.C;
        unsigned long long tl0 = 0;
        for (int sp = 0; sp < NSUB; ++sp) {
          const int p = NP == 2 ? pp : sp;      // the sub-tile this pass loads
          if (NP == 1 && !it.active[p]) continue;
          const int N = it.N[p];
          const int hn = pr * (N / 2);          // this CTA's first B row / column
          const int b_bytes = (N / 2) * BK * 2;
          const int m0 = it.m0[p], n0 = it.n0[p];
          for (int kb = 0; kb < it.num_kb; ++kb) {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            if (P.trace && kb == 0 && sp == 0) tl0 = gtimer();
            uint8_t* a = sA + stage * PA_BYTES;
            uint8_t* b = sB + stage * PB_BYTES;
            const uint32_t fb = full_leader0 + stage * 8;
            const uint32_t fl = full_local0 + stage * 8;
            if (pr == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * (PA_BYTES + b_bytes));
            // L2 prefetch of the HBM-resident dlogits operand only (the other operand of
            // DW / DH items is L2-resident and a prefetch would only add L2 requests)
            const int pk = kb + P.prefetch;
            if (NP == 2 && P.prefetch > 0 && pk < it.num_kb) {
              if (it.type == PT_DW) tma_prefetch_3d(&tmGMN, 0, pk * BK, slot_blk0 + (m0 + hr) / 64 + pp);
              else if (it.type == PT_DH) tma_prefetch_3d(&tmGK64, 0, m0 + hr + pp * 64, slot_blk0 + pk);
            }
            if (it.type == PT_FWD || it.type == PT_G) {
              // A (rows) private to the pair; B (vocabulary rows) common: with NP = 2 this CTA
              // loads the 64-row half `pp` of its 128-row share and multicasts it to its
              // counterpart; with NP = 1 it loads both halves
              tma_load_2d_pair(&tmHcK, fb, a, kb * BK, m0 + hr);
              if (NP == 2) {
                tma_load_2d_pair_mc(&tmWK64, fl, b + pp * 8192, kb * BK, n0 + hn + pp * 64, mc);
              } else {
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) tma_load_2d_pair(&tmWK64, fb, b + h2 * 8192, kb * BK, n0 + hn + h2 * 64);
              }
            } else if (it.type == PT_DW) {
              // A = G^T (vocabulary block) common: 64-column box `pp` (NP = 2) or both
              if (NP == 2) {
                tma_load_3d_pair_mc(&tmGMN, fl, a + pp * 8192, 0, kb * BK, slot_blk0 + (m0 + hr) / 64 + pp, mc);
              } else {
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2)
                  tma_load_3d_pair(&tmGMN, fb, a + h2 * 8192, 0, kb * BK, slot_blk0 + (m0 + hr) / 64 + h2);
              }
              for (int j = 0; j < N / 2 / 64; ++j)
                tma_load_2d_pair(&tmHcMN, fb, b + j * 8192, n0 + hn + j * 64, kb * BK);
            } else {  // PT_DH: A = G rows common (64-row half `pp`, or both), B = W chunk columns private
              if (NP == 2) {
                tma_load_3d_pair_mc(&tmGK64, fl, a + pp * 8192, 0, m0 + hr + pp * 64, slot_blk0 + kb, mc);
              } else {
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2)
                  tma_load_3d_pair(&tmGK64, fb, a + h2 * 8192, 0, m0 + hr + h2 * 64, slot_blk0 + kb);
              }
              for (int j = 0; j < N / 2 / 64; ++j)
                tma_load_2d_pair(&tmWMN, fb, b + j * 8192, n0 + hn + j * 64, c0 + kb * BK);
            }
            if (++stage == PSTAGES) { stage = 0; phase ^= 1; }
          }
        }
        if (P.trace && rank == 0 && it.q < P.trace_cap) {
          P.trace[it.q].t_load0 = tl0;
          P.trace[it.q].t_load1 = gtimer();
        }
      }
    }
  } else if (warp == 1) {
    if (pr == 0) {
      // ===== MMA issuer (every pair leader; whole warp, elected lane issues) =====
      uint32_t stage = 0, phase = 0, rs = 0, rph = 0;
      int acc_it = 0;
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      const uint16_t pair_mask = (uint16_t)(3u << (2 * pp));
      while (true) {
        mbar_wait_cluster(&rfull_bar[rs], rph);
        const QItem it = ring[rs];
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster_relaxed(rempty0 + rs * 8);
        if (++rs == PRING) { rs = 0; rph ^= 1; }
        if (it.type == PT_END) break;
        if (it.num_kb == 0) continue;
        const bool tr = P.trace && rank == 0 && it.q < P.trace_cap;
        unsigned long long fw = 0;
        const unsigned long long tm0 = tr ? gtimer() : 0ull;
        const unsigned long long cm0 = tr ? clock64() : 0ull;
        for (int sp = 0; sp < NSUB; ++sp) {
          const int p = NP == 2 ? pp : sp;
          if (NP == 1 && !it.active[p]) continue;
          const uint32_t acc = acc_it & 1, acc_phase = (acc_it >> 1) & 1;
          ++acc_it;
          mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t tmem_d = tmem_base + acc * PN;
          const int N = it.N[p];
          if (it.type == PT_DW)
            q_mma_item<true, true, NP>(N, it.num_kb, full_bar, empty_bar, a_base, b_base, tmem_d, stage, phase,
                                       tr ? &fw : nullptr);
          else if (it.type == PT_DH)
            q_mma_item<false, true, NP>(N, it.num_kb, full_bar, empty_bar, a_base, b_base, tmem_d, stage, phase,
                                        tr ? &fw : nullptr);
          else
            q_mma_item<false, false, NP>(N, it.num_kb, full_bar, empty_bar, a_base, b_base, tmem_d, stage, phase,
                                         tr ? &fw : nullptr);
          if (elect_one()) umma_commit_mask(&tfull_bar[acc], pair_mask);
          __syncwarp();
        }
        if (tr && lane == 0) {
          P.trace[it.q].t_mma0 = tm0;
          P.trace[it.q].t_mma1 = gtimer();
          P.trace[it.q].t_full_wait = fw;
          P.trace[it.q].r0 = clock64() - cm0;
        }
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue (every CTA) =====
    pairk::PEpi e;
    e.q = warp & 3;
    e.half = (warp - 4) >> 2;
    e.rit = e.q * 32 + lane;
    e.rank = pr;  // the pair epilogues index rows by the rank within the pair
    e.xchg = xchg;
    e.xz = reinterpret_cast<float*>(stage_base);  // forward items never use the store staging
    e.stage = stage_base + (warp - 4) * 4096;
    const bool leader = (threadIdx.x == 128);
    const float scale = (P.mode == 1 && k.nv > 0 && g.reduction != 2)
                            ? (g.reduction == 1 ? *g.dloss : (*g.dloss) / (float)k.nv)
                            : 0.f;  // reduction "none": per-row dloss_c in epi_g
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty_bar[0]), pair_leader);
    uint32_t rs = 0, rph = 0;
    int acc_it = 0;
    while (true) {
      mbar_wait_cluster(&rfull_bar[rs], rph);
      const QItem qit = ring[rs];
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(rempty0 + rs * 8);
      if (++rs == PRING) { rs = 0; rph ^= 1; }
      if (qit.type == PT_END) break;
      const bool have_acc = qit.num_kb > 0;
      for (int sp = 0; sp < NSUB; ++sp) {
        const int p = NP == 2 ? pp : sp;
        const bool active = qit.active[p] != 0;
        // NP = 1 skips inactive sub-tiles entirely (no MMAs were issued for them)
        const bool use_acc = have_acc && (NP == 2 || active);
        uint32_t acc = 0;
        if (use_acc) {
          acc = acc_it & 1;
          const uint32_t acc_phase = (acc_it >> 1) & 1;
          ++acc_it;
          mbar_wait(&tfull_bar[acc], acc_phase);
          tc_fence_after();
        }
        const pairk::PItem it = sub_item(qit, p);
        const uint32_t taddr = tmem_base + acc * PN + ((uint32_t)(e.q * 32) << 16);
        const unsigned long long t_epi0 = P.trace ? gtimer() : 0ull;
        if (!active) {
          // out-of-range sub-tile (odd tile counts): no output
        } else if (it.type == PT_FWD) {
          pairk::epi_fwd(g, taddr, e, it, k.nv);
        } else if (it.type == PT_G) {
          pairk::epi_g(g, taddr, e, it, k.nv, scale, g.gbuf + (size_t)(it.c % P.slots) * slot_rows * g.C, nullptr, 0);
        } else if (it.type == PT_DW) {
          pairk::epi_dw(g, taddr, e, it, have_acc);
        } else {
          if (leader && !(P.strict & 1792)) wait_ge(&dh_flag[it.tile_id], 2 * it.c);
          named_bar_sync(2, PEPI_THREADS);
          fence_proxy_async_global();  // the acquired flag orders the TMA reduce below
          pairk::epi_dh_tma(&tmDH, taddr, e, it);
        }
        if (use_acc) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (pr == 0) mbar_arrive(&tempty_bar[acc]);
            else mbar_arrive_cluster_relaxed(tempty_leader0 + acc * 8);
          }
        }
        if (P.trace && leader && rank == 0 && sp == 0 && qit.q < P.trace_cap) {
          TraceRec& r = P.trace[qit.q];
          r.q_type_c = ((unsigned long long)qit.q << 32) | ((unsigned long long)qit.type << 16) | (unsigned)qit.c;
          r.smid = smid();
          r.t_deq = qit.t_deq;
          r.t_epi0 = t_epi0;
          r.t_epi1 = gtimer();
          r.tile = ((unsigned long long)qit.m0[0] << 32) | (unsigned)qit.n0[0];
          // k-blocks this cluster's MMA window covered (NP = 1 runs both sub-tiles)
          r.pad = NP == 2 ? qit.num_kb : qit.num_kb * ((qit.active[0] != 0) + (qit.active[1] != 0));
          r.r1 = NP;
        }
        if (P.mode == 1) {
          // publish this CTA's share of the sub-tile (4 completions per item in total)
          fence_proxy_async_global();
          named_bar_sync(1, PEPI_THREADS);
          if (leader) {
            __threadfence();
            if (it.type == PT_G) atomicAdd(&g_done[it.c], 1);
            else {
              if (it.type == PT_DH && active) atomicAdd(&dh_flag[it.tile_id], 1);
              atomicAdd(&w_done[it.c], 1);
            }
            atomicAdd(done_total, 1);
          }
        }
      }
    }
  }

  __syncwarp();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair(tmem_base, TMEM_COLS);
}

}  // namespace quadk
}  // namespace cce
