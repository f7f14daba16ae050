// cce_pair.cuh -- the CCE hot path on CTA PAIRS: one persistent kernel, launched in
// clusters of 2, that runs either the forward queue (logit tiles + online-softmax
// epilogue) or the backward queue (recompute + dlogits, dW,
// dH, rows a5-a8) with tcgen05.mma.cta_group::2.
//
// Why pairs: a 1-CTA 128x256 tile loads 48 KB of operands per 64-wide k-block and
// was measured L2->SM bandwidth bound (~100 GB/s per SM, 0.48-0.61 us per k-block
// against a 0.27 us tensor floor).  A pair computes a 256 x N tile with M=256 MMAs:
// each CTA loads its own 128 rows of A and N/2 rows of B (32 KB per k-block at
// N=256), i.e. 1.5x less operand traffic for the same tensor work.
//
// Roles (384 threads per CTA):
//   warp 0   TMA producer (both CTAs): item from the local ring, dependency waits,
//            loads of this CTA's operand halves (the leader arms each full barrier
//            with both CTAs' transaction bytes)
//   warp 1   leader: MMA issuer (one thread, cta_group::2); peer: idle
//   warp 2   TMEM allocator (cta_group::2, 512 columns = 2 x 256 fp32 accumulators)
//   warp 3   leader: scheduler -- dequeues items from the global queue and publishes
//            them into both CTAs' rings up to 4 items ahead
//   warps 4-11  epilogue: warp w reads TMEM lane quarter w%4 and column half (w-4)/4
// The leader dequeues an item, checks its dependencies, and broadcasts it into
// both CTAs' 4-entry item rings (the peer's over DSMEM with release/acquire
// cluster-scope mbarriers).  Full barriers live in the leader; each CTA's TMA
// signals its bytes there.  MMA completion is multicast to both CTAs' empty /
// accumulator-full barriers; both epilogues report accumulator-empty to the leader.
//
// Tile orientation (all types: M = 256 per pair, accumulator row = TMEM lane):
//   FWD  S  = Hc W^T           M = rows,  N = vocab (256), K = D    A,B K-major
//   G    S  = Hc W_c^T -> G    M = rows,  N = vocab (256), K = D    A,B K-major
//   DW   dW = G^T Hc           M = vocab, N = hidden (<=256), K = rows   A,B MN-major
//   DH   dH += G W_c           M = rows,  N = hidden (<=256), K = vocab  A K-, B MN-major
// The chunk dlogits G live in a column-blocked ring [slot][C/64][Npad][64] (bf16), so
// every TMA box of G and every epilogue store is one contiguous run in HBM.
// Hidden-dimension tiles are 256 wide with a 128-wide tail (D = 896 -> 256,256,256,128),
// so no MMA work is wasted and dW / dH rows are written as contiguous vectors.
#pragma once
#include "cce_common.cuh"
#include "cce_p2p.cuh"

namespace cce {
namespace pairk {

constexpr int PM = 256;                  // tile rows per pair
constexpr int HM = 128;                  // tile rows per CTA
constexpr int PN = 256;                  // max tile columns
constexpr int PSTAGES = 6;
constexpr int PA_BYTES = HM * BK * 2;        // 16 KB
constexpr int PB_BYTES = (PN / 2) * BK * 2;  // 16 KB
constexpr int PSTAGE_BYTES = PA_BYTES + PB_BYTES;
constexpr int PRING = 4;
// KPS k-blocks (64 wide) per ring stage, loaded with one 3-D TMA box per operand: the
// per-k-block cost of the single-thread producer (TMA issue, expect_tx, barrier round
// trip) was the limit -- KPS = 2 (3 stages x 64 KB) took the backward's dW / dH / G items
// from 677 / 711 / 684 to 522 / 524 / 572 cycles per k-block (floor 512).
constexpr int KPS = 2;
static_assert(PSTAGES % KPS == 0, "k-blocks per stage");
constexpr int KSTAGES = PSTAGES / KPS;
constexpr int KA_BYTES = KPS * PA_BYTES;
constexpr int KB_BYTES = KPS * PB_BYTES;
constexpr int PEPI_WARPS = 8;
constexpr int PEPI_THREADS = 32 * PEPI_WARPS;
constexpr int PTHREADS = 128 + PEPI_THREADS;
constexpr int PSMEM = PSTAGES * PSTAGE_BYTES + 1024 /*align*/ + 1024 /*barriers+rings*/ + 1024 /*xchg*/ +
                      PEPI_WARPS * 4096 /*epilogue store staging*/;
static_assert(PSMEM <= 232448, "pair kernel shared memory");

// PT_RED (P2P backward): the cross-rank sum of one dH tile, queued after every MMA item
enum PType : int { PT_FWD = 0, PT_G = 1, PT_DW = 2, PT_DH = 3, PT_END = 4, PT_RED = 5 };

struct PItem {
  int type, c, m0, n0, N, num_kb, tile_id, q;
  unsigned long long t_deq, t_ready;
};
static_assert(sizeof(PItem) == 48, "PItem layout");

struct PairParams {
  GemmParams g;
  int mode;        // 0 = forward queue, 1 = backward queue
  int n_chunks;
  int part;        // backward: 0 the whole queue; 1 every item but the last chunk's DW items;
                   // 2 only those (the NCCL dH all-reduce runs between the two launches, on a
                   // side stream, overlapping part 2)
  int slots;       // Gbuf ring slots
  int lookahead;   // backward queue: G of chunk block b + lookahead is queued before W of block b
  int qblock;      // chunks per block of the backward queue ((lookahead + 1) * qblock <= slots)
  // CCE_FLAG_P2P_COMBINE, fused into this kernel (P2P instantiation): when rank r's last-chunk
  // DH(tile) is complete it raises ready[r][tile] in every rank; RED(tile) items (tiles
  // tile % world == rank, queued last) wait for every rank's ready flag, sum the tile's partial
  // dH over the ranks in rank order (loads from peer memory), store the sum into every rank's
  // reduced array and raise done[tile][cta] in every rank -- the exchange overlaps the
  // remaining MMA items tile by tile.
  PeerPtrs peers;
  int world, prank, epoch, tmax;             // tmax: tile capacity of the flag arrays
  unsigned long long ready_off, done_off;    // int flag arrays in every workspace
  unsigned long long dH32_off, dHred_off;    // partial / reduced dH in every workspace
  int* err;                                  // error word (bit 2: a peer never signalled)
  // the last jit_tail items of the queue are dequeued just in time: the scheduler claims the
  // next item only once this pair's producer has reached the last stage of the previous one,
  // so no pair holds claimed-but-unstarted items while others run out of work (the tail)
  int jit_tail;
  int* sched;      // zeroed: [0] head [1] head of part 2 | g_done[n] | w_done[n] | dh_flag[n_dt * t256]
  TraceRec* trace;
  int trace_cap;
};

struct PCounts {
  int nv, t256, n_dt, n_dh, tv;
  int rg;  // row tiles per L2 group (the FWD / G items of a group share its Hc rows through L2)
};

// Hc rows of one L2 group: the forward and G items sweep the vocabulary tiles over a group of
// row tiles whose Hc block (32 MB) stays L2-resident, then move to the next group.  Sweeping ALL rows
// per vocabulary tile re-reads Hc from DRAM once per vocabulary tile when Hc exceeds the L2
// (configs[4] shard: N = 32768, D = 3584, Hc = 235 MB -> 17.8 GB of DRAM reads per forward);
// grouping re-reads only the (vocabulary) operand once per group instead.  At D = 896 every
// row tile fits one group: the order is unchanged.
#ifndef CCE_L2_GROUP_MB
#define CCE_L2_GROUP_MB 32
#endif
constexpr long long L2_GROUP_BYTES = (long long)CCE_L2_GROUP_MB << 20;  // 16 / 32 / 48 / 80 MB A/B: profiles/r02b_l2_group_size.txt
__device__ __forceinline__ int l2_group_rows(int t256, int D) {
  const long long per_tile = (long long)PM * D * 2;
  const int rg = (int)(L2_GROUP_BYTES / per_tile);
  return rg < 1 ? 1 : (rg > t256 ? t256 : rg);
}

// item index i of a (row tiles x vocabulary tiles) block swept group by group: vocabulary
// tile outer, row tile inner within a group of rg row tiles
__device__ __forceinline__ void grouped_tile(int i, int t256, int rg, int ntv, int& row_tile, int& vtile) {
  const int per_group = rg * ntv;
  const int grp = i / per_group, ii = i - grp * per_group;
  const int rows_in = min(rg, t256 - grp * rg);
  vtile = ii / rows_in;
  row_tile = grp * rg + (ii - vtile * rows_in);
}

__device__ __forceinline__ int dtile_N(int D, int dt) {
  const int rem = D - dt * PN;
  return rem >= PN ? PN : ((rem + 127) / 128) * 128;
}

__device__ __forceinline__ PItem make_item(int type, int c, int m0, int n0, int N, int num_kb, int tile_id, int q) {
  PItem it;
  it.type = type; it.c = c; it.m0 = m0; it.n0 = n0; it.N = N; it.num_kb = num_kb; it.tile_id = tile_id; it.q = q;
  it.t_deq = 0; it.t_ready = 0;
  return it;
}

__device__ __forceinline__ int p_chunk_width(const GemmParams& g, int c) {
  const int rem = g.V_local - c * g.C;
  return rem < g.C ? rem : g.C;
}
__device__ __forceinline__ int p_n_g(const PCounts& k, int w) { return k.t256 * ((w + PN - 1) / PN); }
__device__ __forceinline__ int p_n_dw(const PCounts& k, int w) { return ((w + PM - 1) / PM) * k.n_dt; }

// Forward queue: vocabulary tile outer, row tile inner (all row tiles share one W tile in L2).
// Backward queue: G0, G1, W0, G2, W1, ..., W_{n-1}   (W_c = DH(c) items, then DW(c) items).
__device__ PItem decode(const PairParams& P, const PCounts& k, int q) {
  const GemmParams& g = P.g;
  if (P.mode == 0) {
    if (q < k.t256 * k.tv) {
      int rt, vt;
      grouped_tile(q, k.t256, k.rg, k.tv, rt, vt);
      return make_item(PT_FWD, 0, rt * PM, vt * PN, PN, g.D / BK, 0, q);
    }
    return make_item(PT_END, 0, 0, 0, 0, 0, 0, q);
  }
  // chunk blocks of B = P.qblock chunks: G(blocks 0 .. L-1), then for each block b:
  // G(block b + L), W(block b)   (L = P.lookahead; (L + 1) B <= slots)
  const int n = P.n_chunks;
  const int L = P.lookahead, B = P.qblock;
  const int nb = (n + B - 1) / B;
  int r = q;
  for (int ph = 0; ph < (L + 2 * nb) * B; ++ph) {
    const int blk_ph = ph / B, j = ph % B;
    int isG, c;
    if (blk_ph < L) { isG = 1; c = blk_ph * B + j; }
    else {
      const int t = blk_ph - L;
      isG = (t & 1) == 0;
      c = ((t >> 1) + (isG ? L : 0)) * B + j;
    }
    if (c >= n) continue;
    const int w = p_chunk_width(g, c);
    const int c0 = c * g.C;
    if (isG) {
      const int cnt = p_n_g(k, w);
      if (r < cnt) {
        int rt, vt;
        grouped_tile(r, k.t256, k.rg, (w + PN - 1) / PN, rt, vt);
        return make_item(PT_G, c, rt * PM, c0 + vt * PN, PN, g.D / BK, 0, q);
      }
      r -= cnt;
    } else {
      if (r < k.n_dh) {
        const int dt = r % k.n_dt;
        return make_item(PT_DH, c, (r / k.n_dt) * PM, dt * PN, dtile_N(g.D, dt), (w + BK - 1) / BK, r, q);
      }
      r -= k.n_dh;
      const int cnt = p_n_dw(k, w);
      if (r < cnt) {
        const int dt = r % k.n_dt;
        return make_item(PT_DW, c, (r / k.n_dt) * PM, dt * PN, dtile_N(g.D, dt), (k.nv + BK - 1) / BK, 0, q);
      }
      r -= cnt;
    }
  }
  // P2P: this rank's share of the cross-rank dH reduction, after every MMA item
  if (P.world > 1 && P.peers.ws[0] != nullptr) {
    const int tile = P.prank + r * P.world;
    if (tile < k.n_dh) {
      const int dt = tile % k.n_dt;
      return make_item(PT_RED, n - 1, (tile / k.n_dt) * PM, dt * PN, dtile_N(g.D, dt), 0, tile, q);
    }
  }
  return make_item(PT_END, 0, 0, 0, 0, 0, 0, q);
}

// Queue positions [0, total): every item before PT_END (the P2P RED items included).
__device__ __forceinline__ int queue_total(const PairParams& P, const PCounts& k) {
  if (P.mode == 0) return k.t256 * k.tv;
  int total = 0;
  for (int c = 0; c < P.n_chunks; ++c) {
    const int w = p_chunk_width(P.g, c);
    total += p_n_g(k, w) + k.n_dh + p_n_dw(k, w);
  }
  if (P.world > 1 && P.peers.ws[0] != nullptr && k.n_dh > P.prank) total += (k.n_dh - P.prank + P.world - 1) / P.world;
  return total;
}

// ------------------------------------------------------------------ epilogues (per CTA)
struct PEpi {
  int rit;      // row in this CTA's 128-row half == TMEM lane
  int q, half;  // lane quarter, column half
  int rank;
  float* xchg;
  float* xz;    // forward only: 128 floats for the column-half merge of the logit sums
  uint8_t* stage;  // this warp's 4 KB store-staging tile
};

__device__ __forceinline__ void epi_fwd(const GemmParams& p, uint32_t taddr, const PEpi& e, const PItem& it, int nv) {
  const int row = it.m0 + e.rank * HM + e.rit;
  const bool rv = row < nv;
  // the target only counts on the rank that owns it: a label of the NEXT shard can fall in
  // this shard's padded tail tile (local id in [V_local, 256-aligned)), where the logits are masked
  const int yl = rv ? (p.labels_c[row] - p.vocab_offset) : -1;
  const int y = ((unsigned)yl < (unsigned)p.V_local) ? yl : -1;
  const int cb = e.half * (PN / 2);
  float m = -INFINITY, d = 0.f;
  float zs = 0.f;  // sum of the logits (label smoothing's mean z)
  const bool want_zs = p.zs_part != nullptr;
#pragma unroll 1
  for (int j = 0; j < PN / 2 / 32; ++j) {
    float v[32];
    tmem_ld32(taddr + cb + j * 32, v);
    const int col0 = it.n0 + cb + j * 32;
    if (col0 >= p.V_local) break;  // warp-uniform
    if (want_zs) {
      float cs = 0.f;
#pragma unroll
      for (int i = 0; i < 32; ++i) cs += (col0 + i < p.V_local) ? v[i] : 0.f;
      zs += cs;
    }
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
    d = d * ex2((m - mn) * LOG2E) + (s0 + s1);
    m = mn;
    const unsigned off = (unsigned)(y - col0);
    if (off < 32u) {
      float zy = 0.f;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (off == (unsigned)i) zy = v[i];
      p.zy_c[row] = zy;
    }
  }
  float2* x = reinterpret_cast<float2*>(e.xchg);
  if (e.half == 1) {
    x[e.rit] = make_float2(m, d);
    if (want_zs) e.xz[e.rit] = zs;
  }
  named_bar_sync(3 + e.q, 64);
  if (e.half == 0) {
    const float2 o = x[e.rit];
    const float mn = fmaxf(m, o.x);
    const float dd = (d > 0.f ? d * ex2((m - mn) * LOG2E) : 0.f) + (o.y > 0.f ? o.y * ex2((o.x - mn) * LOG2E) : 0.f);
    if (rv) {
      p.part[(size_t)(it.n0 / PN) * p.Npad + row] = make_float2(mn, dd);
      if (want_zs) p.zs_part[(size_t)(it.n0 / PN) * p.Npad + row] = zs + e.xz[e.rit];
    }
  }
  named_bar_sync(3 + e.q, 64);
}

__device__ __forceinline__ void epi_g(const GemmParams& p, uint32_t taddr, const PEpi& e, const PItem& it, int nv,
                                      float scale, const CUtensorMap* tmGst, int gblk0) {
  // G = s (exp(S - lse) - 1[v = y]) with s folded into the exponent.  With
  // label smoothing eps and z-loss lambda:
  //   G = s [(1 + 2 lambda lse) exp(S - lse) - (1 - eps) 1[v = y] - eps / V]
  // Each warp converts 64 columns of its 32 rows at a time into a 4 KB SMEM tile
  // (16-byte chunks XOR-swizzled by row: conflict-free), then writes it out as
  // fully coalesced 512-byte runs of the column-blocked G ring.
  const int row = it.m0 + e.rank * HM + e.rit;
  const bool rv = row < nv;
  // the target only counts on the rank that owns it: a label of the NEXT shard can fall in
  // this shard's padded tail tile (local id in [V_local, 256-aligned)), where the logits are masked
  const int yl = rv ? (p.labels_c[row] - p.vocab_offset) : -1;
  const int y = ((unsigned)yl < (unsigned)p.V_local) ? yl : -1;
  const float lse = rv ? p.lse_c[row] : 0.f;
  if (p.dloss_c) scale = rv ? p.dloss_c[row] : 0.f;       // reduction "none": per-row upstream gradient
  const float sa = scale * (1.f + 2.f * p.z_loss * lse);  // scale of the softmax term
  const float off2 = rv ? (lse * LOG2E - __log2f(fabsf(sa))) : INFINITY;
  const float cu = rv ? -scale * p.ls_eps * p.inv_vtotal : 0.f;  // uniform term
  const float tgt = scale * (1.f - p.ls_eps);                     // one-hot term
  const int c0 = it.c * p.C;
  const int width = min(p.C, p.V_local - c0);
  const int cb = e.half * (PN / 2);
  const int lane = e.rit & 31;
  uint4* stg = reinterpret_cast<uint4*>(e.stage);  // [32 rows][8 x 16 B]
  const int row0 = it.m0 + e.rank * HM + (e.rit & ~31);  // first row of this warp
#pragma unroll
  for (int j2 = 0; j2 < PN / 2 / 64; ++j2) {
    const int lcol64 = (it.n0 - c0) + cb + j2 * 64;  // 64-column block within the chunk
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float v[32];
      tmem_ld32(taddr + cb + j2 * 64 + h * 32, v);
      const int lcol0 = lcol64 + h * 32;
      const int col0 = c0 + lcol0;
      float gg[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) gg[i] = ex2(fmaf(v[i], LOG2E, -off2));
      if (sa < 0.f) {
#pragma unroll
        for (int i = 0; i < 32; ++i) gg[i] = -gg[i];
      }
      if (cu != 0.f) {
#pragma unroll
        for (int i = 0; i < 32; ++i) gg[i] += cu;
      }
      const unsigned toff = (unsigned)(y - col0);
      if (toff < 32u) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (toff == (unsigned)i) gg[i] -= tgt;
      }
      if (lcol0 + 32 > width) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (lcol0 + i >= width) gg[i] = 0.f;
      }
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const int chunk = h * 4 + q4;
        stg[lane * 8 + (chunk ^ (lane & 7))] =
            make_uint4(pack_bf16(gg[8 * q4], gg[8 * q4 + 1]), pack_bf16(gg[8 * q4 + 2], gg[8 * q4 + 3]),
                       pack_bf16(gg[8 * q4 + 4], gg[8 * q4 + 5]), pack_bf16(gg[8 * q4 + 6], gg[8 * q4 + 7]));
      }
    }
    // one TMA store of the warp's 32 x 64 tile (the staging XOR pattern is the 128-byte
    // swizzle the map expects); the next block waits until the store has read the tile
    fence_proxy_async_shared();
    __syncwarp();
    if (lane == 0) {
      tma_store_3d(tmGst, stg, 0, row0, gblk0 + (lcol64 >> 6));
      bulk_commit();
      if (j2 + 1 < PN / 2 / 64) bulk_wait_read<0>();  // the last one is drained by the caller
    }
    __syncwarp();
  }
  // the caller releases the accumulator first (every TMEM read has retired), then drains
  // the stores (bulk_wait_all) before the item is published and before the staging tile is reused
}

__device__ __forceinline__ void epi_dw(const GemmParams& p, uint32_t taddr, const PEpi& e, const PItem& it,
                                       bool have_acc) {
  const int c0 = it.c * p.C;
  const int width = min(p.C, p.V_local - c0);
  const int vrow = it.m0 + e.rank * HM + e.rit;  // vocabulary row within the chunk
  const int hw = it.N / 2;
  const int cb = e.half * hw;
#pragma unroll 1
  for (int j = 0; j < hw / 32; ++j) {
    float v[32];
    if (have_acc) {
      tmem_ld32(taddr + cb + j * 32, v);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.f;
    }
    const int d0 = it.n0 + cb + j * 32;
    if (vrow < width && d0 < p.D) {
      const size_t off = (size_t)(c0 + vrow) * p.D + d0;
      if (p.dw_fp32) {
        // float32 gradient (CCE_FLAG_GRAD_FP32), optionally accumulated into the caller's
        // buffer (CCE_FLAG_ACCUMULATE): each element has exactly one writer, so a plain
        // load-add-store is race-free and deterministic
        float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.dW) + off);
        if (p.dw_accumulate) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 o = dst[i];
            v[4 * i] += o.x; v[4 * i + 1] += o.y; v[4 * i + 2] += o.z; v[4 * i + 3] += o.w;
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      } else {
        uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.dW) + off);
        if (p.dw_accumulate) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const uint4 o = dst[q4];
            const uint32_t w[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) {
              v[8 * q4 + 2 * k2] += __uint_as_float(w[k2] << 16);
              v[8 * q4 + 2 * k2 + 1] += __uint_as_float(w[k2] & 0xffff0000u);
            }
          }
        }
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          dst[q4] = make_uint4(pack_bf16(v[8 * q4], v[8 * q4 + 1]), pack_bf16(v[8 * q4 + 2], v[8 * q4 + 3]),
                               pack_bf16(v[8 * q4 + 4], v[8 * q4 + 5]), pack_bf16(v[8 * q4 + 6], v[8 * q4 + 7]));
      }
    }
  }
}

// Fused AdamW (Alg. Fused AdamW P:2003-2046): the finished dW
// tile is the gradient of these W rows; apply the optimizer step to W (and master / m
// / v) directly instead of writing dW.  Each thread owns one vocabulary row of the
// tile and walks its columns in 8-wide groups (32-byte vectors per state array).  The
// caller has already waited for this chunk's dH items, the only other readers of W_c.
__device__ __forceinline__ void epi_dw_adamw(const GemmParams& p, uint32_t taddr, const PEpi& e, const PItem& it,
                                             bool have_acc, float clip) {
  // TMEM hands each thread one ROW of the dW tile (lane = row), which would make every
  // state access a 32-row scatter (one L1/L2 request per lane: measured 70 us per item,
  // LSU-bound).  So each warp transposes its 32 x 32 fp32 block through its 4 KB
  // staging tile (XOR-swizzled, conflict-free both ways) and then walks the block row
  // by row with lane = column: every m / v / master access is one 128-byte line, every
  // W access one 64-byte run.  ROWS_IN_FLIGHT rows of state are loaded before use.
#ifndef CCE_ADAMW_RIF
#define CCE_ADAMW_RIF 16
#endif
  constexpr int RIF = CCE_ADAMW_RIF;
  const int c0 = it.c * p.C;
  const int width = min(p.C, p.V_local - c0);
  const int hw = it.N / 2;
  const int cb = e.half * hw;
  const int lane = e.rit & 31;
  const int row0 = it.m0 + e.rank * HM + e.q * 32;  // first vocabulary row (within the chunk) of this warp
  const int nrows = max(0, min(32, width - row0));
  float* stg = reinterpret_cast<float*>(e.stage);   // [32 rows][32 cols], column XOR row
#pragma unroll 1
  for (int j = 0; j < hw / 32; ++j) {
    const int d0 = it.n0 + cb + j * 32;
    float acc[32];
    if (have_acc) {
      tmem_ld32(taddr + cb + j * 32, acc);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] = 0.f;
    }
    if (d0 >= p.D || nrows == 0) continue;  // warp-uniform
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 32; ++c) stg[lane * 32 + (c ^ lane)] = acc[c];
    __syncwarp();
    const int d = d0 + lane;
    if (p.grad_in) {  // earlier micro-batches' gradient, added in place in the staging tile
#pragma unroll 4
      for (int rr = 0; rr < nrows; ++rr)
        stg[rr * 32 + (lane ^ rr)] += __ldcs(p.grad_in + (size_t)(c0 + row0 + rr) * p.D + d);
    }
#pragma unroll 1
    for (int r0 = 0; r0 < nrows; r0 += RIF) {
      float m[RIF], v[RIF], th[RIF];
#pragma unroll
      for (int r = 0; r < RIF; ++r) {
        if (r0 + r < nrows) {
          const size_t off = (size_t)(c0 + row0 + r0 + r) * p.D + d;
          m[r] = __ldcs(p.am + off);
          v[r] = __ldcs(p.av + off);
          th[r] = p.master ? __ldcs(p.master + off)
                           : __bfloat162float(p.Win[(size_t)(c0 + row0 + r0 + r) * p.ldw + d]);
        }
      }
#pragma unroll
      for (int r = 0; r < RIF; ++r) {
        if (r0 + r < nrows) {
          const int rr = r0 + r;
          const float gr = stg[rr * 32 + (lane ^ rr)] * clip;
          adamw_elem(gr, th[r], m[r], v[r], p.lr, p.beta1, p.beta2, p.eps, p.wd, p.bc1, p.bc2);
          const size_t off = (size_t)(c0 + row0 + rr) * p.D + d;
          __stcs(p.am + off, m[r]);
          __stcs(p.av + off, v[r]);
          if (p.master) __stcs(p.master + off, th[r]);
          p.Wout[(size_t)(c0 + row0 + rr) * p.ldw + d] = __float2bfloat16_rn(th[r]);
        }
      }
    }
  }
  __syncwarp();
}

// RED(tile): rows of this CTA's half of the tile, warp = 32 rows x its column half; lane =
// four consecutive columns (512-byte runs per row).  Sum over ranks in rank order (the
// same order on every rank: identical reduced dH everywhere), broadcast to every rank.
__device__ __forceinline__ void epi_reduce(const PairParams& P, const PEpi& e, const PItem& it, int nv, bool leader) {
  const GemmParams& g = P.g;
  if (leader) {
    const int* rf = reinterpret_cast<const int*>(P.peers.ws[P.prank] + P.ready_off);
    const unsigned long long t0 = p2p_now();
    for (int q = 0; q < P.world; ++q) {
      while (ld_acquire_sys(rf + q * P.tmax + it.tile_id) < P.epoch) {
        if (p2p_now() - t0 > P2P_TIMEOUT_NS) { atomicOr(P.err, 4); break; }
        __nanosleep(500);
      }
    }
  }
  named_bar_sync(2, PEPI_THREADS);
  const int hw = it.N / 2;
  const int lane = e.rit & 31;
  const int row0 = it.m0 + e.rank * HM + e.q * 32;
  const int col = it.n0 + e.half * hw + lane * 4;
  if (lane * 4 < hw && col < g.D) {
    for (int rr = 0; rr < 32; ++rr) {
      const int row = row0 + rr;
      if (row >= nv) break;
      const size_t idx = (size_t)row * g.D + col;
      float4 acc = *reinterpret_cast<const float4*>(P.peers.ws[0] + P.dH32_off + idx * 4);
      for (int qr = 1; qr < P.world; ++qr) {
        const float4 v = *reinterpret_cast<const float4*>(P.peers.ws[qr] + P.dH32_off + idx * 4);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      for (int qr = 0; qr < P.world; ++qr) *reinterpret_cast<float4*>(P.peers.ws[qr] + P.dHred_off + idx * 4) = acc;
    }
  }
  __threadfence_system();
  named_bar_sync(2, PEPI_THREADS);
  if (leader)
    for (int qr = 0; qr < P.world; ++qr)
      st_release_sys(reinterpret_cast<int*>(P.peers.ws[qr] + P.done_off) + 2 * it.tile_id + e.rank, P.epoch);
}

// dH epilogue through the TMA: each warp moves its 32 rows x 32 columns of the fp32
// accumulator into its 4 KB staging tile (128-byte swizzle: conflict-free) and issues one
// bulk tensor store (first chunk) or bulk reduce-add (later chunks) into dH32; the L2
// performs the adds, so the epilogue never waits on a load.  The caller orders chunk c's
// reduce after chunk c-1's (dh_flag), so every element is summed in chunk order: the
// result is bit-identical to a load-add-store in that order.
__device__ __forceinline__ void epi_dh_tma(const CUtensorMap* tmDH, uint32_t taddr, const PEpi& e,
                                           const PItem& it) {
  const int row0 = it.m0 + e.rank * HM + e.q * 32;
  const int hw = it.N / 2;
  const int cb = e.half * hw;
  const int lane = e.rit & 31;
  uint4* stg = reinterpret_cast<uint4*>(e.stage);  // [32 rows][8 x 16 B]
  const bool add = it.c > 0;
#pragma unroll 1
  for (int j = 0; j < hw / 32; ++j) {
    float v[32];
    tmem_ld32(taddr + cb + j * 32, v);
    if (j > 0) {
      if (lane == 0) bulk_wait_read<0>();  // previous box has left the staging tile
      __syncwarp();
    }
#pragma unroll
    for (int q4 = 0; q4 < 8; ++q4)
      stg[lane * 8 + (q4 ^ (lane & 7))] = make_uint4(__float_as_uint(v[4 * q4]), __float_as_uint(v[4 * q4 + 1]),
                                                     __float_as_uint(v[4 * q4 + 2]), __float_as_uint(v[4 * q4 + 3]));
    fence_proxy_async_shared();
    __syncwarp();
    if (lane == 0) {
      const int d0 = it.n0 + cb + j * 32;
      if (add) tma_reduce_add_2d(tmDH, stg, d0, row0);
      else tma_store_2d(tmDH, stg, d0, row0);
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait_all();
  __syncwarp();
}

// ------------------------------------------------------------------ MMA issue (leader warp)
// All 32 lanes wait on the full barrier; one elected lane issues the K=16 pair MMAs of the
// stage's k-blocks and commits the stage back to both CTAs' empty barriers.
// Stage s holds k-blocks KPS s .. KPS s + KPS - 1.  K-major operands: k-block kh
// 16 KB further; MN-major operands (boxes {64, 64 KPS k-rows, MN blocks}): k-block kh 8 KB
// further and the two 64-wide MN blocks KPS x 8 KB apart (leading byte offset).
template <bool A_MN, bool B_MN>
__device__ __forceinline__ void mma_item_k2(const PItem& it, uint64_t* full_bar, uint64_t* empty_bar, uint32_t a_base,
                                            uint32_t b_base, uint32_t tmem_d, uint32_t& stage, uint32_t& phase) {
  const uint32_t idesc = idesc_bf16_f32(PM, it.N, A_MN ? 1 : 0, B_MN ? 1 : 0);
  const int ns = (it.num_kb + KPS - 1) / KPS;
  for (int st = 0; st < ns; ++st) {
    mbar_wait(&full_bar[stage], phase);
    tc_fence_after();
    if (elect_one()) {
#pragma unroll
      for (int kh = 0; kh < KPS; ++kh) {
        const int kb = KPS * st + kh;
        if (kb < it.num_kb) {
          const uint64_t ad = sdesc_sw128(a_base + stage * KA_BYTES + kh * (A_MN ? 8192 : 16384), A_MN ? KPS * 8192 : 16, 1024);
          const uint64_t bd = sdesc_sw128(b_base + stage * KB_BYTES + kh * (B_MN ? 8192 : 16384), B_MN ? KPS * 8192 : 16, 1024);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_bf16_pair(tmem_d, ad + (uint64_t)(A_MN ? 128 * kk : 2 * kk),
                           bd + (uint64_t)(B_MN ? 128 * kk : 2 * kk), idesc, (kb | kk) ? 1u : 0u);
        }
      }
      umma_commit_pair(&empty_bar[stage]);
    }
    __syncwarp();
    if (++stage == KSTAGES) { stage = 0; phase ^= 1; }
  }
}

// ------------------------------------------------------------------ kernel
// The kernel body, shared by the launch kinds below: the tensor maps are generic pointers
// (kernel parameters for cce_pair_kernel, a global-memory array for cce_pair_group_kernel).
template <int ADAMW, int P2P>
__device__ __forceinline__ void pair_body(const CUtensorMap* tmHcK, const CUtensorMap* tmWK, const CUtensorMap* tmGMN,
                                          const CUtensorMap* tmHcMN, const CUtensorMap* tmGK, const CUtensorMap* tmWMN,
                                          const CUtensorMap* tmDH, const CUtensorMap* tmHcMN3,
                                          const CUtensorMap* tmWMN3, const CUtensorMap* tmGst, const PairParams& P) {
  const GemmParams& g = P.g;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + KSTAGES * KA_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + PSTAGES * PSTAGE_BYTES);
  uint64_t* empty_bar = full_bar + PSTAGES;
  uint64_t* tfull_bar = empty_bar + PSTAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* rfull_bar = tempty_bar + 2;
  uint64_t* rempty_l = rfull_bar + PRING;   // leader: local consumers (MMA + epilogue warps)
  uint64_t* rempty_p = rempty_l + PRING;    // leader: peer consumers (producer + epilogue warps)
  PItem* ring = reinterpret_cast<PItem*>(rempty_p + PRING);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + PRING);
  volatile int* prod_cnt = reinterpret_cast<volatile int*>(tmem_slot + 1);  // leader: items whose last stage the producer reached
  float* xchg = reinterpret_cast<float*>(smem + PSTAGES * PSTAGE_BYTES + 1024);
  uint8_t* stage_base = smem + PSTAGES * PSTAGE_BYTES + 2048;

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  int* head = P.sched;
  int* head2 = P.sched + 1;
  int* g_done = P.sched + 2;
  int* w_done = P.sched + 2 + P.n_chunks;
  int* dh_flag = P.sched + 2 + 2 * P.n_chunks;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(tmHcK); tma_prefetch_desc(tmWK);
    if (P.mode == 1) {
      tma_prefetch_desc(tmGMN); tma_prefetch_desc(tmHcMN); tma_prefetch_desc(tmGK); tma_prefetch_desc(tmWMN);
      tma_prefetch_desc(tmDH);
      tma_prefetch_desc(tmHcMN3); tma_prefetch_desc(tmWMN3); tma_prefetch_desc(tmGst);
    }
    for (int s = 0; s < KSTAGES; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull_bar[b], 1); mbar_init(&tempty_bar[b], 2 * PEPI_WARPS); }
    for (int r = 0; r < PRING; ++r) {
      mbar_init(&rfull_bar[r], 1);
      mbar_init(&rempty_l[r], 2 + PEPI_WARPS);  // leader producer + MMA + epilogue warps
      mbar_init(&rempty_p[r], 1 + PEPI_WARPS);  // peer producer + epilogue warps
    }
    *prod_cnt = 0;
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, TMEM_COLS);
  tc_fence_before();
  cluster_sync_all();
  __syncthreads();  // (also a CTA barrier: compute-sanitizer's racecheck does not model barrier.cluster)
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  PCounts k;
  k.nv = *g.n_valid;
  k.t256 = (k.nv + PM - 1) / PM;
  k.n_dt = (g.D + PN - 1) / PN;
  k.n_dh = k.t256 * k.n_dt;
  k.tv = (g.V_local + PN - 1) / PN;
  k.rg = l2_group_rows(k.t256, g.D);

  if (warp == 3) {
    if (lane == 0 && rank == 0) {
      // ===== scheduler (leader): dequeue items and publish them into both CTAs' rings,
      // up to PRING items ahead of the consumers (hides the atomic and DSMEM latency).
      uint32_t rs = 0, rph = 0;
      // split backward (NCCL): the last chunk's DW items are the queue's last p_n_dw items
      const int total = queue_total(P, k);
      const int q_split = P.part != 0 ? total - p_n_dw(k, p_chunk_width(g, P.n_chunks - 1)) : 0;
      const int jit_from = (P.part == 1 ? q_split : total) - P.jit_tail;
      int published = 0, q_last = -1;
      while (true) {
        if (q_last >= jit_from && published > 0)
          while (*prod_cnt < published) __nanosleep(32);  // just in time: the producer is on its last stage
        const int q = P.part == 2 ? q_split + atomicAdd(head2, 1) : atomicAdd(head, 1);
        q_last = q;
        PItem it = decode(P, k, q);
        if (P.part == 1 && q >= q_split) it = make_item(PT_END, 0, 0, 0, 0, 0, 0, q);
        if (P.trace) it.t_deq = gtimer();
        mbar_wait(&rempty_l[rs], rph ^ 1);
        mbar_wait(&rempty_p[rs], rph ^ 1);
        ring[rs] = it;
        const uint32_t remote = mapa_shared(smem_u32(&ring[rs]), 1);
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&it);
#pragma unroll
        for (int i = 0; i < (int)(sizeof(PItem) / 4); ++i) st_cluster_u32(remote + 4 * i, w[i]);
        mbar_arrive(&rfull_bar[rs]);
        mbar_arrive_cluster(mapa_shared(smem_u32(&rfull_bar[rs]), 1));
        if (++rs == PRING) { rs = 0; rph ^= 1; }
        if (it.type == PT_END) break;
        ++published;
      }
    }
  } else if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs): next item from the local ring, dependencies, loads
      uint32_t stage = 0, phase = 0, rs = 0, rph = 0;
      int n_started = 0;
      const uint32_t full_leader0 = mapa_shared(smem_u32(&full_bar[0]), 0);
      while (true) {
        if (rank == 0) mbar_wait(&rfull_bar[rs], rph);
        else mbar_wait_cluster(&rfull_bar[rs], rph);
        const PItem it = ring[rs];
        if (rank == 0) mbar_arrive(&rempty_l[rs]);
        else mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&rempty_p[rs]), 0));
        if (++rs == PRING) { rs = 0; rph ^= 1; }
        if (it.type == PT_END) break;
        if (P.mode == 1) {
          // dependencies: only on items earlier in the queue (deadlock-free)
          if (it.type == PT_G) {
            if (it.c >= P.slots) {
              const int wc = it.c - P.slots;
              wait_ge(&w_done[wc], 2 * (k.n_dh + p_n_dw(k, p_chunk_width(g, wc))));
            }
          } else {
            wait_ge(&g_done[it.c], 2 * p_n_g(k, p_chunk_width(g, it.c)));
            // DH(c, tile) after DH(c-1, tile) is enforced where the epilogue issues its reduce-add
          }
          fence_proxy_async_global();
        }
        if (P.trace && rank == 0 && it.q < P.trace_cap) P.trace[it.q].t_ready = gtimer();
        // operand loads for this CTA's halves
        const int hr = rank * HM;             // this CTA's first tile row
        const int hn = rank * (it.N / 2);     // this CTA's first B row / column
        const int b_bytes = (it.N / 2) * BK * 2;
        const int slot_blk0 = (it.c % P.slots) * (g.C / 64);  // first 64-column block of the slot
        const int c0 = it.c * g.C;
        unsigned long long tl0 = 0;
        // one 3-D box per operand per stage (KPS k-blocks); a ragged last stage: the k-blocks
        // past num_kb are zero-filled (OOB) or zero rows / columns and their MMAs are skipped
        const int ns = (it.num_kb + KPS - 1) / KPS;
        if (ns == 0 && rank == 0) *prod_cnt = ++n_started;
        for (int st = 0; st < ns; ++st) {
          if (st == ns - 1 && rank == 0) *prod_cnt = ++n_started;  // the scheduler may claim the next item
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (P.trace && st == 0) tl0 = gtimer();
          uint8_t* a = sA + stage * KA_BYTES;
          uint8_t* b = sB + stage * KB_BYTES;
          const uint32_t fb = full_leader0 + stage * 8;
          const int kb0 = KPS * st;
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * KPS * (PA_BYTES + b_bytes));
          if (it.type == PT_FWD || it.type == PT_G) {
            tma_load_3d_pair(tmHcK, fb, a, 0, it.m0 + hr, kb0);
            tma_load_3d_pair(tmWK, fb, b, 0, it.n0 + hn, kb0);
          } else if (it.type == PT_DW) {
            tma_load_3d_pair(tmGMN, fb, a, 0, kb0 * BK, slot_blk0 + (it.m0 + hr) / 64);
            if (it.N / 2 / 64 == 2) tma_load_3d_pair(tmHcMN3, fb, b, 0, kb0 * BK, (it.n0 + hn) / 64);
            else tma_load_2d_pair(tmHcMN, fb, b, it.n0 + hn, kb0 * BK);
          } else {  // PT_DH
            tma_load_3d_pair(tmGK, fb, a, 0, it.m0 + hr, slot_blk0 + kb0);
            if (it.N / 2 / 64 == 2) tma_load_3d_pair(tmWMN3, fb, b, 0, c0 + kb0 * BK, (it.n0 + hn) / 64);
            else tma_load_2d_pair(tmWMN, fb, b, it.n0 + hn, c0 + kb0 * BK);
          }
          if (++stage == KSTAGES) { stage = 0; phase ^= 1; }
        }
        if (P.trace && rank == 0 && it.q < P.trace_cap) {
          P.trace[it.q].t_load0 = tl0;
          P.trace[it.q].t_load1 = gtimer();
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ===== MMA issuer (leader): the whole warp runs the loop so every operand is
      // warp-uniform; one elected lane issues the MMAs and commits.
      uint32_t stage = 0, phase = 0, rs = 0, rph = 0;
      int acc_it = 0;
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      while (true) {
        mbar_wait(&rfull_bar[rs], rph);
        const PItem it = ring[rs];
        __syncwarp();
        if (lane == 0) mbar_arrive(&rempty_l[rs]);
        if (++rs == PRING) { rs = 0; rph ^= 1; }
        if (it.type == PT_END) break;
        if (it.num_kb == 0) continue;
        const uint32_t acc = acc_it & 1, acc_phase = (acc_it >> 1) & 1;
        ++acc_it;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * PN;
        const unsigned long long tm0 = P.trace ? gtimer() : 0ull;
        const unsigned long long cm0 = P.trace ? clock64() : 0ull;
        if (it.type == PT_DW)
          mma_item_k2<true, true>(it, full_bar, empty_bar, a_base, b_base, tmem_d, stage, phase);
        else if (it.type == PT_DH)
          mma_item_k2<false, true>(it, full_bar, empty_bar, a_base, b_base, tmem_d, stage, phase);
        else
          mma_item_k2<false, false>(it, full_bar, empty_bar, a_base, b_base, tmem_d, stage, phase);
        if (elect_one()) umma_commit_pair(&tfull_bar[acc]);
        __syncwarp();
        if (P.trace && lane == 0 && it.q < P.trace_cap) {
          P.trace[it.q].t_mma0 = tm0;
          P.trace[it.q].t_mma1 = gtimer();
          P.trace[it.q].r0 = clock64() - cm0;
        }
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue (both CTAs) =====
    PEpi e;
    e.q = warp & 3;
    e.half = (warp - 4) >> 2;
    e.rit = e.q * 32 + lane;
    e.rank = rank;
    e.xchg = xchg;
    e.xz = reinterpret_cast<float*>(stage_base);  // forward items never use the store staging
    e.stage = stage_base + (warp - 4) * 4096;
    const bool leader = (threadIdx.x == 128);
    const float scale = (P.mode == 1 && k.nv > 0 && g.reduction != 2)
                            ? (g.reduction == 1 ? *g.dloss : (*g.dloss) / (float)k.nv)
                            : 0.f;  // reduction "none": per-row dloss_c in epi_g
    const float clip = (ADAMW && g.clip_coef) ? *g.clip_coef : 1.f;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    uint32_t rs = 0, rph = 0;
    int acc_it = 0;
    while (true) {
      if (rank == 0) mbar_wait(&rfull_bar[rs], rph);
      else mbar_wait_cluster(&rfull_bar[rs], rph);
      const PItem it = ring[rs];
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(&rempty_l[rs]);
        else mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&rempty_p[rs]), 0));
      }
      if (++rs == PRING) { rs = 0; rph ^= 1; }
      if (it.type == PT_END) break;
      const bool have_acc = it.num_kb > 0;
      uint32_t acc = 0;
      if (have_acc) {
        acc = acc_it & 1;
        const uint32_t acc_phase = (acc_it >> 1) & 1;
        ++acc_it;
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
      }
      const uint32_t taddr = tmem_base + acc * PN + ((uint32_t)(e.q * 32) << 16);
      const unsigned long long t_epi0 = P.trace ? gtimer() : 0ull;
      if (it.type == PT_FWD) {
        if constexpr (!ADAMW) epi_fwd(g, taddr, e, it, k.nv);
      } else if (it.type == PT_G) {
        epi_g(g, taddr, e, it, k.nv, scale, tmGst, (it.c % P.slots) * (g.C / 64));
      } else if (it.type == PT_RED) {
        if constexpr (P2P) epi_reduce(P, e, it, k.nv, leader);
      } else if (it.type == PT_DW) {
        if constexpr (ADAMW) {
          // the chunk's dH tiles read W_c through the TMA: the update waits until every
          // DH(c, row tile, this hidden tile) item is complete (earlier in the queue)
          if (g.adamw_inplace && warp == 4) {
            const int dt = it.n0 / PN;
            for (int rt = lane; rt < k.t256; rt += 32) wait_ge(&dh_flag[rt * k.n_dt + dt], 2 * (it.c + 1));
          }
          named_bar_sync(2, PEPI_THREADS);
          epi_dw_adamw(g, taddr, e, it, have_acc, clip);
        } else {
          epi_dw(g, taddr, e, it, have_acc);
        }
      } else {
        // DH(c-1, tile) halves published; re-acquire so the .cg loads below see them
        if (leader) wait_ge(&dh_flag[it.tile_id], 2 * it.c);
        named_bar_sync(2, PEPI_THREADS);
        fence_proxy_async_global();  // the acquired flag orders the TMA reduce below
        epi_dh_tma(tmDH, taddr, e, it);
      }
      if (have_acc) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (rank == 0) mbar_arrive(&tempty_bar[acc]);
          else mbar_arrive_cluster_relaxed(tempty_leader0 + acc * 8);  // TMEM reads retired (wait::ld)
        }
      }
      if (it.type == PT_G) {  // epi_g's last dlogits store: in global memory before publishing
        if (lane == 0) bulk_wait_all();
        __syncwarp();
      }
      if (P.mode == 0 && P.trace && leader && rank == 0 && it.q < P.trace_cap) {
        P.trace[it.q].q_type_c = ((unsigned long long)it.q << 32) | ((unsigned long long)it.type << 16) | (unsigned)it.c;
        P.trace[it.q].smid = smid();
        P.trace[it.q].t_deq = it.t_deq;
        P.trace[it.q].t_epi0 = t_epi0;
        P.trace[it.q].t_epi1 = gtimer();
        P.trace[it.q].pad = it.num_kb;
      }
      if (P.mode == 1) {
        // publish this CTA's half of the item: every thread's stores are ordered before
        // the named barrier; the publishing thread's gpu-scope fence is cumulative
        fence_proxy_async_global();
        named_bar_sync(1, PEPI_THREADS);
        if (leader) {
          __threadfence();
          if (P.trace && rank == 0 && it.q < P.trace_cap) {
            TraceRec& r = P.trace[it.q];
            r.q_type_c = ((unsigned long long)it.q << 32) | ((unsigned long long)it.type << 16) | (unsigned)it.c;
            r.smid = smid();
            r.t_deq = it.t_deq;
            r.t_epi0 = t_epi0;
            r.t_epi1 = gtimer();
            r.tile = ((unsigned long long)it.m0 << 32) | (unsigned)it.n0;
            r.pad = it.num_kb;
          }
          if (it.type == PT_G) atomicAdd(&g_done[it.c], 1);
          else if (it.type != PT_RED) {
            if (it.type == PT_DH) {
              const int old = atomicAdd(&dh_flag[it.tile_id], 1);
              if constexpr (P2P) {
                // the second half of the last chunk's tile: its partial dH is final here ->
                // ready[prank][tile] in every rank (after a system-scope fence)
                if (it.c == P.n_chunks - 1 && old == 2 * P.n_chunks - 1) {
                  __threadfence_system();
                  for (int qr = 0; qr < P.world; ++qr)
                    st_release_sys(reinterpret_cast<int*>(P.peers.ws[qr] + P.ready_off) + P.prank * P.tmax + it.tile_id,
                                   P.epoch);
                }
              }
            }
            atomicAdd(&w_done[it.c], 1);
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


// ADAMW = 1: the backward queue with AdamW fused into the dW epilogue (cce_backward_adamw);
// a separate instantiation so its epilogue's register demand leaves the default kernel alone.
template <int ADAMW, int P2P>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PTHREADS, 1)
    cce_pair_kernel(const __grid_constant__ CUtensorMap tmHcK, const __grid_constant__ CUtensorMap tmWK,
                    const __grid_constant__ CUtensorMap tmGMN, const __grid_constant__ CUtensorMap tmHcMN,
                    const __grid_constant__ CUtensorMap tmGK, const __grid_constant__ CUtensorMap tmWMN,
                    const __grid_constant__ CUtensorMap tmDH, const __grid_constant__ CUtensorMap tmHcMN3,
                    const __grid_constant__ CUtensorMap tmWMN3, const __grid_constant__ CUtensorMap tmGst,
                    const PairParams P) {
  pair_body<ADAMW, P2P>(&tmHcK, &tmWK, &tmGMN, &tmHcMN, &tmGK, &tmWMN, &tmDH, &tmHcMN3, &tmWMN3, &tmGst, P);
}

// One rank's launch of the backward queue, as the group kernel below reads it.
struct alignas(64) PairLaunch {
  CUtensorMap m[10];  // HcK, WK, GMN, HcMN, GK, WMN, DH, HcMN3, WMN3, Gst
  PairParams P;
};

// One-GPU emulation of `world` ranks exchanging over peer memory (cce_p2p_attach_group):
// ONE launch holds every rank's backward queue, CTA pairs [r ppr, (r + 1) ppr) serving rank
// r, so the ranks' kernels are co-resident by construction -- ranks whose kernels wait on one
// another are never separate launches time-sliced on one GPU.  Same body as the P2P kernel.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PTHREADS, 1)
    cce_pair_group_kernel(const PairLaunch* __restrict__ L, int pairs_per_rank) {
  const PairLaunch& R = L[(blockIdx.x >> 1) / pairs_per_rank];
  pair_body<0, 1>(&R.m[0], &R.m[1], &R.m[2], &R.m[3], &R.m[4], &R.m[5], &R.m[6], &R.m[7], &R.m[8], &R.m[9], R.P);
}

}  // namespace pairk
}  // namespace cce
