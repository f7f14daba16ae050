// cce_p2p.cuh -- the vocabulary-sharded exchange done by our own kernels over peer memory
// (CCE_FLAG_P2P_COMBINE): every rank's workspace is mapped into
// every other rank (CUDA IPC), and
//   a9  the merged per-row stats are PUSHED into each rank's all-ranks array by the
//       kernel that produced them (k_merge_tiles, stores over NVLink), whose last block then
//       raises a release flag per source rank in every peer; k_finalize_loss waits for them;
//   a10 inside the backward kernel (cce_pair.cuh, RED items): as soon as every rank's
//       last-chunk dH tile is final, the tile's owner (tile % world) sums it over the ranks
//       in rank order (loads over NVLink, deterministic) and stores the sum into every
//       rank's reduced-dH array (a reduce-scatter and an all-gather fused, overlapping the
//       remaining MMA items tile by tile); the dH scatter (k_scatter_dH) waits for it.
// Flags are epoch counters (one step = one epoch) in each rank's workspace; waits are
// bounded (a missing peer sets the error word instead of hanging the GPU).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace cce {

constexpr int P2P_MAX = 8;                // ranks
constexpr int P2P_STATS = 0;  // flag kind: per-row stats pushed (the other kinds are per tile)
constexpr unsigned long long P2P_TIMEOUT_NS = 5000000000ull;

struct PeerPtrs {
  char* ws[P2P_MAX];  // workspace base of every rank (own rank: the local workspace)
};

__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long p2p_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Raise flag (kind, rank) = epoch in every rank (one thread; the kernel before it on the
// stream fenced its peer stores at system scope).
__global__ void k_p2p_signal(PeerPtrs peers, unsigned long long flags_off, int kind, int rank, int world, int epoch) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    __threadfence_system();
    for (int r = 0; r < world; ++r)
      st_release_sys(reinterpret_cast<int*>(peers.ws[r] + flags_off) + kind * P2P_MAX + rank, epoch);
  }
}

// Wait until every tile's RED item raised done[tile][cta] for this epoch (tiles from the
// device-side n_valid); bounded: on timeout set err bit 4 (used before the RMSNorm backward;
// the dH scatter waits itself).
__global__ void k_p2p_wait_tiles(const int* __restrict__ done, const int* __restrict__ n_valid, int D, int epoch,
                                 int* err) {
  const int t256 = (*n_valid + 255) / 256, n_dt = (D + 255) / 256;
  const int n = 2 * t256 * n_dt;
  const unsigned long long t0 = p2p_now();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    while (ld_acquire_sys(done + i) < epoch) {
      if (p2p_now() - t0 > P2P_TIMEOUT_NS) {
        atomicOr(err, 4);
        return;
      }
      __nanosleep(1000);
    }
  }
}

}  // namespace cce
