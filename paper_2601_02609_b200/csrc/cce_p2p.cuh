// cce_p2p.cuh -- the vocabulary-sharded exchange done by our own kernels over peer memory
// (CCE_FLAG_P2P_COMBINE): every rank's workspace is mapped into
// every other rank (CUDA IPC), and
//   a9  the merged per-row stats are PUSHED into each rank's all-ranks array by the
//       kernel that produced them (k_p2p_push_stats, stores over NVLink), then a release
//       flag per (kind, source rank) is raised in every peer and waited for;
//   a10 each rank sums ITS row slice of the partial dH over all ranks in rank order (loads
//       over NVLink, deterministic) and stores the sum into every rank's reduced-dH array
//       (a reduce-scatter and an all-gather fused into one kernel).
// Flags are epoch counters (one step = one epoch) in each rank's workspace; waits are
// bounded (a missing peer sets the error word instead of hanging the GPU).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace cce {

constexpr int P2P_MAX = 8;                // ranks
constexpr int P2P_STATS = 0, P2P_READY = 1, P2P_DONE = 2;  // flag kinds
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

// This rank's stats rows -> slot `rank` of every rank's all-ranks array (rank-major [world][Npad]).
__global__ void k_p2p_push_stats(const float4* __restrict__ stats, int Npad, const int* __restrict__ n_valid,
                                 PeerPtrs peers, unsigned long long stats_all_off, int rank, int world) {
  const int nv = *n_valid;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
    const float4 v = stats[i];
    for (int r = 0; r < world; ++r)
      reinterpret_cast<float4*>(peers.ws[r] + stats_all_off)[(size_t)rank * Npad + i] = v;
  }
  __threadfence_system();
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

// Wait until every rank raised (kind) for this epoch; bounded: on timeout set err bit 4.
__global__ void k_p2p_wait(const int* __restrict__ flags, int kind, int world, int epoch, int* err) {
  const int r = threadIdx.x;
  if (r >= world) return;
  const int* f = flags + kind * P2P_MAX + r;
  const unsigned long long t0 = p2p_now();
  while (ld_acquire_sys(f) < epoch) {
    if (p2p_now() - t0 > P2P_TIMEOUT_NS) {
      atomicOr(err, 4);
      return;
    }
    __nanosleep(1000);
  }
}

// a10: rows [rank S, (rank + 1) S) of the compact dH (S = ceil(n_valid / world)): the sum of
// all ranks' partials in rank order, stored into every rank's reduced array.
__global__ void k_p2p_reduce_dH(PeerPtrs peers, unsigned long long dH32_off, unsigned long long dHred_off, int D,
                                const int* __restrict__ n_valid, int rank, int world) {
  const int nv = *n_valid;
  const int S = (nv + world - 1) / world;
  const int r0 = rank * S, r1 = min(nv, r0 + S);
  if (r1 <= r0) return;
  const int vec = D / 4;
  const long long total = (long long)(r1 - r0) * vec;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long e = (long long)r0 * vec + i;  // float4 index into [Npad][D]
    float4 acc = reinterpret_cast<const float4*>(peers.ws[0] + dH32_off)[e];
    for (int q = 1; q < world; ++q) {
      const float4 v = reinterpret_cast<const float4*>(peers.ws[q] + dH32_off)[e];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    for (int q = 0; q < world; ++q) reinterpret_cast<float4*>(peers.ws[q] + dHred_off)[e] = acc;
  }
  __threadfence_system();
}

}  // namespace cce
