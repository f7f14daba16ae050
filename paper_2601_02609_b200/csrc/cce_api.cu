// cce_api.cu -- host side of the C ABI declared in include/cce.h: argument
// validation, workspace layout, TMA tensor maps, kernel launches and the
// vocabulary-sharded NCCL combine.  No host synchronisation on the hot path.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/cce.h"
#include "cce_aux.cuh"
#include "cce_common.cuh"
#include "cce_designb.cuh"
#include "cce_p2p.cuh"
#include "cce_pair.cuh"

using namespace cce;

#ifndef CCE_JIT_TAIL
// the last CCE_JIT_TAIL queue items are claimed just in time (pairk::PairParams::jit_tail):
// measured (interleaved A/B, profiles/r02b_ab_jit_tail.txt) 6% faster on a 1/8 vocabulary shard
// (0.556 -> 0.524 ms per step), neutral on the whole vocabulary; claiming EVERY item just in
// time starves the pipeline (+20%)
#define CCE_JIT_TAIL 400
#endif
#ifndef CCE_LOOKAHEAD
#define CCE_LOOKAHEAD 1  // backward queue: G of chunk c + LOOKAHEAD is queued before W of chunk c
#endif
#ifndef CCE_CHUNK
#define CCE_CHUNK 8192  // vocabulary rows per backward chunk (Gbuf = Npad x CCE_CHUNK bf16)
#endif

// ------------------------------------------------------------------ handle
struct cce_handle {
  cce_config cfg;
  int device = 0;
  int num_sms = 148;
  int64_t chunk = CCE_CHUNK;  // backward vocabulary chunk (compile-time; multiple of 256)
  int slots = GBUF_SLOTS;     // dlogits ring slots
  // state saved by the forward for the backward (like autograd-saved tensors)
  bool have_fwd = false;
  const void* W = nullptr;
  int64_t N = 0, D = 0, V_local = 0, ldw = 0;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  // RMSNorm prologue (cce_forward_rmsnorm): the un-normalised rows and the scale, saved
  // for cce_backward_rmsnorm
  bool norm = false;
  // split-phase combine (CCE_FLAG_EXTERNAL_COMBINE): outputs of the pending finish calls
  bool fwd_pending = false, bwd_pending = false;
  float* p_loss = nullptr;
  float* p_lse = nullptr;
  int32_t* p_nv = nullptr;
  void* p_dH = nullptr;
  // cce_step_host_async: per staging buffer, the event after which its inputs are consumed
  struct Stage { const void* buf; cudaEvent_t consumed; };
  Stage stages[4] = {};
  cudaEvent_t ev_copied = nullptr;
  // CCE_FLAG_P2P_COMBINE: peers' workspaces (CUDA IPC), the attached local workspace, step epoch
  PeerPtrs peers = {};
  void* opened[P2P_MAX] = {};
  void* p2p_ws = nullptr;
  bool p2p_attached = false;
  int epoch = 0;
  int64_t p2p_N = 0, p2p_D = 0;  // the problem size the P2P flag arrays were laid out for
  // cce_p2p_attach_group (one-GPU emulation of `group_n` ranks in one process): the group's
  // handles in rank order; each rank's forward tail and backward launch + tail are deferred
  // until the group's last rank calls, which issues them for every rank (one backward launch)
  cce_handle* group[P2P_MAX] = {};
  int group_n = 0;
  bool group_broken = false;  // another member was destroyed: this handle refuses further steps
  bool grp_fwd_pending = false, grp_bwd_pending = false;
  cudaStream_t grp_stream = nullptr;
  pairk::PairLaunch grp_launch;             // this rank's prepared backward launch (host copy)
  bool grp_has_launch = false;
  void* grp_dH = nullptr;
  void* grp_dgamma = nullptr;
  bool grp_norm = false;
  pairk::PairLaunch* grp_launch_dev = nullptr;  // last rank: every rank's launch, device copy
  const void* nX = nullptr;
  int64_t ldx = 0;
  const void* gamma = nullptr;
  int64_t launches = 0;
  // NCCL backward: side stream for the dH all-reduce overlapping the last chunk's dW items
  cudaStream_t side = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  bool dH_reduced = false;  // this backward's all-reduce was already issued (split launch)
  void* trace = nullptr;  // cce_debug_trace: per-item records of the backward
  size_t trace_bytes = 0;
  void* fwd_trace = nullptr;  // ... and of the forward (second half of the buffer)
  size_t fwd_trace_bytes = 0;
  // profiling (cce_profile_enable): event pairs per launch, tagged with a class
  bool prof = false;
  struct Rec { cudaEvent_t a, b; int cls; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t ev() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
};

// Brackets one kernel launch with events when profiling is on.
struct ProfScope {
  cce_handle* h;
  cudaStream_t s;
  int cls;
  cudaEvent_t a = nullptr;
  ProfScope(cce_handle* h_, cudaStream_t s_, int cls_) : h(h_), s(s_), cls(cls_) {
    if (h->prof) {
      a = h->ev();
      cudaEventRecord(a, s);
    }
    h->launches++;
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = h->ev();
      cudaEventRecord(b, s);
      h->recs.push_back({a, b, cls});
    }
  }
};

// ------------------------------------------------------------------ driver entry points
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

// 2-D bf16 tensor map over a row-major matrix [rows][cols] with row stride
// `ld` elements, box {64 (cols), box_rows}, 128-byte swizzle, zero OOB fill.
static bool make_map(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t ld,
                     uint32_t box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 2-D fp32 tensor map over a row-major matrix [rows][cols] (row stride `ld` elements),
// box {box_cols, box_rows}, 128-byte swizzle (box_cols * 4 == 128): the dH32 target of
// the TMA store / reduce-add epilogue.
static bool make_map_f32(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t ld,
                         uint32_t box_cols, uint32_t box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3-D bf16 view of a row-major matrix [rows][cols] (row stride `ld` elements) as 64-column
// blocks: dims {64, rows, cols / 64}, strides {ld * 2 bytes, 128 bytes}; box {64, box_rows,
// box_blocks}.  One TMA instruction then fetches box_blocks MN-major 64-column boxes that
// land in shared memory exactly as box_blocks separate 2-D boxes would (8 KB apart).
static bool make_map_colblocks(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t ld,
                               uint32_t box_rows, uint32_t box_blocks) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {64, rows, cols / 64};
  cuuint64_t strides[2] = {ld * 2, 128};
  cuuint32_t box[3] = {64, box_rows, box_blocks};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static bool make_map_blocked2(CUtensorMap* m, const void* base, uint64_t rows, uint64_t blocks, uint32_t box_rows,
                              uint32_t box_blocks) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {64, rows, blocks};
  cuuint64_t strides[2] = {128, rows * 128};
  cuuint32_t box[3] = {64, box_rows, box_blocks};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// ------------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclId {
  char internal[128];
};
typedef int (*nccl_get_id_t)(NcclId*);
typedef int (*nccl_init_t)(void**, int, NcclId, int);
typedef int (*nccl_destroy_t)(void*);
typedef int (*nccl_allgather_t)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef int (*nccl_allreduce_t)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_reducescatter_t)(const void*, void*, size_t, int, int, void*, cudaStream_t);
struct Nccl {
  bool ok = false;
  nccl_get_id_t get_id;
  nccl_init_t init;
  nccl_destroy_t destroy;
  nccl_allgather_t allgather;
  nccl_allreduce_t allreduce;
  nccl_reducescatter_t reducescatter;
};
const int kNcclFloat32 = 7, kNcclSum = 0;

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the one torch already loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.get_id = (nccl_get_id_t)dlsym(h, "ncclGetUniqueId");
    n.init = (nccl_init_t)dlsym(h, "ncclCommInitRank");
    n.destroy = (nccl_destroy_t)dlsym(h, "ncclCommDestroy");
    n.allgather = (nccl_allgather_t)dlsym(h, "ncclAllGather");
    n.allreduce = (nccl_allreduce_t)dlsym(h, "ncclAllReduce");
    n.reducescatter = (nccl_reducescatter_t)dlsym(h, "ncclReduceScatter");
    n.ok = n.get_id && n.init && n.destroy && n.allgather && n.allreduce && n.reducescatter;
  });
  return n;
}
}  // namespace

// ------------------------------------------------------------------ workspace layout
namespace {
constexpr int RMS_GP = 256;  // blocks of the RMSNorm backward (dgamma partials)

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Layout {
  int64_t Npad, Tv, C;
  int64_t n_chunks, sched_ints;
  size_t scal, pos, idx, labels_c, Hc, part, zs_part, zy_c, stats, stats_all, lse_c, loss_rows, dloss_c, gbuf,
      dH32, sched, rstd_c, gpart, dHo, p2p_flags, p2p_ready, p2p_done, dHred, b_opart, b_spart, b_U, total;
  int64_t b_maxseg;  // CCE_FLAG_DESIGN_B: forward partial slots (units k tiles + t)
  int64_t p2p_tmax;  // dH tiles the P2P flag arrays hold: ceil(D/256) x Npad/256
  int64_t seq_slice;  // CCE_FLAG_DH_SEQ_SHARD: rows per rank of the original-order dH (0 otherwise)
};

constexpr int DSB_GRID = 148;  // design-B kernel: one CTA per SM (partial slots are laid out for this grid)

Layout layout(int64_t N, int64_t D, int64_t V_local, int world, int64_t chunk, int slots, uint32_t flags = 0) {
  const bool seq = (flags & CCE_FLAG_DH_SEQ_SHARD) != 0;
  const bool p2p = (flags & CCE_FLAG_P2P_COMBINE) != 0;
  Layout L;
  L.Npad = align_up((size_t)(N > 0 ? N : 1), 256);  // pair tiles are 256 rows
  L.Tv = (V_local + BN - 1) / BN;
  if (L.Tv < 1) L.Tv = 1;
  int64_t C = chunk;
  const int64_t vr = (int64_t)align_up((size_t)(V_local > 0 ? V_local : 1), BN);
  if (vr < C) C = vr;
  L.C = C;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  L.p2p_flags = L.p2p_ready = L.p2p_done = L.dHred = 0;
  L.p2p_tmax = ((D + 255) / 256) * (L.Npad / 256);
  if (p2p) {
    // the regions peers read or write come first, at offsets that depend only on (N, D, world)
    // (shard sizes V_local differ between ranks): flags, all-ranks stats, reduced dH, partial dH
    L.p2p_flags = take(3 * P2P_MAX * 4);
    L.p2p_ready = take((size_t)P2P_MAX * L.p2p_tmax * 4);  // ready[rank][tile]
    L.p2p_done = take((size_t)2 * L.p2p_tmax * 4);         // done[tile][cta of the pair]
    // double-buffered by step parity: rank r's next forward pushes into the other half
    // while a slower peer may still be reading this step's (forward-only loops too)
    L.stats_all = take((size_t)2 * world * L.Npad * 16);
    L.dHred = take((size_t)L.Npad * D * 4);
    L.dH32 = take((size_t)L.Npad * D * 4);
  }
  L.scal = take(64);
  L.pos = take((size_t)(N > 0 ? N : 1) * 4);
  L.idx = take((size_t)L.Npad * 4);
  L.labels_c = take((size_t)L.Npad * 4);
  L.Hc = take((size_t)L.Npad * D * 2);
  L.part = take((size_t)L.Tv * L.Npad * 8);
  L.zs_part = take((size_t)L.Tv * L.Npad * 4);  // label smoothing only: per-tile logit sums
  L.zy_c = take((size_t)L.Npad * 4);
  L.stats = take((size_t)L.Npad * 16);
  if (!p2p) L.stats_all = take((size_t)world * L.Npad * 16);
  L.lse_c = take((size_t)L.Npad * 4);
  L.loss_rows = take((size_t)L.Npad * 4);
  L.dloss_c = take((size_t)L.Npad * 4);  // reduction "none": upstream gradients of the valid rows
  L.gbuf = take((size_t)slots * L.Npad * L.C * 2);  // ring of N x chunk dlogits (never N x V)
  if (!p2p) L.dH32 = take((size_t)L.Npad * D * 4);
  L.n_chunks = (V_local + L.C - 1) / L.C;
  // backward work queue: head | g_done[n] | w_done[n] | dh_flag[tiles_d * ceil(Npad/BN)]
  L.sched_ints = 2 + 2 * L.n_chunks + ((D + 127) / 128) * ((L.Npad + BN - 1) / BN);
  L.sched = take((size_t)L.sched_ints * 4);
  L.rstd_c = take((size_t)L.Npad * 4);            // RMSNorm prologue: rstd per compact row
  L.gpart = take((size_t)RMS_GP * D * 4);          // RMSNorm backward: per-block dgamma partials
  // CCE_FLAG_DH_SEQ_SHARD: this rank's partial dH in original row order, world x slice rows
  L.seq_slice = seq ? (N + world - 1) / world : 0;
  L.dHo = take(seq ? (size_t)world * L.seq_slice * D * 4 : 0);
  // CCE_FLAG_DESIGN_B: per-CTA O' / (m, d_nt, z_y) partials of the forward, U [Npad][D] fp32
  const bool db = (flags & CCE_FLAG_DESIGN_B) != 0;
  const int64_t btiles = (L.Npad + dsb::NX - 1) / dsb::NX;
  L.b_maxseg = db ? dsb::fwd_slots_max(btiles, DSB_GRID) : 0;  // forward partial slots
  L.b_opart = take(db ? (size_t)L.b_maxseg * dsb::NX * D * 4 : 0);
  L.b_spart = take(db ? (size_t)L.b_maxseg * dsb::NX * 16 : 0);
  L.b_U = take(db ? (size_t)L.Npad * D * 4 : 0);
  L.total = o;
  return L;
}

template <typename T>
T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int grid_for(long long work, int threads, int cap) {
  long long g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

cce_status launch_pair(cce_handle* h, const CUtensorMap& m0, const CUtensorMap& m1, const CUtensorMap& m2,
                       const CUtensorMap& m3, const CUtensorMap& m4, const CUtensorMap& m5, const CUtensorMap& m6,
                       const pairk::PairParams& pp, cudaStream_t s, int prof_class, const CUtensorMap* m7 = nullptr,
                       const CUtensorMap* m8 = nullptr, const CUtensorMap* m9 = nullptr, int pairs = 0) {
  const CUtensorMap& x7 = m7 ? *m7 : m3;
  const CUtensorMap& x8 = m8 ? *m8 : m5;
  const CUtensorMap& x9 = m9 ? *m9 : m4;
  // the >48 KB dynamic shared memory opt-in is per device: set on every launch (cheap,
  // thread-safe, correct when one process drives several GPUs)
  const cudaFuncAttribute a = cudaFuncAttributeMaxDynamicSharedMemorySize;
  if (cudaFuncSetAttribute(pairk::cce_pair_kernel<0, 0>, a, pairk::PSMEM) != cudaSuccess ||
      cudaFuncSetAttribute(pairk::cce_pair_kernel<1, 0>, a, pairk::PSMEM) != cudaSuccess ||
      cudaFuncSetAttribute(pairk::cce_pair_kernel<0, 1>, a, pairk::PSMEM) != cudaSuccess)
    return CCE_ERR_CUDA;
  const int grid = pairs > 0 ? 2 * pairs : (h->num_sms / 2) * 2;  // whole CTA pairs
  {
    ProfScope ps(h, s, prof_class);
    if (pp.g.adamw)
      pairk::cce_pair_kernel<1, 0><<<grid, pairk::PTHREADS, pairk::PSMEM, s>>>(m0, m1, m2, m3, m4, m5, m6, x7, x8, x9, pp);
    else if (pp.world > 1)
      pairk::cce_pair_kernel<0, 1><<<grid, pairk::PTHREADS, pairk::PSMEM, s>>>(m0, m1, m2, m3, m4, m5, m6, x7, x8, x9, pp);
    else
      pairk::cce_pair_kernel<0, 0><<<grid, pairk::PTHREADS, pairk::PSMEM, s>>>(m0, m1, m2, m3, m4, m5, m6, x7, x8, x9, pp);
  }
  return cudaGetLastError() == cudaSuccess ? CCE_OK : CCE_ERR_CUDA;
}
}  // namespace

namespace {
cce_status launch_designb(cce_handle* h, const CUtensorMap& tX, const CUtensorMap& tY1, const CUtensorMap& tY2,
                          const dsb::Params& P, cudaStream_t s, int prof_class) {
  if (cudaFuncSetAttribute(dsb::cce_designb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dsb::SMEM) !=
      cudaSuccess)
    return CCE_ERR_CUDA;
  {
    ProfScope ps(h, s, prof_class);
    dsb::cce_designb_kernel<<<DSB_GRID, dsb::THREADS, dsb::SMEM, s>>>(tX, tY1, tY2, P);
  }
  return cudaGetLastError() == cudaSuccess ? CCE_OK : CCE_ERR_CUDA;
}
}  // namespace

// ------------------------------------------------------------------ API
extern "C" {

void cce_config_default(cce_config* cfg) {
  if (!cfg) return;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->ignore_index = -100;
  cfg->vocab_total = 0;
  cfg->vocab_offset = 0;
  cfg->rank = 0;
  cfg->world = 1;
  cfg->nccl_comm = nullptr;
  cfg->flags = CCE_FLAG_NONE;
}

const char* cce_status_string(cce_status s) {
  switch (s) {
    case CCE_OK: return "CCE_OK";
    case CCE_ERR_INVALID_VALUE: return "CCE_ERR_INVALID_VALUE";
    case CCE_ERR_UNSUPPORTED: return "CCE_ERR_UNSUPPORTED";
    case CCE_ERR_LABEL_RANGE: return "CCE_ERR_LABEL_RANGE";
    case CCE_ERR_NO_FORWARD: return "CCE_ERR_NO_FORWARD";
    case CCE_ERR_WORKSPACE: return "CCE_ERR_WORKSPACE";
    case CCE_ERR_CUDA: return "CCE_ERR_CUDA";
    case CCE_ERR_NCCL: return "CCE_ERR_NCCL";
  }
  return "CCE_ERR_UNKNOWN";
}

const char* cce_build_info(void) {
  return "cce sm_100a tcgen05.mma.cta_group::2 / TMA pair engine, tiles 256x256, BK=64 x 2 per stage, 3 stages, chunk=8192";
}

cce_status cce_create(cce_handle** out, const cce_config* cfg) {
  if (!out || !cfg) return CCE_ERR_INVALID_VALUE;
  *out = nullptr;
  if (cfg->vocab_total <= 0 || cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world ||
      cfg->vocab_offset < 0 || cfg->vocab_offset > cfg->vocab_total)
    return CCE_ERR_INVALID_VALUE;
  // world > 1 needs a communicator; world == 1 may carry one (a 1-rank comm runs the
  // same NCCL collectives -- identities -- which lets one GPU exercise that path)
  if (cfg->world > 1 && cfg->nccl_comm == nullptr && !(cfg->flags & (CCE_FLAG_EXTERNAL_COMBINE | CCE_FLAG_P2P_COMBINE)))
    return CCE_ERR_INVALID_VALUE;
  if ((cfg->flags & CCE_FLAG_P2P_COMBINE) &&
      (cfg->nccl_comm || cfg->world > P2P_MAX ||
       (cfg->flags & (CCE_FLAG_EXTERNAL_COMBINE | CCE_FLAG_DH_SEQ_SHARD))))
    return CCE_ERR_UNSUPPORTED;
  const uint32_t known = CCE_FLAG_GRAD_FP32 | CCE_FLAG_ACCUMULATE | CCE_FLAG_EXTERNAL_COMBINE | CCE_FLAG_DH_SEQ_SHARD |
                         CCE_FLAG_P2P_COMBINE | CCE_FLAG_DESIGN_B;
  if (cfg->flags & ~known) return CCE_ERR_INVALID_VALUE;
  // design B: one unsharded GPU, the plain cross-entropy (its U is the dH of exactly that loss)
  if ((cfg->flags & CCE_FLAG_DESIGN_B) &&
      (cfg->world != 1 || cfg->nccl_comm || cfg->label_smoothing != 0.f || cfg->z_loss != 0.f ||
       (cfg->flags & (CCE_FLAG_EXTERNAL_COMBINE | CCE_FLAG_DH_SEQ_SHARD | CCE_FLAG_P2P_COMBINE))))
    return CCE_ERR_UNSUPPORTED;
  if (cfg->vocab_total > 0x7fffffffLL) return CCE_ERR_UNSUPPORTED;
  if (!(cfg->label_smoothing >= 0.f && cfg->label_smoothing < 1.f) || !(cfg->z_loss >= 0.f && cfg->z_loss < 1e30f))
    return CCE_ERR_INVALID_VALUE;
  if (cfg->reduction < CCE_REDUCTION_MEAN || cfg->reduction > CCE_REDUCTION_NONE) return CCE_ERR_INVALID_VALUE;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return CCE_ERR_UNSUPPORTED;
  int major = 0, sms = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return CCE_ERR_CUDA;
  if (major != 10) return CCE_ERR_UNSUPPORTED;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cce_handle* h = new cce_handle();
  h->cfg = *cfg;
  h->device = dev;
  h->num_sms = sms > 0 ? sms : 148;
  *out = h;
  return CCE_OK;
}

cce_status cce_destroy(cce_handle* h) {
  if (!h) return CCE_ERR_INVALID_VALUE;
  for (auto& r : h->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : h->pool) cudaEventDestroy(e);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->ev_a) cudaEventDestroy(h->ev_a);
  if (h->ev_b) cudaEventDestroy(h->ev_b);
  for (auto& e : h->stages)
    if (e.consumed) cudaEventDestroy(e.consumed);
  if (h->ev_copied) cudaEventDestroy(h->ev_copied);
  for (auto p : h->opened)
    if (p) cudaIpcCloseMemHandle(p);
  if (h->grp_launch_dev) cudaFree(h->grp_launch_dev);
  for (int q = 0; q < h->group_n; ++q)  // the other members must not reach this handle any more
    if (h->group[q] && h->group[q] != h) h->group[q]->group_broken = true;
  delete h;
  return CCE_OK;
}

size_t cce_workspace_bytes(const cce_handle* h, int64_t N, int64_t D, int64_t V_local) {
  if (!h || N < 0 || D <= 0 || V_local < 0) return 0;
  return layout(N, D, V_local, h->cfg.world, h->chunk, h->slots, h->cfg.flags).total;
}

int64_t cce_kernel_launches(const cce_handle* h) { return h ? h->launches : 0; }

cce_status cce_debug_trace(cce_handle* h, void* dev_buf, size_t bytes) {
  if (!h || (bytes && !dev_buf)) return CCE_ERR_INVALID_VALUE;
  // first half: backward items, second half: forward items
  const size_t half = (bytes / 2) / sizeof(TraceRec) * sizeof(TraceRec);
  h->trace = bytes ? dev_buf : nullptr;
  h->trace_bytes = half;
  h->fwd_trace = bytes ? static_cast<char*>(dev_buf) + half : nullptr;
  h->fwd_trace_bytes = half;
  return CCE_OK;
}

cce_status cce_profile_enable(cce_handle* h, int32_t on) {
  if (!h) return CCE_ERR_INVALID_VALUE;
  h->prof = on != 0;
  return CCE_OK;
}

cce_status cce_profile_read(cce_handle* h, double* ms_out, int64_t* launches_out, int32_t reset) {
  if (!h) return CCE_ERR_INVALID_VALUE;
  double ms[CCE_PROF_CLASSES] = {0};
  int64_t cnt[CCE_PROF_CLASSES] = {0};
  for (auto& r : h->recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) return CCE_ERR_CUDA;
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) return CCE_ERR_CUDA;
    ms[r.cls] += t;
    cnt[r.cls] += 1;
  }
  for (int i = 0; i < CCE_PROF_CLASSES; ++i) {
    if (ms_out) ms_out[i] = ms[i];
    if (launches_out) launches_out[i] = cnt[i];
  }
  if (reset) {
    for (auto& r : h->recs) {
      h->pool.push_back(r.a);
      h->pool.push_back(r.b);
    }
    h->recs.clear();
  }
  return CCE_OK;
}

struct NormArgs {
  const void* gamma;
  float eps;
};

static cce_status forward_impl(cce_handle* h, const void* H, int64_t N, int64_t D, int64_t ldh, const void* W,
                               int64_t V_local, int64_t ldw, const int32_t* labels, float* loss, float* lse,
                               int32_t* n_valid, void* workspace, size_t workspace_bytes, void* stream,
                               const NormArgs* norm);
static cce_status forward_tail(cce_handle* h, const float4* stats_all, float* loss, float* lse, int32_t* n_valid,
                               cudaStream_t s, const int* wait_flags = nullptr);

cce_status cce_forward(cce_handle* h, const void* H, int64_t N, int64_t D, int64_t ldh, const void* W,
                       int64_t V_local, int64_t ldw, const int32_t* labels, float* loss, float* lse,
                       int32_t* n_valid, void* workspace, size_t workspace_bytes, void* stream) {
  return forward_impl(h, H, N, D, ldh, W, V_local, ldw, labels, loss, lse, n_valid, workspace, workspace_bytes, stream,
                      nullptr);
}

cce_status cce_forward_rmsnorm(cce_handle* h, const void* X, int64_t N, int64_t D, int64_t ldx, const void* gamma,
                               float eps, const void* W, int64_t V_local, int64_t ldw, const int32_t* labels,
                               float* loss, float* lse, int32_t* n_valid, void* workspace, size_t workspace_bytes,
                               void* stream) {
  // eps > 0 (Def. RMSNorm): an all-zero row would otherwise give rstd = inf
  if (!h || !gamma || !(eps > 0.f) || !std::isfinite(eps)) return CCE_ERR_INVALID_VALUE;
  if (!aligned16(gamma) || D > 8192) return CCE_ERR_UNSUPPORTED;
  NormArgs na{gamma, eps};
  return forward_impl(h, X, N, D, ldx, W, V_local, ldw, labels, loss, lse, n_valid, workspace, workspace_bytes, stream,
                      &na);
}

static cce_status forward_impl(cce_handle* h, const void* H, int64_t N, int64_t D, int64_t ldh, const void* W,
                               int64_t V_local, int64_t ldw, const int32_t* labels, float* loss, float* lse,
                               int32_t* n_valid, void* workspace, size_t workspace_bytes, void* stream,
                               const NormArgs* norm) {
  if (!h || !loss || h->group_broken) return CCE_ERR_INVALID_VALUE;
  if (N < 0 || D <= 0 || V_local < 0 || ldh < D || ldw < D) return CCE_ERR_INVALID_VALUE;
  if (N > 0 && (!H || !labels)) return CCE_ERR_INVALID_VALUE;
  if (V_local > 0 && !W) return CCE_ERR_INVALID_VALUE;
  if (h->cfg.vocab_offset + V_local > h->cfg.vocab_total) return CCE_ERR_INVALID_VALUE;
  if (D % 64 != 0 || N > (1LL << 30) || V_local > (1LL << 30)) return CCE_ERR_UNSUPPORTED;
  if ((N > 0 && !aligned16(H)) || (V_local > 0 && !aligned16(W)) || (ldh * 2) % 16 || (ldw * 2) % 16)
    return CCE_ERR_UNSUPPORTED;
  const Layout L = layout(N, D, V_local, h->cfg.world, h->chunk, h->slots, h->cfg.flags);
  if (!workspace || workspace_bytes < L.total || !aligned16(workspace)) return CCE_ERR_WORKSPACE;
  if ((h->cfg.flags & CCE_FLAG_P2P_COMBINE) &&
      (!h->p2p_attached || workspace != h->p2p_ws || N != h->p2p_N || D != h->p2p_D))
    return CCE_ERR_INVALID_VALUE;  // peers address this workspace (layout of the attached N, D)
  // P2P: every rank's backward kernel raises its dH-tile flags and runs its share of the
  // cross-rank reduction; an empty shard would launch no kernel and stall its peers
  if ((h->cfg.flags & CCE_FLAG_P2P_COMBINE) && h->cfg.world > 1 && V_local == 0) return CCE_ERR_UNSUPPORTED;
  if (!get_encode()) return CCE_ERR_CUDA;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  void* ws = workspace;
  int* nvp = at<int>(ws, L.scal);
  int* errp = nvp + 1;

  // a0: label scan + compaction (it also writes n_valid and the label-error word of this
  // forward, and resets zy_c, the forward queue counters and the finalize counter)
  if (N == 0 && cudaMemsetAsync(nvp, 0, 16, s) != cudaSuccess) return CCE_ERR_CUDA;
  if (N > 0) {
    { ProfScope ps(h, s, 4);
    k_label_scan<<<1, 1024, 0, s>>>(labels, (int)N, h->cfg.ignore_index, (long long)h->cfg.vocab_total,
                                    at<int>(ws, L.pos), at<int>(ws, L.idx), at<int>(ws, L.labels_c), nvp, errp,
                                    at<float>(ws, L.zy_c), (int)L.Npad, at<int>(ws, L.sched), nvp + 2); }
    { ProfScope ps(h, s, 4);
    if (norm)  // RMSNorm prologue: normalise the valid rows on the way into Hc, cache rstd
      k_gather_rmsnorm<<<grid_for(L.Npad, 8, 8 * h->num_sms), 256, 0, s>>>(
          static_cast<const __nv_bfloat16*>(H), ldh, (int)D, (int)L.Npad, at<int>(ws, L.idx), nvp,
          static_cast<const __nv_bfloat16*>(norm->gamma), norm->eps, at<__nv_bfloat16>(ws, L.Hc),
          at<float>(ws, L.rstd_c));
    else
      k_gather_rows<<<grid_for((long long)L.Npad * D / 8, 256, 4 * h->num_sms), 256, 0, s>>>(
          static_cast<const __nv_bfloat16*>(H), ldh, (int)D, (int)L.Npad, at<int>(ws, L.idx), nvp,
          at<__nv_bfloat16>(ws, L.Hc)); }
  }

  const bool dB = (h->cfg.flags & CCE_FLAG_DESIGN_B) != 0;
  if (dB && D > dsb::D_MAX) return CCE_ERR_UNSUPPORTED;
  float4* stats = at<float4>(ws, L.stats);
  if (dB) {
    // design B (rows a1-a4 with a3): logits, online softmax and the dH numerator O' in one
    // kernel, then the merge of the per-CTA partials into (m, d, z_y) and U
    if (N > 0 && V_local > 0) {
      CUtensorMap tX, tY1, tY2;
      if (!make_map_colblocks(&tX, at<void>(ws, L.Hc), D, L.Npad, D, dsb::NX, (uint32_t)(D / 64)) ||
          !make_map_colblocks(&tY1, W, D, V_local, ldw, dsb::YM, 2) ||
          !make_map_colblocks(&tY2, W, D, V_local, ldw, dsb::YM, 2))
        return CCE_ERR_CUDA;
      dsb::Params bp{};
      bp.mode = 0;
      bp.D = (int)D; bp.V_local = (int)V_local; bp.vocab_offset = (int)h->cfg.vocab_offset; bp.Npad = (int)L.Npad;
      bp.n_valid = nvp;
      bp.labels_c = at<int>(ws, L.labels_c);
      bp.opart = at<float>(ws, L.b_opart);
      bp.spart = at<float4>(ws, L.b_spart);
      cce_status st = launch_designb(h, tX, tY1, tY2, bp, s, 0);
      if (st != CCE_OK) return st;
    }
    if (N > 0) {
      ProfScope ps(h, s, 4);
      if (V_local > 0) {
        dsb::k_merge_designb<<<(unsigned)((L.Npad + 7) / 8), 256, 0, s>>>(
            at<float>(ws, L.b_opart), at<float4>(ws, L.b_spart), DSB_GRID, (int)V_local,
            (int)h->cfg.vocab_offset, (int)D, nvp, at<int>(ws, L.labels_c), static_cast<const __nv_bfloat16*>(W), ldw,
            stats, at<float>(ws, L.b_U));
      }
    }
  }
  // a1 + a2: tcgen05 logit tiles with the online-softmax epilogue
  if (!dB && N > 0 && V_local > 0) {
    GemmParams p{};
    p.D = (int)D;
    p.V_local = (int)V_local;
    p.Npad = (int)L.Npad;
    p.C = (int)L.C;
    p.vocab_offset = (int)h->cfg.vocab_offset;
    p.n_valid = nvp;
    p.labels_c = at<int>(ws, L.labels_c);
    p.part = at<float2>(ws, L.part);
    p.zy_c = at<float>(ws, L.zy_c);
    p.ls_eps = h->cfg.label_smoothing;
    p.z_loss = h->cfg.z_loss;
    p.inv_vtotal = (float)(1.0 / (double)h->cfg.vocab_total);
    p.zs_part = h->cfg.label_smoothing > 0.f ? at<float>(ws, L.zs_part) : nullptr;
    // KPS k-blocks per box (column-block views)
    CUtensorMap tA, tB;
    if (!make_map_colblocks(&tA, at<void>(ws, L.Hc), D, L.Npad, D, pairk::HM, pairk::KPS) ||
        !make_map_colblocks(&tB, W, D, V_local, ldw, pairk::PN / 2, pairk::KPS))
      return CCE_ERR_CUDA;
    pairk::PairParams pp{};
    pp.g = p;
    pp.mode = 0;
    pp.n_chunks = 0;
    pp.slots = h->slots;
    pp.jit_tail = CCE_JIT_TAIL;
    pp.sched = at<int>(ws, L.sched);
    pp.trace = static_cast<TraceRec*>(h->fwd_trace);
    pp.trace_cap = (int)(h->fwd_trace_bytes / sizeof(TraceRec));
    cce_status st = launch_pair(h, tA, tB, tA, tA, tA, tA, tA, pp, s, 0);
    if (st != CCE_OK) return st;
  }

  // a4: merge tiles -> per-rank stats; a9: allgather across vocabulary shards
  bool merged_final = false;
  if (!dB && N > 0) {
    // an empty shard (V_local == 0) merges zero tiles: (m=-inf, d=0, z_y=0) for every row
    ProfScope ps(h, s, 4);
    StatsPush push{};
    if (h->cfg.flags & CCE_FLAG_P2P_COMBINE) {  // a9 fused: every rank's slot `rank`, including ours
      const size_t half = (size_t)((h->epoch + 1) & 1) * h->cfg.world * L.Npad;  // this step's half
      for (int r = 0; r < h->cfg.world; ++r) {
        push.dst[r] = reinterpret_cast<float4*>(h->peers.ws[r] + L.stats_all) + half + (size_t)h->cfg.rank * L.Npad;
        push.flag[r] = reinterpret_cast<int*>(h->peers.ws[r] + L.p2p_flags) + P2P_STATS * P2P_MAX + h->cfg.rank;
      }
      push.n = h->cfg.world;
      push.epoch = h->epoch + 1;  // this forward's epoch (incremented below)
      push.counter = nvp + 3;
    }
    // one rank, no exchange: the finalize (lse, row losses, the deterministic loss reduction)
    // runs in the merge kernel's tail
    MergeFinalize fin{};
    if (h->cfg.world == 1 && !h->cfg.nccl_comm && !(h->cfg.flags & (CCE_FLAG_EXTERNAL_COMBINE | CCE_FLAG_P2P_COMBINE))) {
      const bool none = h->cfg.reduction == CCE_REDUCTION_NONE;
      fin.on = 1;
      fin.pos = at<int>(ws, L.pos);
      fin.idx = at<int>(ws, L.idx);
      fin.N = (int)N;
      fin.lse_out = lse;
      fin.lse_c = at<float>(ws, L.lse_c);
      fin.loss_rows = at<float>(ws, L.loss_rows);
      fin.loss_tok = none ? loss : nullptr;
      fin.ls_eps = h->cfg.label_smoothing;
      fin.z_loss = h->cfg.z_loss;
      fin.inv_vtotal = (float)(1.0 / (double)h->cfg.vocab_total);
      fin.err = errp;
      fin.loss = none ? nullptr : loss;
      fin.n_valid_out = n_valid;
      fin.sum = h->cfg.reduction == CCE_REDUCTION_SUM ? 1 : 0;
      fin.counter = nvp + 2;
      merged_final = true;
    }
    k_merge_tiles<<<(unsigned)((L.Npad + 31) / 32), 32 * MERGE_SL, 0, s>>>(
        at<float2>(ws, L.part), V_local > 0 ? (int)L.Tv : 0, (int)L.Npad, at<float>(ws, L.zy_c), nvp,
        (h->cfg.label_smoothing > 0.f && V_local > 0) ? at<float>(ws, L.zs_part) : nullptr, stats, push, fin);
  }
  h->have_fwd = false;
  h->norm = norm != nullptr;
  h->nX = H;
  h->ldx = ldh;
  h->gamma = norm ? norm->gamma : nullptr;
  h->W = W;
  h->N = N;
  h->D = D;
  h->V_local = V_local;
  h->ldw = ldw;
  h->ws = workspace;
  h->ws_bytes = workspace_bytes;
  if (h->cfg.flags & CCE_FLAG_P2P_COMBINE) {
    // a9 over peer memory: push this rank's stats into every rank's all-ranks array, raise
    // the flag, wait for every rank's
    // (the merge above stored the stats into every rank and raised this rank's flag everywhere)
    const int epoch = ++h->epoch;
    if (N == 0)
      k_p2p_signal<<<1, 32, 0, s>>>(h->peers, (unsigned long long)L.p2p_flags, P2P_STATS, h->cfg.rank, h->cfg.world,
                                    epoch);
    if (h->group_n) {
      // one-GPU group emulation: every rank pushes and signals before any rank waits
      h->grp_fwd_pending = true;
      h->grp_stream = s;
      h->p_loss = loss;
      h->p_lse = lse;
      h->p_nv = n_valid;
      if (h->cfg.rank + 1 < h->group_n) return cudaGetLastError() == cudaSuccess ? CCE_OK : CCE_ERR_CUDA;
      for (int q = 0; q < h->group_n; ++q) {
        cce_handle* g = h->group[q];
        if (!g->grp_fwd_pending || g->epoch != epoch || g->grp_stream != s) return CCE_ERR_NO_FORWARD;
      }
      for (int q = 0; q < h->group_n; ++q) {
        cce_handle* g = h->group[q];
        g->grp_fwd_pending = false;
        const Layout Lq = layout(g->N, g->D, g->V_local, g->cfg.world, g->chunk, g->slots, g->cfg.flags);
        const cce_status st = forward_tail(g, at<float4>(g->ws, Lq.stats_all) + (size_t)(epoch & 1) * g->cfg.world * Lq.Npad,
                                           g->p_loss, g->p_lse, g->p_nv, s, at<int>(g->ws, Lq.p2p_flags) + P2P_STATS * P2P_MAX);
        if (st != CCE_OK) return st;
      }
      return CCE_OK;
    }
    return forward_tail(h, at<float4>(ws, L.stats_all) + (size_t)(epoch & 1) * h->cfg.world * L.Npad, loss, lse,
                        n_valid, s, at<int>(ws, L.p2p_flags) + P2P_STATS * P2P_MAX);  // the wait runs in the finalize
  }
  if (h->cfg.flags & CCE_FLAG_EXTERNAL_COMBINE) {
    // a9 done by the caller: it gathers every rank's `stats` into `stats_all`, then calls
    // cce_forward_finish (cce_combine_offsets locates both in the workspace)
    if (cudaGetLastError() != cudaSuccess) return CCE_ERR_CUDA;
    h->fwd_pending = true;
    h->p_loss = loss;
    h->p_lse = lse;
    h->p_nv = n_valid;
    return CCE_OK;
  }
  const float4* stats_all = stats;
  if (h->cfg.nccl_comm) {
    Nccl& n = nccl();
    if (!n.ok) return CCE_ERR_NCCL;
    if (n.allgather(stats, at<float4>(ws, L.stats_all), (size_t)L.Npad * 4, kNcclFloat32, h->cfg.nccl_comm, s) != 0)
      return CCE_ERR_NCCL;
    stats_all = at<float4>(ws, L.stats_all);
  }
  if (merged_final) {
    if (cudaGetLastError() != cudaSuccess) return CCE_ERR_CUDA;
    h->have_fwd = true;
    return CCE_OK;
  }
  return forward_tail(h, stats_all, loss, lse, n_valid, s);
}

// a4 (global) + loss: per-row LSE / loss from the (gathered) per-rank stats.
static cce_status forward_tail(cce_handle* h, const float4* stats_all, float* loss, float* lse, int32_t* n_valid,
                               cudaStream_t s, const int* wait_flags) {
  const int64_t N = h->N;
  const Layout L = layout(N, h->D, h->V_local, h->cfg.world, h->chunk, h->slots, h->cfg.flags);
  void* ws = h->ws;
  int* nvp = at<int>(ws, L.scal);
  int* errp = nvp + 1;
  if (N > 0) {
    // per-row LSE / loss and, in the last block, the deterministic loss reduction
    ProfScope ps(h, s, 4);
    k_finalize_loss<<<grid_for(N, 256, 8 * h->num_sms), 256, 0, s>>>(
        stats_all, h->cfg.world, (int)L.Npad, at<int>(ws, L.pos), (int)N, lse, at<float>(ws, L.lse_c),
        at<float>(ws, L.loss_rows), h->cfg.label_smoothing, h->cfg.z_loss, (float)(1.0 / (double)h->cfg.vocab_total),
        h->cfg.reduction == CCE_REDUCTION_NONE ? loss : nullptr, nvp, errp,
        h->cfg.reduction == CCE_REDUCTION_NONE ? nullptr : loss, n_valid, h->cfg.reduction == CCE_REDUCTION_SUM ? 1 : 0,
        nvp + 2, wait_flags, h->epoch, errp);
  } else {
    ProfScope ps(h, s, 4);
    k_loss<<<1, 1024, 0, s>>>(at<float>(ws, L.loss_rows), nvp, errp,
                              h->cfg.reduction == CCE_REDUCTION_NONE ? nullptr : loss, n_valid,
                              h->cfg.reduction == CCE_REDUCTION_SUM ? 1 : 0);
  }
  if (cudaGetLastError() != cudaSuccess) return CCE_ERR_CUDA;
  h->have_fwd = true;
  return CCE_OK;
}

cce_status cce_forward_finish(cce_handle* h, void* stream) {
  if (!h) return CCE_ERR_INVALID_VALUE;
  if (!h->fwd_pending) return CCE_ERR_NO_FORWARD;
  h->fwd_pending = false;
  const Layout L = layout(h->N, h->D, h->V_local, h->cfg.world, h->chunk, h->slots, h->cfg.flags);
  return forward_tail(h, at<float4>(h->ws, L.stats_all), h->p_loss, h->p_lse, h->p_nv,
                      static_cast<cudaStream_t>(stream));
}

cce_status cce_combine_offsets(const cce_handle* h, int64_t N, int64_t D, int64_t V_local, int64_t* out4) {
  if (!h || !out4 || N < 0 || D <= 0 || V_local < 0) return CCE_ERR_INVALID_VALUE;
  const Layout L = layout(N, D, V_local, h->cfg.world, h->chunk, h->slots, h->cfg.flags);
  out4[0] = (int64_t)L.stats;      // this rank's stats: float [Npad][4] (m, d, z_y, sum z)
  out4[1] = (int64_t)L.stats_all;  // all ranks' stats: float [world][Npad][4], rank-major
  // this rank's partial dH: float [Npad][D] compact valid rows, or with CCE_FLAG_DH_SEQ_SHARD
  // float [world x slice][D] in original row order (rank r's slice at r x slice rows)
  out4[2] = (h->cfg.flags & CCE_FLAG_DH_SEQ_SHARD) ? (int64_t)L.dHo : (int64_t)L.dH32;
  out4[3] = L.Npad;
  return CCE_OK;
}

static cce_status launch_adamw(const cce_adamw_params* opt, const void* grad, int grad_fp32, int64_t n, void* W_bf16,
                               cudaStream_t s) {
  if (n <= 0) return CCE_OK;
  AdamwArgs a;
  a.lr = opt->lr; a.b1 = opt->beta1; a.b2 = opt->beta2; a.eps = opt->eps; a.wd = opt->weight_decay;
  a.bc1 = opt->bias_correction1; a.bc2 = opt->bias_correction2;
  a.clip = opt->clip_coef; a.master = opt->master; a.m = opt->m; a.v = opt->v; a.grad_in = opt->grad_in;
  a.grad = grad; a.grad_fp32 = grad_fp32; a.w = static_cast<__nv_bfloat16*>(W_bf16); a.n = n;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long groups = n / 8 > 0 ? n / 8 : 1;
  k_adamw<<<grid_for(groups, 256, 8 * sms), 256, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? CCE_OK : CCE_ERR_CUDA;
}

static bool adamw_params_ok(const cce_adamw_params* o) {
  return o && o->m && o->v && o->bias_correction1 > 0.f && o->bias_correction2 > 0.f;
}

static bool adamw_aligned(const cce_adamw_params* o) {
  return aligned16(o->m) && aligned16(o->v) && (!o->master || aligned16(o->master)) &&
         (!o->grad_in || aligned16(o->grad_in));
}

static cce_status backward_impl(cce_handle* h, const float* dloss, void* dH, void* dW, const cce_adamw_params* opt,
                                void* stream, void* dgamma = nullptr, bool norm = false);
static cce_status backward_tail(cce_handle* h, void* dH, void* dgamma, bool norm, cudaStream_t s);
static cce_status group_backward(cce_handle* h, void* dH, void* dgamma, bool norm, cudaStream_t s);

cce_status cce_backward_rmsnorm(cce_handle* h, const float* dloss, void* dX, void* dgamma, void* dW, void* stream) {
  if (!h) return CCE_ERR_INVALID_VALUE;
  if (h->cfg.flags & (CCE_FLAG_EXTERNAL_COMBINE | CCE_FLAG_DH_SEQ_SHARD)) return CCE_ERR_UNSUPPORTED;
  if (!h->have_fwd || !h->norm) return CCE_ERR_NO_FORWARD;
  if (!dgamma) return CCE_ERR_INVALID_VALUE;
  if (!aligned16(dgamma)) return CCE_ERR_UNSUPPORTED;
  return backward_impl(h, dloss, dX, dW, nullptr, stream, dgamma, true);
}

cce_status cce_backward(cce_handle* h, const float* dloss, void* dH, void* dW, void* stream) {
  return backward_impl(h, dloss, dH, dW, nullptr, stream);
}

cce_status cce_backward_adamw(cce_handle* h, const float* dloss, void* dH, const cce_adamw_params* opt,
                              void* stream) {
  if (!h) return CCE_ERR_INVALID_VALUE;
  if (!h->have_fwd) return CCE_ERR_NO_FORWARD;
  if (!adamw_params_ok(opt)) return CCE_ERR_INVALID_VALUE;
  if (h->cfg.flags & (CCE_FLAG_EXTERNAL_COMBINE | CCE_FLAG_P2P_COMBINE)) return CCE_ERR_UNSUPPORTED;
  if (h->cfg.flags & CCE_FLAG_ACCUMULATE) return CCE_ERR_UNSUPPORTED;
  if (!adamw_aligned(opt) || (h->D % 8) != 0 || (opt->W_out && !aligned16(opt->W_out))) return CCE_ERR_UNSUPPORTED;
  return backward_impl(h, dloss, dH, const_cast<void*>(h->W), opt, stream);
}

cce_status cce_adamw_step(const cce_adamw_params* opt, const void* grad, int32_t grad_fp32, int64_t n, void* W_bf16,
                          void* stream) {
  if (!adamw_params_ok(opt) || n < 0 || (!opt->master && !W_bf16)) return CCE_ERR_INVALID_VALUE;
  if (!adamw_aligned(opt) || (W_bf16 && !aligned16(W_bf16)) || (grad && !aligned16(grad)))
    return CCE_ERR_UNSUPPORTED;
  return launch_adamw(opt, grad, grad_fp32 ? 1 : 0, n, W_bf16, static_cast<cudaStream_t>(stream));
}

// CCE_FLAG_DH_SEQ_SHARD: this rank's reduced slice of the original-order dH -> dH [n_r, D]
static cce_status seq_rows_out(cce_handle* h, const Layout& L, void* dH, cudaStream_t s) {
  const int64_t slice = L.seq_slice, r = h->cfg.rank;
  const int64_t n_r = std::max<int64_t>(0, std::min<int64_t>(slice, h->N - r * slice));
  if (n_r == 0) return CCE_OK;
  ProfScope ps(h, s, 4);
  k_rows_out<<<grid_for(n_r * h->D / 8, 256, 8 * h->num_sms), 256, 0, s>>>(
      at<float>(h->ws, L.dHo) + r * slice * h->D, (int)n_r, (int)h->D, dH,
      (h->cfg.flags & CCE_FLAG_GRAD_FP32) ? 1 : 0, (h->cfg.flags & CCE_FLAG_ACCUMULATE) ? 1 : 0);
  return cudaGetLastError() == cudaSuccess ? CCE_OK : CCE_ERR_CUDA;
}

static cce_status backward_impl(cce_handle* h, const float* dloss, void* dH, void* dW, const cce_adamw_params* opt,
                                void* stream, void* dgamma, bool norm) {
  if (!h || h->group_broken) return CCE_ERR_INVALID_VALUE;
  if (!h->have_fwd) return CCE_ERR_NO_FORWARD;
  if (!dloss || (h->N > 0 && !dH) || (h->V_local > 0 && !dW)) return CCE_ERR_INVALID_VALUE;
  if ((dH && !aligned16(dH)) || (dW && !aligned16(dW))) return CCE_ERR_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t N = h->N, D = h->D, V_local = h->V_local;
  const Layout L = layout(N, D, V_local, h->cfg.world, h->chunk, h->slots, h->cfg.flags);
  void* ws = h->ws;
  int* nvp = at<int>(ws, L.scal);
  float* dH32 = at<float>(ws, L.dH32);
  h->dH_reduced = false;

  const bool dB = (h->cfg.flags & CCE_FLAG_DESIGN_B) != 0;
  if (dB && opt) return CCE_ERR_UNSUPPORTED;
  if (dB && V_local > 0 && N > 0) {
    // design B backward (rows a5-a7 with a6 on chip): S recompute, G in shared memory, dW;
    // dH = s U (the forward's numerator), scaled into dH32 for the common tail below
    const float* dloss_c = nullptr;
    if (h->cfg.reduction == CCE_REDUCTION_NONE) {
      ProfScope ps(h, s, 4);
      k_gather_dloss<<<grid_for(L.Npad, 256, 2 * h->num_sms), 256, 0, s>>>(dloss, at<int>(ws, L.idx), nvp,
                                                                           (int)L.Npad, at<float>(ws, L.dloss_c));
      dloss_c = at<float>(ws, L.dloss_c);
    }
    void* Hc = at<void>(ws, L.Hc);
    CUtensorMap tX, tY1, tY2;
    if (!make_map_colblocks(&tX, h->W, D, V_local, h->ldw, dsb::NX, (uint32_t)(D / 64)) ||
        !make_map_colblocks(&tY1, Hc, D, L.Npad, D, dsb::YM, 2) || !make_map_colblocks(&tY2, Hc, D, L.Npad, D, dsb::YM, 2))
      return CCE_ERR_CUDA;
    dsb::Params bp{};
    bp.mode = 1;
    bp.D = (int)D; bp.V_local = (int)V_local; bp.vocab_offset = (int)h->cfg.vocab_offset; bp.Npad = (int)L.Npad;
    bp.n_valid = nvp;
    bp.labels_c = at<int>(ws, L.labels_c);
    bp.lse_c = at<float>(ws, L.lse_c);
    bp.dloss = dloss;
    bp.dloss_c = dloss_c;
    bp.reduction = h->cfg.reduction;
    bp.dW = dW;
    bp.dw_fp32 = (h->cfg.flags & CCE_FLAG_GRAD_FP32) ? 1 : 0;
    bp.dw_accumulate = (h->cfg.flags & CCE_FLAG_ACCUMULATE) ? 1 : 0;
    cce_status st = launch_designb(h, tX, tY1, tY2, bp, s, 1);
    if (st != CCE_OK) return st;
    ProfScope ps(h, s, 4);
    dsb::k_scale_rows<<<grid_for(L.Npad * D, 256, 8 * h->num_sms), 256, 0, s>>>(
        at<float>(ws, L.b_U), dH32, (int)D, nvp, dloss, dloss_c, h->cfg.reduction);
  } else if (V_local > 0 && N > 0) {
    void* Hc = at<void>(ws, L.Hc);
    void* G = at<void>(ws, L.gbuf);
    GemmParams p{};
    p.D = (int)D;
    p.V_local = (int)V_local;
    p.Npad = (int)L.Npad;
    p.C = (int)L.C;
    p.vocab_offset = (int)h->cfg.vocab_offset;
    p.n_valid = nvp;
    p.labels_c = at<int>(ws, L.labels_c);
    p.lse_c = at<float>(ws, L.lse_c);
    p.dloss = dloss;
    p.gbuf = at<__nv_bfloat16>(ws, L.gbuf);
    p.dW = dW;
    p.reduction = h->cfg.reduction;
    p.dw_fp32 = (h->cfg.flags & CCE_FLAG_GRAD_FP32) ? 1 : 0;
    p.dw_accumulate = (h->cfg.flags & CCE_FLAG_ACCUMULATE) ? 1 : 0;
    p.dloss_c = nullptr;
    if (opt) {
      p.adamw = 1;
      p.lr = opt->lr; p.beta1 = opt->beta1; p.beta2 = opt->beta2; p.eps = opt->eps; p.wd = opt->weight_decay;
      p.bc1 = opt->bias_correction1; p.bc2 = opt->bias_correction2;
      p.clip_coef = opt->clip_coef; p.master = opt->master; p.am = opt->m; p.av = opt->v; p.grad_in = opt->grad_in;
      p.Win = static_cast<const __nv_bfloat16*>(h->W);
      p.Wout = static_cast<__nv_bfloat16*>(opt->W_out ? opt->W_out : dW);
      p.adamw_inplace = (p.Wout == p.Win) ? 1 : 0;
      p.ldw = (int)h->ldw;
      p.dW = nullptr;
    }
    if (h->cfg.reduction == CCE_REDUCTION_NONE) {
      ProfScope ps(h, s, 4);
      k_gather_dloss<<<grid_for(L.Npad, 256, 2 * h->num_sms), 256, 0, s>>>(dloss, at<int>(ws, L.idx), nvp,
                                                                           (int)L.Npad, at<float>(ws, L.dloss_c));
      p.dloss_c = at<float>(ws, L.dloss_c);
    }
    p.dH32 = dH32;
    p.ls_eps = h->cfg.label_smoothing;
    p.z_loss = h->cfg.z_loss;
    p.inv_vtotal = (float)(1.0 / (double)h->cfg.vocab_total);
    const int slots = h->slots;
    // CTA-pair persistent backward: G / DW / DH tiles of every chunk from one work queue.
    // One TMA instruction per operand per stage: K-major boxes of KPS 64-column blocks
    // (Hc, W_c, dlogits rows), MN-major boxes of two 64-column blocks x KPS k-blocks
    // (dlogits columns, Hc / W_c for the 256-wide hidden tiles; the 2-D maps serve the
    // 128-wide tail tile).
    CUtensorMap mHcK, mWK, mGMN, mHcMN, mGK, mWMN, mHcMN3, mWMN3, mGst, mDH;
    const uint32_t kr = pairk::KPS * 64;  // k-rows per box (MN-major operands)
    if (!make_map_colblocks(&mHcMN3, Hc, D, L.Npad, D, kr, 2) ||
        !make_map_colblocks(&mWMN3, h->W, D, V_local, h->ldw, kr, 2) ||
        !make_map_colblocks(&mHcK, Hc, D, L.Npad, D, pairk::HM, pairk::KPS) ||
        !make_map_colblocks(&mWK, h->W, D, V_local, h->ldw, pairk::PN / 2, pairk::KPS) ||
        !make_map_blocked2(&mGMN, G, L.Npad, slots * (L.C / 64), kr, 2) ||
        !make_map(&mHcMN, Hc, D, L.Npad, D, kr) ||
        !make_map_blocked2(&mGK, G, L.Npad, slots * (L.C / 64), pairk::HM, pairk::KPS) ||
        !make_map(&mWMN, h->W, D, V_local, h->ldw, kr) ||
        !make_map_blocked2(&mGst, G, L.Npad, slots * (L.C / 64), 32, 1) ||  // dlogits TMA stores
        !make_map_f32(&mDH, dH32, D, L.Npad, D, 32, 32))
      return CCE_ERR_CUDA;
    if (cudaMemsetAsync(at<int>(ws, L.sched), 0, (size_t)L.sched_ints * 4, s) != cudaSuccess) return CCE_ERR_CUDA;
    pairk::PairParams pp{};
    pp.g = p;
    pp.mode = 1;
    pp.n_chunks = (int)L.n_chunks;
    pp.slots = slots;
    pp.jit_tail = CCE_JIT_TAIL;
    // queue order: G of chunk c + 1 is queued before W of chunk c (deadlock-free iff
    // (lookahead + 1) * qblock <= slots; measured: larger blocks / lookaheads are equal)
    pp.qblock = 1;
    pp.lookahead = CCE_LOOKAHEAD;
    pp.sched = at<int>(ws, L.sched);
    pp.trace = static_cast<TraceRec*>(h->trace);
    pp.trace_cap = (int)(h->trace_bytes / sizeof(TraceRec));
    if ((h->cfg.flags & CCE_FLAG_P2P_COMBINE) && h->cfg.world > 1) {
      pp.peers = h->peers;
      pp.world = h->cfg.world;
      pp.prank = h->cfg.rank;
      pp.epoch = h->epoch;
      pp.tmax = (int)L.p2p_tmax;
      pp.ready_off = L.p2p_ready;
      pp.done_off = L.p2p_done;
      pp.dH32_off = L.dH32;
      pp.dHred_off = L.dHred;
      pp.err = nvp + 1;
    }
    // NCCL dH all-reduce (a10) overlapped with the last chunk's dW items: the backward queue
    // runs as two launches; after the first (every dH tile final) the all-reduce starts on a
    // side stream while the second launch, on 8 fewer CTA pairs so NCCL's kernels find free
    // SMs, finishes dW
    const bool split = h->cfg.nccl_comm != nullptr && !(h->cfg.flags & CCE_FLAG_DH_SEQ_SHARD) && !norm;
    cce_status st;
    if (h->group_n) {
      // one-GPU group emulation: the launch is issued for every rank at once by the last rank
      const CUtensorMap* ms[10] = {&mHcK, &mWK, &mGMN, &mHcMN, &mGK, &mWMN, &mDH, &mHcMN3, &mWMN3, &mGst};
      for (int i = 0; i < 10; ++i) h->grp_launch.m[i] = *ms[i];
      h->grp_launch.P = pp;
      h->grp_has_launch = true;
    } else if (!split) {
      st = launch_pair(h, mHcK, mWK, mGMN, mHcMN, mGK, mWMN, mDH, pp, s, 1, &mHcMN3, &mWMN3, &mGst);
      if (st != CCE_OK) return st;
    } else {
      if (!h->side && (cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking) != cudaSuccess ||
                       cudaEventCreateWithFlags(&h->ev_a, cudaEventDisableTiming) != cudaSuccess ||
                       cudaEventCreateWithFlags(&h->ev_b, cudaEventDisableTiming) != cudaSuccess))
        return CCE_ERR_CUDA;
      pp.part = 1;
      st = launch_pair(h, mHcK, mWK, mGMN, mHcMN, mGK, mWMN, mDH, pp, s, 1, &mHcMN3, &mWMN3, &mGst);
      if (st != CCE_OK) return st;
      if (cudaEventRecord(h->ev_a, s) != cudaSuccess || cudaStreamWaitEvent(h->side, h->ev_a, 0) != cudaSuccess)
        return CCE_ERR_CUDA;
      Nccl& n = nccl();
      if (!n.ok) return CCE_ERR_NCCL;
      if (n.allreduce(dH32, dH32, (size_t)L.Npad * D, kNcclFloat32, kNcclSum, h->cfg.nccl_comm, h->side) != 0)
        return CCE_ERR_NCCL;
      if (cudaEventRecord(h->ev_b, h->side) != cudaSuccess) return CCE_ERR_CUDA;
      pp.part = 2;
      st = launch_pair(h, mHcK, mWK, mGMN, mHcMN, mGK, mWMN, mDH, pp, s, 1, &mHcMN3, &mWMN3, &mGst,
                       std::max(1, h->num_sms / 2 - 8));
      if (st != CCE_OK) return st;
      if (cudaStreamWaitEvent(s, h->ev_b, 0) != cudaSuccess) return CCE_ERR_CUDA;
      h->dH_reduced = true;
    }
  } else if (V_local > 0 && N == 0 && opt) {
    // no rows: zero gradient, the optimizer step still applies (decay, moment decay)
    if (h->ldw != D) return CCE_ERR_UNSUPPORTED;
    void* wout = opt->W_out ? opt->W_out : dW;
    if (wout != dW && !opt->master &&
        cudaMemcpyAsync(wout, dW, (size_t)V_local * D * 2, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return CCE_ERR_CUDA;  // theta is read from W_out below
    cce_status st = launch_adamw(opt, nullptr, 0, V_local * D, wout, s);
    if (st != CCE_OK) return st;
  } else if (V_local > 0 && N == 0) {
    // no rows: dW = 0 (unchanged when accumulating)
    if (!(h->cfg.flags & CCE_FLAG_ACCUMULATE) &&
        cudaMemsetAsync(dW, 0, (size_t)V_local * D * ((h->cfg.flags & CCE_FLAG_GRAD_FP32) ? 4 : 2), s) != cudaSuccess)
      return CCE_ERR_CUDA;
  }
  if (h->group_n) return group_backward(h, dH, dgamma, norm, s);
  return backward_tail(h, dH, dgamma, norm, s);
}

// Everything after the backward kernel: the dH exchange (a10), the scatter to the original
// rows (or the RMSNorm backward / the sequence-sharded slice).
static cce_status backward_tail(cce_handle* h, void* dH, void* dgamma, bool norm, cudaStream_t s) {
  const int64_t N = h->N, D = h->D, V_local = h->V_local;
  const Layout L = layout(N, D, V_local, h->cfg.world, h->chunk, h->slots, h->cfg.flags);
  void* ws = h->ws;
  int* nvp = at<int>(ws, L.scal);
  float* dH32 = at<float>(ws, L.dH32);
  const bool seq = (h->cfg.flags & CCE_FLAG_DH_SEQ_SHARD) != 0;
  float* dHo = seq ? at<float>(ws, L.dHo) : nullptr;
  const int* p2p_done = nullptr;  // peer-memory exchange: the scatter waits for the reduced tiles
  if (N > 0) {
    if (V_local == 0 && cudaMemsetAsync(dH32, 0, (size_t)L.Npad * D * 4, s) != cudaSuccess) return CCE_ERR_CUDA;
    if (seq) {
      // sequence-sharded dH: this rank's partial in ORIGINAL row order (ignored rows 0, pad
      // rows up to world x slice zeroed), the array the reduce-scatter splits by rank
      ProfScope ps(h, s, 4);
      k_scatter_dH<<<grid_for((long long)N * D / 8, 256, 8 * h->num_sms), 256, 0, s>>>(dH32, at<int>(ws, L.pos),
                                                                                       (int)N, (int)D, dHo, 1, 0);
      const int64_t pad = h->cfg.world * L.seq_slice - N;
      if (pad > 0 && cudaMemsetAsync(dHo + N * D, 0, (size_t)pad * D * 4, s) != cudaSuccess) return CCE_ERR_CUDA;
    }
    if (h->cfg.flags & CCE_FLAG_EXTERNAL_COMBINE) {
      // a10 done by the caller: it sums every rank's partial dH32 in place, then calls
      // cce_backward_finish (the scatter to dH)
      if (cudaGetLastError() != cudaSuccess) return CCE_ERR_CUDA;
      h->bwd_pending = true;
      h->p_dH = dH;
      return CCE_OK;
    }
    if ((h->cfg.flags & CCE_FLAG_P2P_COMBINE) && h->cfg.world > 1) {
      // a10 over peer memory, fused into the backward kernel (RED items, tile by tile): here
      // only wait until every tile's reduced dH has arrived in this rank's reduced array
      // (the dH scatter below waits for every tile's done flags itself; the RMSNorm backward
      // reads the reduced dH from its own kernel, so a wait launch precedes it)
      if (norm) k_p2p_wait_tiles<<<1, 256, 0, s>>>(at<int>(ws, L.p2p_done), nvp, (int)D, h->epoch, nvp + 1);
      else p2p_done = at<int>(ws, L.p2p_done);
      dH32 = at<float>(ws, L.dHred);
    }
    if (h->cfg.nccl_comm && !h->dH_reduced) {
      // a10: dH partials summed over the vocabulary shards (all-reduce), or reduce-scattered
      // by sequence slice (CCE_FLAG_DH_SEQ_SHARD; in place: rank r's slice at r x slice rows)
      Nccl& n = nccl();
      if (!n.ok) return CCE_ERR_NCCL;
      if (seq) {
        const size_t cnt = (size_t)L.seq_slice * D;
        if (n.reducescatter(dHo, dHo + (size_t)h->cfg.rank * cnt, cnt, kNcclFloat32, kNcclSum, h->cfg.nccl_comm, s) != 0)
          return CCE_ERR_NCCL;
      } else if (n.allreduce(dH32, dH32, (size_t)L.Npad * D, kNcclFloat32, kNcclSum, h->cfg.nccl_comm, s) != 0) {
        return CCE_ERR_NCCL;
      }
    }
    if (seq) return seq_rows_out(h, L, dH, s);
    if (norm) {
      // RMSNorm backward from the unrounded fp32 dH: dX (valid rows), dgamma, zeros for ignored rows
      const int gf = (h->cfg.flags & CCE_FLAG_GRAD_FP32) ? 1 : 0, ac = (h->cfg.flags & CCE_FLAG_ACCUMULATE) ? 1 : 0;
      const size_t sm = (size_t)RMS_BWD_WARPS * D * 4;
      if (sm > 48 * 1024 &&
          cudaFuncSetAttribute(k_rmsnorm_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
        return CCE_ERR_CUDA;
      { ProfScope ps(h, s, 4);
      k_rmsnorm_bwd<<<RMS_GP, 32 * RMS_BWD_WARPS, sm, s>>>(
          dH32, static_cast<const __nv_bfloat16*>(h->nX), h->ldx, at<int>(ws, L.idx), nvp,
          static_cast<const __nv_bfloat16*>(h->gamma), at<float>(ws, L.rstd_c), (int)D, dH, gf, ac,
          at<float>(ws, L.gpart)); }
      { ProfScope ps(h, s, 4);
      k_dgamma_reduce<<<grid_for(D, 256, 64), 256, 0, s>>>(at<float>(ws, L.gpart), RMS_GP, (int)D, dgamma, gf, ac); }
      if (!ac) {
        ProfScope ps(h, s, 4);
        k_zero_ignored<<<grid_for((long long)N * D / 8, 256, 4 * h->num_sms), 256, 0, s>>>(at<int>(ws, L.pos), (int)N,
                                                                                         (int)D, dH, gf);
      }
      if (cudaGetLastError() != cudaSuccess) return CCE_ERR_CUDA;
      return CCE_OK;
    }
    ProfScope ps(h, s, 4);
    k_scatter_dH<<<grid_for((long long)N * D / 8, 256, 8 * h->num_sms), 256, 0, s>>>(
        dH32, at<int>(ws, L.pos), (int)N, (int)D, dH, (h->cfg.flags & CCE_FLAG_GRAD_FP32) ? 1 : 0,
        (h->cfg.flags & CCE_FLAG_ACCUMULATE) ? 1 : 0, p2p_done, nvp, h->epoch, nvp + 1);
  } else if (norm && !(h->cfg.flags & CCE_FLAG_ACCUMULATE)) {
    // no rows: dgamma = 0
    if (cudaMemsetAsync(dgamma, 0, (size_t)D * ((h->cfg.flags & CCE_FLAG_GRAD_FP32) ? 4 : 2), s) != cudaSuccess)
      return CCE_ERR_CUDA;
  }
  if (cudaGetLastError() != cudaSuccess) return CCE_ERR_CUDA;
  return CCE_OK;
}

// One-GPU group emulation (cce_p2p_attach_group): ranks 0 .. n-2 only record their launch and
// tail; the last rank issues ONE backward launch holding every rank's queue on its own CTA
// pairs (co-resident by construction, cooperative when the driver accepts it), then every
// rank's tail in rank order.
static cce_status group_backward(cce_handle* h, void* dH, void* dgamma, bool norm, cudaStream_t s) {
  h->grp_bwd_pending = true;
  h->grp_dH = dH;
  h->grp_dgamma = dgamma;
  h->grp_norm = norm;
  h->grp_stream = s;
  const int n = h->group_n;
  if (h->cfg.rank + 1 < n) return cudaGetLastError() == cudaSuccess ? CCE_OK : CCE_ERR_CUDA;
  int with_kernel = 0;
  for (int q = 0; q < n; ++q) {
    const cce_handle* g = h->group[q];
    if (!g->grp_bwd_pending || g->grp_stream != s || g->epoch != h->epoch) return CCE_ERR_NO_FORWARD;
    with_kernel += g->grp_has_launch ? 1 : 0;
  }
  if (with_kernel != 0 && with_kernel != n) return CCE_ERR_UNSUPPORTED;  // (empty shards are refused in P2P mode)
  if (with_kernel == n) {
    std::vector<pairk::PairLaunch> all(n);
    for (int q = 0; q < n; ++q) all[q] = h->group[q]->grp_launch;
    if (cudaMemcpyAsync(h->grp_launch_dev, all.data(), sizeof(pairk::PairLaunch) * n, cudaMemcpyHostToDevice, s) !=
        cudaSuccess)
      return CCE_ERR_CUDA;
    if (cudaFuncSetAttribute(pairk::cce_pair_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             pairk::PSMEM) != cudaSuccess)
      return CCE_ERR_CUDA;
    const int ppr = (h->num_sms / 2) / n;  // CTA pairs per rank
    ProfScope ps(h, s, 1);
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(2 * ppr * n);
    lc.blockDim = dim3(pairk::PTHREADS);
    lc.dynamicSmemBytes = pairk::PSMEM;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    const pairk::PairLaunch* dev = h->grp_launch_dev;
    if (cudaLaunchKernelEx(&lc, pairk::cce_pair_group_kernel, dev, ppr) != cudaSuccess) {
      (void)cudaGetLastError();  // cooperative + cluster launch refused: a plain launch of the same grid
      lc.numAttrs = 0;
      if (cudaLaunchKernelEx(&lc, pairk::cce_pair_group_kernel, dev, ppr) != cudaSuccess) return CCE_ERR_CUDA;
    }
  }
  for (int q = 0; q < n; ++q) {
    cce_handle* g = h->group[q];
    g->grp_bwd_pending = false;
    g->grp_has_launch = false;
    const cce_status st = backward_tail(g, g->grp_dH, g->grp_dgamma, g->grp_norm, s);
    if (st != CCE_OK) return st;
  }
  return CCE_OK;
}

cce_status cce_backward_finish(cce_handle* h, void* stream) {
  if (!h) return CCE_ERR_INVALID_VALUE;
  if (!h->bwd_pending) return CCE_ERR_NO_FORWARD;
  h->bwd_pending = false;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Layout L = layout(h->N, h->D, h->V_local, h->cfg.world, h->chunk, h->slots, h->cfg.flags);
  if (h->cfg.flags & CCE_FLAG_DH_SEQ_SHARD) return seq_rows_out(h, L, h->p_dH, s);
  ProfScope ps(h, s, 4);
  k_scatter_dH<<<grid_for((long long)h->N * h->D / 8, 256, 8 * h->num_sms), 256, 0, s>>>(
      at<float>(h->ws, L.dH32), at<int>(h->ws, L.pos), (int)h->N, (int)h->D, h->p_dH,
      (h->cfg.flags & CCE_FLAG_GRAD_FP32) ? 1 : 0, (h->cfg.flags & CCE_FLAG_ACCUMULATE) ? 1 : 0);
  return cudaGetLastError() == cudaSuccess ? CCE_OK : CCE_ERR_CUDA;
}

typedef CUresult (*PFN_addrRange)(CUdeviceptr*, size_t*, CUdeviceptr);

cce_status cce_p2p_export(const void* dev_ptr, void* handle_out, int64_t* offset_out) {
  if (!dev_ptr || !handle_out || !offset_out) return CCE_ERR_INVALID_VALUE;
  static PFN_addrRange range = nullptr;
  if (!range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return CCE_ERR_CUDA;
    range = reinterpret_cast<PFN_addrRange>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS) return CCE_ERR_CUDA;
  cudaIpcMemHandle_t mh;
  if (cudaIpcGetMemHandle(&mh, reinterpret_cast<void*>(base)) != cudaSuccess) return CCE_ERR_CUDA;
  std::memcpy(handle_out, &mh, sizeof(mh));
  *offset_out = (int64_t)(reinterpret_cast<uintptr_t>(dev_ptr) - (uintptr_t)base);
  return CCE_OK;
}

cce_status cce_p2p_attach(cce_handle* h, void* workspace, int64_t N, int64_t D, const void* handles,
                          const int64_t* offsets) {
  if (!h || !workspace || !handles || !offsets || N < 0 || D <= 0) return CCE_ERR_INVALID_VALUE;
  if (!(h->cfg.flags & CCE_FLAG_P2P_COMBINE) || h->p2p_attached) return CCE_ERR_INVALID_VALUE;
  if (!aligned16(workspace)) return CCE_ERR_UNSUPPORTED;
  const int world = h->cfg.world, rank = h->cfg.rank;
  for (int r = 0; r < world; ++r) {
    if (r == rank) {
      h->peers.ws[r] = static_cast<char*>(workspace);
      continue;
    }
    cudaIpcMemHandle_t mh;
    std::memcpy(&mh, static_cast<const char*>(handles) + (size_t)r * CCE_P2P_HANDLE_BYTES, sizeof(mh));
    void* base = nullptr;
    if (cudaIpcOpenMemHandle(&base, mh, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return CCE_ERR_CUDA;
    h->opened[r] = base;
    h->peers.ws[r] = static_cast<char*>(base) + offsets[r];
  }
  // this rank's flags start at 0 (every rank attaches before any rank's first step)
  const Layout L = layout(N, D, 0, world, h->chunk, h->slots, h->cfg.flags);
  if (cudaMemset(workspace, 0, L.stats_all) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
    return CCE_ERR_CUDA;
  h->p2p_N = N;
  h->p2p_D = D;
  h->p2p_ws = workspace;
  h->p2p_attached = true;
  h->epoch = 0;
  return CCE_OK;
}

cce_status cce_p2p_attach_group(cce_handle* const* hs, void* const* workspaces, int32_t world, int64_t N, int64_t D) {
  if (!hs || !workspaces || world < 2 || world > P2P_MAX || N < 0 || D <= 0) return CCE_ERR_INVALID_VALUE;
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) return CCE_ERR_CUDA;
  for (int r = 0; r < world; ++r) {
    const cce_handle* h = hs[r];
    if (!h || !workspaces[r] || !(h->cfg.flags & CCE_FLAG_P2P_COMBINE) || h->p2p_attached || h->cfg.world != world ||
        h->cfg.rank != r || h->device != dev)
      return CCE_ERR_INVALID_VALUE;
    if (!aligned16(workspaces[r])) return CCE_ERR_UNSUPPORTED;
    for (int q = 0; q < r; ++q)
      if (hs[q] == h) return CCE_ERR_INVALID_VALUE;
  }
  cce_handle* last = hs[world - 1];
  if (cudaMalloc(&last->grp_launch_dev, sizeof(pairk::PairLaunch) * world) != cudaSuccess) return CCE_ERR_CUDA;
  const Layout L = layout(N, D, 0, world, last->chunk, last->slots, last->cfg.flags);
  for (int r = 0; r < world; ++r) {
    cce_handle* h = hs[r];
    for (int q = 0; q < world; ++q) {
      h->peers.ws[q] = static_cast<char*>(workspaces[q]);
      h->group[q] = hs[q];
    }
    h->group_n = world;
    if (cudaMemset(workspaces[r], 0, L.stats_all) != cudaSuccess) return CCE_ERR_CUDA;  // flags start at 0
    h->p2p_N = N;
    h->p2p_D = D;
    h->p2p_ws = workspaces[r];
    h->p2p_attached = true;
    h->epoch = 0;
  }
  return cudaDeviceSynchronize() == cudaSuccess ? CCE_OK : CCE_ERR_CUDA;
}

cce_status cce_get_error(cce_handle* h, void* stream) {
  if (!h) return CCE_ERR_INVALID_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!h->ws) return CCE_OK;
  const Layout L = layout(h->N, h->D, h->V_local, h->cfg.world, h->chunk, h->slots, h->cfg.flags);
  int* errp = at<int>(h->ws, L.scal) + 1;
  int err = 0;
  if (cudaMemcpyAsync(&err, errp, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess) return CCE_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return CCE_ERR_CUDA;
  if (err) {
    if (cudaMemsetAsync(errp, 0, 4, s) != cudaSuccess) return CCE_ERR_CUDA;
    return (err & 4) ? CCE_ERR_NCCL : CCE_ERR_LABEL_RANGE;  // bit 2: a peer never signalled (P2P)
  }
  return CCE_OK;
}

size_t cce_host_staging_bytes(int64_t N, int64_t D) {
  if (N < 0 || D <= 0) return 0;
  return align_up((size_t)N * D * 2, 256) + align_up((size_t)(N > 0 ? N : 1) * 4, 256) + 256;
}

static cce_status step_host_impl(cce_handle* h, const void* H_host, int64_t N, int64_t D, const int32_t* labels_host,
                                 const void* W, int64_t V_local, int64_t ldw, float* loss_host, void* dH, void* dW,
                                 void* dev_inputs, size_t dev_inputs_bytes, void* workspace, size_t workspace_bytes,
                                 void* stream, void* copy_stream, bool sync) {
  if (!h || !loss_host || (N > 0 && (!H_host || !labels_host))) return CCE_ERR_INVALID_VALUE;
  if (N < 0 || D <= 0) return CCE_ERR_INVALID_VALUE;
  if (h->cfg.flags & CCE_FLAG_EXTERNAL_COMBINE) return CCE_ERR_UNSUPPORTED;
  if (!dev_inputs || dev_inputs_bytes < cce_host_staging_bytes(N, D) || !aligned16(dev_inputs))
    return CCE_ERR_WORKSPACE;
  if (h->cfg.reduction == CCE_REDUCTION_NONE) return CCE_ERR_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaStream_t cs = copy_stream ? static_cast<cudaStream_t>(copy_stream) : s;
  char* base = static_cast<char*>(dev_inputs);
  void* Hd = base;
  int32_t* yd = reinterpret_cast<int32_t*>(base + align_up((size_t)N * D * 2, 256));
  float* scal = reinterpret_cast<float*>(base + align_up((size_t)N * D * 2, 256) + align_up((size_t)(N > 0 ? N : 1) * 4, 256));
  float* loss_d = scal;
  float* dloss_d = scal + 1;
  cce_handle::Stage* stg = nullptr;
  if (cs != s) {
    // the staging buffer's previous step must be done with it before the copy overwrites it
    for (auto& e : h->stages)
      if (e.buf == dev_inputs) { stg = &e; break; }
    if (!stg) {
      for (auto& e : h->stages)
        if (!e.buf) { stg = &e; break; }
      if (!stg) return CCE_ERR_INVALID_VALUE;  // more than four staging buffers in rotation
      stg->buf = dev_inputs;
      if (cudaEventCreateWithFlags(&stg->consumed, cudaEventDisableTiming) != cudaSuccess) return CCE_ERR_CUDA;
      if (cudaEventRecord(stg->consumed, s) != cudaSuccess) return CCE_ERR_CUDA;
    }
    if (!h->ev_copied && cudaEventCreateWithFlags(&h->ev_copied, cudaEventDisableTiming) != cudaSuccess)
      return CCE_ERR_CUDA;
    if (cudaStreamWaitEvent(cs, stg->consumed, 0) != cudaSuccess) return CCE_ERR_CUDA;
  }
  if (N > 0) {
    if (cudaMemcpyAsync(Hd, H_host, (size_t)N * D * 2, cudaMemcpyHostToDevice, cs) != cudaSuccess) return CCE_ERR_CUDA;
    if (cudaMemcpyAsync(yd, labels_host, (size_t)N * 4, cudaMemcpyHostToDevice, cs) != cudaSuccess) return CCE_ERR_CUDA;
  }
  if (cs != s) {
    if (cudaEventRecord(h->ev_copied, cs) != cudaSuccess || cudaStreamWaitEvent(s, h->ev_copied, 0) != cudaSuccess)
      return CCE_ERR_CUDA;
  }
  cce_status st = cce_forward(h, N > 0 ? Hd : nullptr, N, D, D, W, V_local, ldw, N > 0 ? yd : nullptr, loss_d, nullptr,
                              nullptr, workspace, workspace_bytes, stream);
  if (st != CCE_OK) return st;
  {
    ProfScope ps(h, s, 4);
    k_set_scalar<<<1, 1, 0, s>>>(dloss_d, 1.0f);
  }
  st = cce_backward(h, dloss_d, dH, dW, stream);
  if (st != CCE_OK) return st;
  if (cudaMemcpyAsync(loss_host, loss_d, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess) return CCE_ERR_CUDA;
  if (stg && cudaEventRecord(stg->consumed, s) != cudaSuccess) return CCE_ERR_CUDA;
  if (sync && cudaStreamSynchronize(s) != cudaSuccess) return CCE_ERR_CUDA;
  return CCE_OK;
}

cce_status cce_step_host(cce_handle* h, const void* H_host, int64_t N, int64_t D, const int32_t* labels_host,
                         const void* W, int64_t V_local, int64_t ldw, float* loss_host, void* dH, void* dW,
                         void* dev_inputs, size_t dev_inputs_bytes, void* workspace, size_t workspace_bytes,
                         void* stream) {
  return step_host_impl(h, H_host, N, D, labels_host, W, V_local, ldw, loss_host, dH, dW, dev_inputs, dev_inputs_bytes,
                        workspace, workspace_bytes, stream, nullptr, true);
}

cce_status cce_step_host_async(cce_handle* h, const void* H_host, int64_t N, int64_t D, const int32_t* labels_host,
                               const void* W, int64_t V_local, int64_t ldw, float* loss_host, void* dH, void* dW,
                               void* dev_inputs, size_t dev_inputs_bytes, void* workspace, size_t workspace_bytes,
                               void* stream, void* copy_stream) {
  return step_host_impl(h, H_host, N, D, labels_host, W, V_local, ldw, loss_host, dH, dW, dev_inputs, dev_inputs_bytes,
                        workspace, workspace_bytes, stream, copy_stream, false);
}

cce_status cce_nccl_unique_id(void* id_out) {
  if (!id_out) return CCE_ERR_INVALID_VALUE;
  Nccl& n = nccl();
  if (!n.ok) return CCE_ERR_NCCL;
  return n.get_id(static_cast<NcclId*>(id_out)) == 0 ? CCE_OK : CCE_ERR_NCCL;
}

cce_status cce_nccl_comm_init(void** comm_out, int32_t world, const void* id, int32_t rank) {
  if (!comm_out || !id || world < 1 || rank < 0 || rank >= world) return CCE_ERR_INVALID_VALUE;
  Nccl& n = nccl();
  if (!n.ok) return CCE_ERR_NCCL;
  NcclId uid;
  std::memcpy(&uid, id, sizeof(uid));
  return n.init(comm_out, world, uid, rank) == 0 ? CCE_OK : CCE_ERR_NCCL;
}

cce_status cce_nccl_comm_destroy(void* comm) {
  if (!comm) return CCE_ERR_INVALID_VALUE;
  Nccl& n = nccl();
  if (!n.ok) return CCE_ERR_NCCL;
  return n.destroy(comm) == 0 ? CCE_OK : CCE_ERR_NCCL;
}

}  // extern "C"
