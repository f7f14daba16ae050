"""B200-native fused linear cross-entropy (Cut Cross-Entropy, arxiv 2601.02609).

Thin Python binding over the C ABI in ``include/cce.h`` (``libcce.so``).  This
module only marshals arguments: every step of the forward and backward runs in
the library's sm_100a kernels.  PyTorch is used for device memory, streams and
process groups only.  There is no CPU fallback: if the extension is missing or
no sm_100 device is present, calls raise.

Public API
  cce_create / cce_destroy / cce_workspace_bytes / cce_forward / cce_backward /
  cce_get_error / cce_step_host / cce_nccl_*      -- same names as the C ABI
  CCEHandle                                        -- owns a handle + workspace
  linear_cross_entropy(H, W, labels, ...)          -- autograd entry point
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libcce.so")

CCE_OK = 0
STATUS = {0: "CCE_OK", 1: "CCE_ERR_INVALID_VALUE", 2: "CCE_ERR_UNSUPPORTED", 3: "CCE_ERR_LABEL_RANGE",
          4: "CCE_ERR_NO_FORWARD", 5: "CCE_ERR_WORKSPACE", 6: "CCE_ERR_CUDA", 7: "CCE_ERR_NCCL"}

# every symbol include/cce.h declares
EXPORTS = ["cce_config_default", "cce_create", "cce_destroy", "cce_workspace_bytes", "cce_forward", "cce_backward",
           "cce_get_error", "cce_host_staging_bytes", "cce_step_host", "cce_nccl_unique_id", "cce_nccl_comm_init",
           "cce_nccl_comm_destroy", "cce_status_string", "cce_kernel_launches", "cce_build_info",
           "cce_profile_enable", "cce_profile_read", "cce_debug_trace", "cce_backward_adamw", "cce_adamw_step",
           "cce_forward_rmsnorm", "cce_backward_rmsnorm", "cce_combine_offsets", "cce_forward_finish",
           "cce_backward_finish", "cce_step_host_async", "cce_p2p_export", "cce_p2p_attach",
           "cce_p2p_attach_group"]
PROF_CLASSES = ("fwd_logits_lse", "bwd", "bwd_dW", "bwd_dH", "aux")
# "bwd" is the persistent backward kernel (recompute + dlogits + dW + dH)
FLAG_GRAD_FP32 = 64
FLAG_ACCUMULATE = 128
FLAG_EXTERNAL_COMBINE = 256
FLAG_DH_SEQ_SHARD = 512
FLAG_P2P_COMBINE = 1024
FLAG_DESIGN_B = 2048
REDUCTION_MEAN, REDUCTION_SUM, REDUCTION_NONE = 0, 1, 2
_REDUCTIONS = {"mean": REDUCTION_MEAN, "sum": REDUCTION_SUM, "none": REDUCTION_NONE}


class CCEError(RuntimeError):
    def __init__(self, status: int, where: str = ""):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)}")


class cce_config(ctypes.Structure):
    _fields_ = [("ignore_index", ctypes.c_int32), ("vocab_total", ctypes.c_int64), ("vocab_offset", ctypes.c_int64),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("nccl_comm", ctypes.c_void_p),
                ("flags", ctypes.c_uint32), ("label_smoothing", ctypes.c_float), ("z_loss", ctypes.c_float),
                ("reduction", ctypes.c_int32)]


class cce_adamw_params(ctypes.Structure):
    """Mirror of cce.h cce_adamw_params (fused AdamW, Alg. Fused AdamW P:2003-2046)."""
    _fields_ = [("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float), ("eps", ctypes.c_float),
                ("weight_decay", ctypes.c_float), ("bias_correction1", ctypes.c_float),
                ("bias_correction2", ctypes.c_float), ("clip_coef", ctypes.c_void_p), ("master", ctypes.c_void_p),
                ("m", ctypes.c_void_p), ("v", ctypes.c_void_p), ("grad_in", ctypes.c_void_p),
                ("W_out", ctypes.c_void_p)]


_lib = None


def lib():
    """Load libcce.so (build it first with paper_2601_02609_b200.build.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        p, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
        st = ctypes.c_int
        L.cce_config_default.argtypes = [ctypes.POINTER(cce_config)]
        L.cce_config_default.restype = None
        L.cce_create.argtypes = [ctypes.POINTER(p), ctypes.POINTER(cce_config)]
        L.cce_create.restype = st
        L.cce_destroy.argtypes = [p]
        L.cce_destroy.restype = st
        L.cce_workspace_bytes.argtypes = [p, i64, i64, i64]
        L.cce_workspace_bytes.restype = sz
        L.cce_forward.argtypes = [p, p, i64, i64, i64, p, i64, i64, p, p, p, p, p, sz, p]
        L.cce_forward.restype = st
        L.cce_backward.argtypes = [p, p, p, p, p]
        L.cce_backward.restype = st
        L.cce_combine_offsets.argtypes = [p, i64, i64, i64, p]
        L.cce_combine_offsets.restype = st
        L.cce_forward_finish.argtypes = [p, p]
        L.cce_forward_finish.restype = st
        L.cce_backward_finish.argtypes = [p, p]
        L.cce_backward_finish.restype = st
        L.cce_forward_rmsnorm.argtypes = [p, p, i64, i64, i64, p, ctypes.c_float, p, i64, i64, p, p, p, p, p, sz, p]
        L.cce_forward_rmsnorm.restype = st
        L.cce_backward_rmsnorm.argtypes = [p, p, p, p, p, p]
        L.cce_backward_rmsnorm.restype = st
        L.cce_backward_adamw.argtypes = [p, p, p, ctypes.POINTER(cce_adamw_params), p]
        L.cce_backward_adamw.restype = st
        L.cce_adamw_step.argtypes = [ctypes.POINTER(cce_adamw_params), p, i32, i64, p, p]
        L.cce_adamw_step.restype = st
        L.cce_get_error.argtypes = [p, p]
        L.cce_get_error.restype = st
        L.cce_host_staging_bytes.argtypes = [i64, i64]
        L.cce_host_staging_bytes.restype = sz
        L.cce_step_host.argtypes = [p, p, i64, i64, p, p, i64, i64, p, p, p, p, sz, p, sz, p]
        L.cce_step_host.restype = st
        L.cce_p2p_export.argtypes = [p, p, p]
        L.cce_p2p_export.restype = st
        L.cce_p2p_attach.argtypes = [p, p, i64, i64, p, p]
        L.cce_p2p_attach.restype = st
        if hasattr(L, "cce_p2p_attach_group"):  # (older builds, loaded by scripts/ab.py, lack it)
            L.cce_p2p_attach_group.argtypes = [p, p, i32, i64, i64]
            L.cce_p2p_attach_group.restype = st
        L.cce_step_host_async.argtypes = [p, p, i64, i64, p, p, i64, i64, p, p, p, p, sz, p, sz, p, p]
        L.cce_step_host_async.restype = st
        L.cce_nccl_unique_id.argtypes = [p]
        L.cce_nccl_unique_id.restype = st
        L.cce_nccl_comm_init.argtypes = [ctypes.POINTER(p), i32, p, i32]
        L.cce_nccl_comm_init.restype = st
        L.cce_nccl_comm_destroy.argtypes = [p]
        L.cce_nccl_comm_destroy.restype = st
        L.cce_status_string.argtypes = [st]
        L.cce_status_string.restype = ctypes.c_char_p
        L.cce_kernel_launches.argtypes = [p]
        L.cce_kernel_launches.restype = i64
        L.cce_profile_enable.argtypes = [p, i32]
        L.cce_profile_enable.restype = st
        L.cce_profile_read.argtypes = [p, p, p, i32]
        L.cce_profile_read.restype = st
        L.cce_debug_trace.argtypes = [p, p, sz]
        L.cce_debug_trace.restype = st
        L.cce_build_info.argtypes = []
        L.cce_build_info.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(status: int, where: str):
    if status != CCE_OK:
        raise CCEError(status, where)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


# ----------------------------------------------------------------- C-ABI mirrors
def cce_create(vocab_total: int, ignore_index: int = -100, vocab_offset: int = 0, rank: int = 0, world: int = 1,
               nccl_comm=None, flags: int = 0, label_smoothing: float = 0.0, z_loss: float = 0.0,
               reduction: int = REDUCTION_MEAN) -> ctypes.c_void_p:
    cfg = cce_config()
    lib().cce_config_default(ctypes.byref(cfg))
    cfg.ignore_index = ignore_index
    cfg.vocab_total = vocab_total
    cfg.vocab_offset = vocab_offset
    cfg.rank = rank
    cfg.world = world
    cfg.nccl_comm = nccl_comm
    cfg.flags = flags
    cfg.label_smoothing = label_smoothing
    cfg.z_loss = z_loss
    cfg.reduction = _REDUCTIONS.get(reduction, reduction) if isinstance(reduction, str) else reduction
    h = ctypes.c_void_p()
    _check(lib().cce_create(ctypes.byref(h), ctypes.byref(cfg)), "cce_create")
    return h


def cce_destroy(h):
    _check(lib().cce_destroy(h), "cce_destroy")


def cce_workspace_bytes(h, N: int, D: int, V_local: int) -> int:
    return int(lib().cce_workspace_bytes(h, N, D, V_local))


def _check_layout(where, *rows_major, vec=()):
    """The C ABI takes a row stride only: rows must be dense (stride(1) == 1) and the
    1-D arrays contiguous, else the kernels would read the wrong elements."""
    for t in rows_major:
        if t is not None and t.dim() == 2 and t.shape[1] > 1 and t.stride(1) != 1:
            raise ValueError(f"{where}: 2-D inputs need unit column stride (got strides {tuple(t.stride())})")
    for t in vec:
        if t is not None and not t.is_contiguous():
            raise ValueError(f"{where}: 1-D inputs must be contiguous")


def cce_forward(h, H, W, labels, loss, lse, n_valid, workspace, stream=None):
    _check_layout("cce_forward", H, W, vec=(labels, lse))
    N, D = H.shape
    V_local = W.shape[0]
    _check(lib().cce_forward(h, _ptr(H), N, D, H.stride(0), _ptr(W), V_local, W.stride(0), _ptr(labels), _ptr(loss),
                             _ptr(lse), _ptr(n_valid), _ptr(workspace), workspace.numel() * workspace.element_size(),
                             _stream(stream)), "cce_forward")


def cce_forward_rmsnorm(h, X, gamma, eps, W, labels, loss, lse, n_valid, workspace, stream=None):
    _check_layout("cce_forward_rmsnorm", X, W, vec=(gamma, labels, lse))
    N, D = X.shape
    V_local = W.shape[0]
    _check(lib().cce_forward_rmsnorm(h, _ptr(X), N, D, X.stride(0), _ptr(gamma), float(eps), _ptr(W), V_local,
                                     W.stride(0), _ptr(labels), _ptr(loss), _ptr(lse), _ptr(n_valid),
                                     _ptr(workspace), workspace.numel() * workspace.element_size(), _stream(stream)),
           "cce_forward_rmsnorm")


def cce_backward_rmsnorm(h, dloss, dX, dgamma, dW, stream=None):
    _check(lib().cce_backward_rmsnorm(h, _ptr(dloss), _ptr(dX), _ptr(dgamma), _ptr(dW), _stream(stream)),
           "cce_backward_rmsnorm")


def cce_backward(h, dloss, dH, dW, stream=None):
    _check(lib().cce_backward(h, _ptr(dloss), _ptr(dH), _ptr(dW), _stream(stream)), "cce_backward")


def adamw_params(m, v, lr, step, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, clip_coef=None,
                 master=None, grad_in=None, W_out=None) -> cce_adamw_params:
    """Marshal the optimizer state (torch float32 tensors) into cce_adamw_params; the bias
    corrections 1 - beta^t come from the host step counter (no device sync)."""
    o = cce_adamw_params()
    o.lr, o.beta1, o.beta2, o.eps, o.weight_decay = lr, beta1, beta2, eps, weight_decay
    o.bias_correction1 = 1.0 - beta1 ** step
    o.bias_correction2 = 1.0 - beta2 ** step
    o.clip_coef = None if clip_coef is None else clip_coef.data_ptr()
    o.master = None if master is None else master.data_ptr()
    o.m, o.v = m.data_ptr(), v.data_ptr()
    o.grad_in = None if grad_in is None else grad_in.data_ptr()
    o.W_out = None if W_out is None else W_out.data_ptr()
    return o


def cce_backward_adamw(h, dloss, dH, opt: cce_adamw_params, stream=None):
    _check(lib().cce_backward_adamw(h, _ptr(dloss), _ptr(dH), ctypes.byref(opt), _stream(stream)),
           "cce_backward_adamw")


def cce_adamw_step(opt: cce_adamw_params, grad, n: int, W_bf16=None, stream=None):
    import torch
    g32 = 1 if (grad is not None and grad.dtype == torch.float32) else 0
    _check(lib().cce_adamw_step(ctypes.byref(opt), _ptr(grad), g32, n, _ptr(W_bf16), _stream(stream)),
           "cce_adamw_step")


def cce_combine_offsets(h, N: int, D: int, V_local: int):
    """(stats_off, stats_all_off, dH32_off, Npad): byte offsets into the workspace for the
    split-phase combine (FLAG_EXTERNAL_COMBINE)."""
    out = (ctypes.c_int64 * 4)()
    _check(lib().cce_combine_offsets(h, N, D, V_local, out), "cce_combine_offsets")
    return tuple(int(x) for x in out)


def cce_forward_finish(h, stream=None):
    _check(lib().cce_forward_finish(h, _stream(stream)), "cce_forward_finish")


def cce_backward_finish(h, stream=None):
    _check(lib().cce_backward_finish(h, _stream(stream)), "cce_backward_finish")


def cce_get_error(h, stream=None) -> int:
    return int(lib().cce_get_error(h, _stream(stream)))


def cce_host_staging_bytes(N: int, D: int) -> int:
    return int(lib().cce_host_staging_bytes(N, D))


def cce_step_host(h, H_host, labels_host, W, dH, dW, staging, workspace, stream=None) -> float:
    N, D = H_host.shape
    out = ctypes.c_float()
    _check(lib().cce_step_host(h, ctypes.c_void_p(H_host.data_ptr()), N, D, ctypes.c_void_p(labels_host.data_ptr()),
                               _ptr(W), W.shape[0], W.stride(0), ctypes.byref(out), _ptr(dH), _ptr(dW),
                               _ptr(staging), staging.numel() * staging.element_size(), _ptr(workspace),
                               workspace.numel() * workspace.element_size(), _stream(stream)), "cce_step_host")
    return out.value


def cce_step_host_async(h, H_host, labels_host, W, dH, dW, staging, workspace, loss_host, stream=None,
                        copy_stream=None):
    """Enqueue one end-to-end step (host H / labels in, loss out to loss_host, a pinned float32
    tensor element or array) without synchronising; see cce.h."""
    N, D = H_host.shape
    _check(lib().cce_step_host_async(h, ctypes.c_void_p(H_host.data_ptr()), N, D,
                                     ctypes.c_void_p(labels_host.data_ptr()), _ptr(W), W.shape[0], W.stride(0),
                                     ctypes.c_void_p(loss_host.data_ptr()), _ptr(dH), _ptr(dW), _ptr(staging),
                                     staging.numel() * staging.element_size(), _ptr(workspace),
                                     workspace.numel() * workspace.element_size(), _stream(stream),
                                     None if copy_stream is None else ctypes.c_void_p(copy_stream.cuda_stream)),
           "cce_step_host_async")


def cce_p2p_export(t):
    """(64-byte CUDA IPC handle, byte offset) of the allocation holding tensor t."""
    buf = ctypes.create_string_buffer(64)
    off = ctypes.c_int64()
    _check(lib().cce_p2p_export(ctypes.c_void_p(t.data_ptr()), buf, ctypes.byref(off)), "cce_p2p_export")
    return buf.raw, off.value


def cce_p2p_attach(h, workspace, N: int, D: int, handles, offsets):
    """handles / offsets: per rank (lists indexed by rank), from every rank's cce_p2p_export;
    N, D: the problem size of the steps that follow."""
    blob = ctypes.create_string_buffer(b"".join(bytes(x) for x in handles), 64 * len(handles))
    offs = (ctypes.c_int64 * len(offsets))(*offsets)
    _check(lib().cce_p2p_attach(h, _ptr(workspace), N, D, blob, offs), "cce_p2p_attach")


def cce_p2p_attach_group(handles, workspaces, N: int, D: int):
    """One-GPU emulation of the peer-memory exchange (cce.h): handles[r] / workspaces[r] of
    ranks 0 .. world-1 in one process.  Then call every rank's forward in rank order, then every
    rank's backward in rank order, on one stream."""
    world = len(handles)
    hs = (ctypes.c_void_p * world)(*[h.value if isinstance(h, ctypes.c_void_p) else h for h in handles])
    ws = (ctypes.c_void_p * world)(*[w.data_ptr() for w in workspaces])
    _check(lib().cce_p2p_attach_group(hs, ws, world, N, D), "cce_p2p_attach_group")


def cce_kernel_launches(h) -> int:
    return int(lib().cce_kernel_launches(h))


def cce_profile_enable(h, on: bool = True):
    _check(lib().cce_profile_enable(h, 1 if on else 0), "cce_profile_enable")


def cce_profile_read(h, reset: bool = True):
    """{class: (ms, launches)} for the kernels recorded since the last reset (synchronises)."""
    ms = (ctypes.c_double * len(PROF_CLASSES))()
    n = (ctypes.c_int64 * len(PROF_CLASSES))()
    _check(lib().cce_profile_read(h, ms, n, 1 if reset else 0), "cce_profile_read")
    return {c: (ms[i], n[i]) for i, c in enumerate(PROF_CLASSES)}


def cce_debug_trace(h, buf=None):
    """Record the next backward's per-item timeline into `buf` (uint8 CUDA tensor) or disable (None)."""
    _check(lib().cce_debug_trace(h, _ptr(buf), 0 if buf is None else buf.numel() * buf.element_size()),
           "cce_debug_trace")


def cce_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().cce_nccl_unique_id(buf), "cce_nccl_unique_id")
    return buf.raw


def cce_nccl_comm_init(world: int, uid: bytes, rank: int) -> ctypes.c_void_p:
    comm = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    _check(lib().cce_nccl_comm_init(ctypes.byref(comm), world, buf, rank), "cce_nccl_comm_init")
    return comm


def cce_nccl_comm_destroy(comm):
    _check(lib().cce_nccl_comm_destroy(comm), "cce_nccl_comm_destroy")


# ----------------------------------------------------------------- convenience
def shard_range(V: int, rank: int, world: int):
    """Contiguous vocabulary shard [lo, hi) owned by `rank` (sizes differ by at most 1;
    any size is allowed, including empty shards when world > V)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return rank * V // world, (rank + 1) * V // world


class CCEHandle:
    """A library handle plus a cached device workspace (torch-allocated)."""

    def __init__(self, vocab_total: int, ignore_index: int = -100, vocab_offset: int = 0, rank: int = 0,
                 world: int = 1, nccl_comm=None, flags: int = 0, label_smoothing: float = 0.0, z_loss: float = 0.0,
                 reduction="mean"):
        self.h = cce_create(vocab_total, ignore_index, vocab_offset, rank, world, nccl_comm, flags, label_smoothing,
                            z_loss, reduction)
        self.reduction = _REDUCTIONS.get(reduction, reduction) if isinstance(reduction, str) else reduction
        self.vocab_total = vocab_total
        self.ignore_index = ignore_index
        self._ws = None
        # bumped by every forward: the backward computes gradients for the LAST forward on
        # this handle (cce.h: one forward/backward pair in flight), so autograd checks it
        self.generation = 0

    def workspace(self, N, D, V_local, device):
        import torch
        need = cce_workspace_bytes(self.h, N, D, V_local)
        if self._ws is None or self._ws.numel() < need or self._ws.device != device:
            self._ws = torch.empty(need, dtype=torch.uint8, device=device)
        return self._ws

    def forward(self, H, W, labels, want_lse=True, stream=None):
        import torch
        N, D = H.shape
        ws = self.workspace(N, D, W.shape[0], H.device)
        loss = (torch.empty(N, dtype=torch.float32, device=H.device) if self.reduction == REDUCTION_NONE
                else torch.empty((), dtype=torch.float32, device=H.device))
        lse = torch.empty(N, dtype=torch.float32, device=H.device) if want_lse else None
        nv = torch.empty((), dtype=torch.int32, device=H.device)
        self.generation += 1
        cce_forward(self.h, H, W, labels, loss, lse, nv, ws, stream)
        return loss, lse, nv

    def backward(self, dloss, dH, dW, stream=None):
        cce_backward(self.h, dloss, dH, dW, stream)

    def forward_rmsnorm(self, X, gamma, eps, W, labels, want_lse=True, stream=None):
        """The path on H = bf16(RMSNorm(X)) (gamma: [D] bf16); rstd cached for the backward."""
        import torch
        N, D = X.shape
        ws = self.workspace(N, D, W.shape[0], X.device)
        loss = (torch.empty(N, dtype=torch.float32, device=X.device) if self.reduction == REDUCTION_NONE
                else torch.empty((), dtype=torch.float32, device=X.device))
        lse = torch.empty(N, dtype=torch.float32, device=X.device) if want_lse else None
        nv = torch.empty((), dtype=torch.int32, device=X.device)
        self.generation += 1
        cce_forward_rmsnorm(self.h, X, gamma, eps, W, labels, loss, lse, nv, ws, stream)
        return loss, lse, nv

    def backward_rmsnorm(self, dloss, dX, dgamma, dW, stream=None):
        cce_backward_rmsnorm(self.h, dloss, dX, dgamma, dW, stream)

    def backward_adamw(self, dloss, dH, opt: cce_adamw_params, stream=None):
        """Backward with AdamW fused into the dW epilogue: the W given to the last forward
        (and opt's master / m / v) is updated in place; dW is never materialised."""
        cce_backward_adamw(self.h, dloss, dH, opt, stream)

    def launches(self) -> int:
        return cce_kernel_launches(self.h)

    def close(self):
        if self.h is not None:
            cce_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _check_inputs(H, W, labels):
    import torch
    if not (H.is_cuda and W.is_cuda and labels.is_cuda):
        raise ValueError("linear_cross_entropy: tensors must be on a CUDA device (no CPU fallback)")
    if not (H.device == W.device == labels.device):
        raise ValueError("linear_cross_entropy: H, W and labels must be on the same device")
    if H.dtype != torch.bfloat16 or W.dtype != torch.bfloat16 or labels.dtype != torch.int32:
        raise TypeError("linear_cross_entropy: H, W must be bfloat16 and labels int32")
    _check_layout("linear_cross_entropy", H, W, vec=(labels,))


def _make_function():
    import torch

    class CCEFunction(torch.autograd.Function):
        @staticmethod
        def forward(ctx, H, W, labels, handle):
            loss, lse, nv = handle.forward(H, W, labels)
            # the library keeps this forward's state in the handle (like autograd-saved
            # tensors: H, W, labels must stay alive and unmodified until the backward);
            # a later forward on the same handle replaces it, which backward detects
            ctx.handle = handle
            ctx.generation = handle.generation
            ctx.meta = (tuple(H.shape), tuple(W.shape), H.dtype, H.device)
            ctx.keep = (H, W, labels)  # keep-alive only (never read back)
            ctx.mark_non_differentiable(lse, nv)
            return loss, lse, nv

        @staticmethod
        def backward(ctx, dloss, _dlse, _dnv):
            import torch
            if ctx.handle.generation != ctx.generation:
                raise RuntimeError("linear_cross_entropy: the CCEHandle ran another forward before this "
                                   "backward (one forward/backward pair in flight per handle, cce.h); "
                                   "use one handle per loss call")
            hs, ws, dt, dev = ctx.meta
            dH = torch.empty(hs, dtype=dt, device=dev)
            dW = torch.empty(ws, dtype=dt, device=dev)
            if dloss is None:
                shape = (hs[0],) if ctx.handle.reduction == REDUCTION_NONE else ()
                dloss = torch.zeros(shape, dtype=torch.float32, device=dev)
            ctx.handle.backward(dloss.contiguous().float(), dH, dW)
            ctx.keep = None
            return dH, dW, None, None

    return CCEFunction


_CCEFunction = None


def linear_cross_entropy(H, W, labels, ignore_index: int = -100, handle: CCEHandle | None = None,
                         return_lse: bool = False, label_smoothing: float = 0.0, z_loss: float = 0.0,
                         reduction: str = "mean"):
    """Cross-entropy of softmax(H W^T) against labels, fused and never materialising the
    [N, V] logits.  H [N,D] bf16, W [V,D] bf16, labels [N] int32.  reduction: "mean"
    (over non-ignored rows), "sum", or "none" (per-token losses, 0 for ignored rows)."""
    global _CCEFunction
    _check_inputs(H, W, labels)
    if _CCEFunction is None:
        _CCEFunction = _make_function()
    if handle is None:
        handle = CCEHandle(vocab_total=W.shape[0], ignore_index=ignore_index, label_smoothing=label_smoothing,
                           z_loss=z_loss, reduction=reduction)
    loss, lse, nv = _CCEFunction.apply(H, W, labels, handle)
    return (loss, lse) if return_lse else loss
