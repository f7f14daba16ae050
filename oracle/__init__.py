"""CPU oracle for the fused linear cross-entropy hot path (arxiv 2601.02609).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2601_02609_b200``) never imports it and
shares no code with it.

The arithmetic lives in ``oracle/cce_oracle.c`` (plain C, fp64, OpenMP); this
module only marshals numpy arrays into it.  See that file's header for the
definitions and their citations (PAPER.md lines).  Parity status: every
function here is pinned by ``tests/test_oracle_pins.py`` (closed forms,
finite differences, a library routine, paper/SPEC worked examples).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cce_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK = 0
ERR_LABEL_RANGE = 1


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, IEEE semantics, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
               "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", _LIB, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        p = ctypes.c_void_p
        i64 = ctypes.c_int64
        i32 = ctypes.c_int32
        f64 = ctypes.c_double
        L.oracle_cce.argtypes = [p, p, p, i64, i64, i64, i32, f64, p, p, p, p, p]
        L.oracle_cce.restype = ctypes.c_int
        L.oracle_dlogits.argtypes = [p, p, p, i64, i64, i64, i32, f64, p]
        L.oracle_dlogits.restype = ctypes.c_int
        L.oracle_cce_reg.argtypes = [p, p, p, i64, i64, i64, i32, f64, f64, f64, p, p, p, p, p]
        L.oracle_cce_full.argtypes = [p, p, p, i64, i64, i64, i32, f64, f64, ctypes.c_int, f64, p, p, p, p, p, p]
        L.oracle_cce_full.restype = ctypes.c_int
        L.oracle_cce_reg.restype = ctypes.c_int
        L.oracle_dlogits_reg.argtypes = [p, p, p, i64, i64, i64, i32, f64, f64, f64, p]
        L.oracle_dlogits_reg.restype = ctypes.c_int
        L.oracle_cce_rows.argtypes = [p, p, p, i64, i64, f64, p, i64, p, p, p]
        L.oracle_cce_rows.restype = ctypes.c_int
        L.oracle_dW_rows.argtypes = [p, p, p, i64, i64, i32, p, f64, p, i64, p]
        L.oracle_dW_rows.restype = ctypes.c_int
        L.oracle_online_lse.argtypes = [p, i64]
        L.oracle_online_lse.restype = f64
        L.oracle_partial_stats.argtypes = [p, p, p, i64, i64, i64, i64, i32, p, p, p]
        L.oracle_partial_stats.restype = ctypes.c_int
        L.oracle_adamw_step.argtypes = [p, p, p, p, i64, f64, f64, f64, f64, f64, f64, f64, f64]
        L.oracle_adamw_step.restype = None
        L.oracle_rmsnorm_fwd.argtypes = [p, p, i64, i64, f64, p, p]
        L.oracle_rmsnorm_fwd.restype = None
        L.oracle_rmsnorm_bwd.argtypes = [p, p, p, p, p, i64, i64, p, p]
        L.oracle_rmsnorm_bwd.restype = None
        L.oracle_to_bf16.argtypes = [p, i64, p]
        L.oracle_to_bf16.restype = None
        L.oracle_validate.argtypes = [p, i64, i64, i32, p]
        L.oracle_validate.restype = ctypes.c_int
        L.oracle_num_threads.argtypes = []
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _bits(a) -> np.ndarray:
    """bf16 bit patterns (uint16) -> fp64, exactly; fp64 arrays pass through."""
    a = np.ascontiguousarray(a)
    if a.dtype == np.float64:
        return a
    if a.dtype != np.uint16:
        raise TypeError("inputs are bf16 bit patterns (uint16) or fp64 arrays")
    return np.ascontiguousarray((a.astype(np.uint32) << 16).view(np.float32).astype(np.float64))


def _check(rc: int):
    if rc == ERR_LABEL_RANGE:
        raise OracleError("label out of range")
    if rc != OK:
        raise OracleError(f"oracle error {rc}")


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def cce(H_bits, W_bits, labels, ignore_index=-100, dloss=1.0, grads=True, label_smoothing=0.0, z_loss=0.0,
        reduction="mean"):
    """Full forward+backward.  Returns dict(loss, lse[N], n_valid, dH[N,D], dW[V,D]) in fp64.
    label_smoothing (eps) and z_loss (lambda) follow oracle_cce_reg.
    reduction "mean" | "sum" | "none"; with "none" loss is the [N] per-row array and
    dloss an [N] array of upstream gradients."""
    H = _bits(H_bits); W = _bits(W_bits)
    y = np.ascontiguousarray(labels, dtype=np.int32)
    N, D = H.shape
    V = W.shape[0]
    assert W.shape[1] == D and y.shape == (N,)
    red = {"mean": 0, "sum": 1, "none": 2}[reduction]
    loss = np.zeros(N if red == 2 else 1, np.float64)
    lse = np.zeros(N, np.float64)
    nv = np.zeros(1, np.int64)
    dH = np.zeros((N, D), np.float64) if grads else None
    dW = np.zeros((V, D), np.float64) if grads else None
    if red == 2:
        drows = np.ascontiguousarray(np.broadcast_to(np.asarray(dloss, np.float64), (N,)))
        dscal = 0.0
    else:
        drows, dscal = None, float(dloss)
    _check(lib().oracle_cce_full(_ptr(H), _ptr(W), _ptr(y), N, D, V, ignore_index, float(label_smoothing),
                                 float(z_loss), red, dscal, _ptr(drows), _ptr(loss), _ptr(lse), _ptr(nv), _ptr(dH),
                                 _ptr(dW)))
    return {"loss": loss if red == 2 else float(loss[0]), "lse": lse, "n_valid": int(nv[0]), "dH": dH, "dW": dW}


def dlogits(H_bits, W_bits, labels, ignore_index=-100, dloss=1.0, label_smoothing=0.0, z_loss=0.0):
    H = _bits(H_bits); W = _bits(W_bits)
    y = np.ascontiguousarray(labels, dtype=np.int32)
    N, D = H.shape
    V = W.shape[0]
    G = np.zeros((N, V), np.float64)
    _check(lib().oracle_dlogits_reg(_ptr(H), _ptr(W), _ptr(y), N, D, V, ignore_index, float(label_smoothing),
                                    float(z_loss), float(dloss), _ptr(G)))
    return G


def rows(H_bits, W_bits, labels, row_idx, scale=None):
    """lse, z_y (and dH rows if ``scale`` is given) for the listed valid rows."""
    H = _bits(H_bits); W = _bits(W_bits)
    y = np.ascontiguousarray(labels, dtype=np.int32)
    r = np.ascontiguousarray(row_idx, dtype=np.int64)
    D = H.shape[1]
    V = W.shape[0]
    lse = np.zeros(len(r), np.float64)
    zy = np.zeros(len(r), np.float64)
    dH = np.zeros((len(r), D), np.float64) if scale is not None else None
    _check(lib().oracle_cce_rows(_ptr(H), _ptr(W), _ptr(y), D, V,
                                 float(scale) if scale is not None else 0.0,
                                 _ptr(r), len(r), _ptr(lse), _ptr(zy), _ptr(dH)))
    return lse, zy, dH


def dW_rows(H_bits, W_bits, labels, lse, scale, vrows, ignore_index=-100):
    H = _bits(H_bits); W = _bits(W_bits)
    y = np.ascontiguousarray(labels, dtype=np.int32)
    lse = np.ascontiguousarray(lse, dtype=np.float64)
    vr = np.ascontiguousarray(vrows, dtype=np.int64)
    N, D = H.shape
    out = np.zeros((len(vr), D), np.float64)
    _check(lib().oracle_dW_rows(_ptr(H), _ptr(W), _ptr(y), N, D, ignore_index, _ptr(lse),
                                float(scale), _ptr(vr), len(vr), _ptr(out)))
    return out


def online_lse(x) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(lib().oracle_online_lse(_ptr(x), len(x)))


def partial_stats(H_bits, W_local_bits, labels, vocab_offset, ignore_index=-100):
    H = _bits(H_bits); W = _bits(W_local_bits)
    y = np.ascontiguousarray(labels, dtype=np.int32)
    N, D = H.shape
    Vl = W.shape[0]
    m = np.zeros(N); d = np.zeros(N); zy = np.zeros(N)
    _check(lib().oracle_partial_stats(_ptr(H), _ptr(W) if Vl > 0 else None, _ptr(y), N, D, Vl,
                                      int(vocab_offset), ignore_index, _ptr(m), _ptr(d), _ptr(zy)))
    return m, d, zy


def validate(labels, V, ignore_index=-100) -> int:
    y = np.ascontiguousarray(labels, dtype=np.int32)
    nv = np.zeros(1, np.int64)
    _check(lib().oracle_validate(_ptr(y), len(y), int(V), ignore_index, _ptr(nv)))
    return int(nv[0])


def adamw_step(theta, grad, m, v, lr, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, clip_coef=1.0, step=1):
    """One AdamW step (oracle_adamw_step) on copies; returns (theta, m, v) in fp64.
    Bias corrections 1 - beta^step are computed here (host side)."""
    th = np.ascontiguousarray(theta, dtype=np.float64).copy()
    g = np.ascontiguousarray(grad, dtype=np.float64)
    mm = np.ascontiguousarray(m, dtype=np.float64).copy()
    vv = np.ascontiguousarray(v, dtype=np.float64).copy()
    assert th.shape == g.shape == mm.shape == vv.shape
    bc1 = 1.0 - beta1 ** step
    bc2 = 1.0 - beta2 ** step
    lib().oracle_adamw_step(_ptr(th), _ptr(g), _ptr(mm), _ptr(vv), th.size, float(lr), float(beta1), float(beta2),
                            float(eps), float(weight_decay), float(clip_coef), bc1, bc2)
    return th, mm, vv


# ----------------------------------------------------------------- RMSNorm prologue (NEXT #4)
def rmsnorm_fwd(x, gamma, eps=1e-6):
    """Def. RMSNorm: returns (y [N,D], rstd [N]) in fp64 (oracle_rmsnorm_fwd)."""
    X = _bits(x)
    if X.ndim == 1:
        X = X[None, :]
    g = _bits(gamma)
    N, D = X.shape
    assert g.shape == (D,)
    y = np.zeros((N, D), np.float64)
    r = np.zeros(N, np.float64)
    lib().oracle_rmsnorm_fwd(_ptr(X), _ptr(g), N, D, float(eps), _ptr(y), _ptr(r))
    return y, r


def rmsnorm_bwd(dy, x, gamma, rstd, skip=None):
    """Exact gradient of Def. RMSNorm (oracle_rmsnorm_bwd; reading R18): (dx, dgamma) fp64."""
    X = _bits(x)
    g = _bits(gamma)
    dY = np.ascontiguousarray(dy, dtype=np.float64)
    N, D = X.shape
    r = np.ascontiguousarray(rstd, dtype=np.float64)
    sk = None if skip is None else np.ascontiguousarray(skip, dtype=np.int32)
    dx = np.zeros((N, D), np.float64)
    dg = np.zeros(D, np.float64)
    lib().oracle_rmsnorm_bwd(_ptr(dY), _ptr(X), _ptr(g), _ptr(r), _ptr(sk), N, D, _ptr(dx), _ptr(dg))
    return dx, dg


def to_bf16(a):
    """fp64 -> bf16 bit patterns (uint16), round to nearest even via fp32."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = np.zeros(a.shape, np.uint16)
    lib().oracle_to_bf16(_ptr(a), a.size, _ptr(out))
    return out


def cce_rmsnorm(X_bits, gamma_bits, W_bits, labels, eps=1e-6, ignore_index=-100, dloss=1.0, **cce_kwargs):
    """The path with the RMSNorm prologue: H = bf16(RMSNorm(X)) (the CE path consumes bf16
    H), the CE oracle on H (cce_kwargs: label_smoothing, z_loss, reduction), then
    the RMSNorm backward of its dH.  Returns oracle.cce's dict plus dX [N,D], dgamma [D],
    rstd [N] and H_bits."""
    y, rstd = rmsnorm_fwd(X_bits, gamma_bits, eps)
    H_bits = to_bf16(y)
    out = cce(H_bits, W_bits, labels, ignore_index=ignore_index, dloss=dloss, **cce_kwargs)
    skip = (np.asarray(labels) == ignore_index).astype(np.int32)
    dx, dg = rmsnorm_bwd(out["dH"], X_bits, gamma_bits, rstd, skip)
    out.update(dX=dx, dgamma=dg, rstd=rstd, H_bits=H_bits)
    return out
