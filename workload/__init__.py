"""Seeded synthetic inputs shaped like the paper's workloads.

This module is the ONE thing shared by the CUDA path's tests/bench and the
oracle: it draws random numbers and lays them out.  It holds none of the
method's arithmetic (no logits, no softmax, no gradients).

Determinism.  Every value is a pure function of (seed, stream, counter) through
a counter-based splitmix64 hash evaluated with numpy uint64 integer ops, so the
same inputs come out bit-for-bit on any machine (no transcendental functions,
no BLAS, no platform-dependent SIMD reductions on the value path):

* "normal" draws use an Irwin-Hall(4) sum of four 16-bit uniforms from one
  64-bit hash, rescaled to unit variance (support +-3.46 sigma).  Hidden states
  after the final RMSNorm are roughly unit-scale (SURVEY 8d "flat" regime).
* bf16 values are produced by IEEE round-to-nearest-even from fp32 bits.
* Zipf(1.1) labels (BPE-like frequency skew) use a CDF built with
  Python's libm ``math.pow``; labels are additionally stored next to any golden
  values so a 1-ulp libm difference can never silently change a fixture.

Workload recipes:
  tiny     N=64 (1x64),  D=64,   V=1000,   exactly 6 of 64 ignored (10%)
  qwen05b  N=8192 (8x1024), D=896, V=151936, packed padding, 40% ignored
           (N_valid = 4915 after the trim rule)
  mem      N=16384 (4x4096), D=2048, V=151936
  llama8b  N=16384 (4x4096), D=4096, V=128256
  qwen7b   N=32768 (8x4096), D=3584, V=152064
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

M64 = (1 << 64) - 1
IGNORE_INDEX = -100

# streams (independent counter spaces)
S_H, S_W, S_LABEL, S_PACK, S_PERM, S_PLANT = 1, 2, 3, 4, 5, 6


def _splitmix64(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64, copy=False)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def _key(seed: int, stream: int) -> np.uint64:
    k = _splitmix64(np.array([(seed * 0x632BE59BD9B4E019 + stream * 0x9E3779B97F4A7C15) & M64],
                             dtype=np.uint64))
    return k[0]


def hash_u64(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """count 64-bit hashes for counters [start, start+count)."""
    ctr = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _splitmix64(ctr + _key(seed, stream))


def uniform01(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """Uniform in (0,1) with 53-bit resolution, exact in fp64."""
    h = hash_u64(seed, stream, start, count)
    return ((h >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def randint(seed: int, stream: int, start: int, count: int, lo: int, hi: int) -> np.ndarray:
    """Integers uniform in [lo, hi] (inclusive), via 53-bit uniforms (bias < 2^-40)."""
    u = uniform01(seed, stream, start, count)
    return lo + np.floor(u * (hi - lo + 1)).astype(np.int64)


def normal_f64(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """Irwin-Hall(4) approximately-normal draws, unit variance, exact in fp64."""
    h = hash_u64(seed, stream, start, count)
    m = np.uint64(0xFFFF)
    s = ((h & m) + ((h >> np.uint64(16)) & m) + ((h >> np.uint64(32)) & m) + (h >> np.uint64(48)))
    u = (s.astype(np.float64) + 2.0) * (1.0 / 65536.0)      # sum of four U(0,1), mean 2, var 1/3
    return (u - 2.0) * math.sqrt(3.0)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """IEEE fp32 -> bf16 bit patterns, round-to-nearest-even (no NaNs expected)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))
    return (b >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def normal_bf16(seed: int, stream: int, rows: int, cols: int, std: float,
                chunk_elems: int = 1 << 23, row_start: int = 0) -> np.ndarray:
    """[rows, cols] bf16 bit patterns of std * N(0,1)-ish draws (counter = row*cols+col),
    for global rows [row_start, row_start+rows) -- a shard is generated directly."""
    total = rows * cols
    base = row_start * cols
    out = np.empty(total, dtype=np.uint16)
    for s in range(0, total, chunk_elems):
        c = min(chunk_elems, total - s)
        out[s:s + c] = f32_to_bf16_bits((normal_f64(seed, stream, base + s, c) * std).astype(np.float32))
    return out.reshape(rows, cols)


def _as_i64(c: int) -> int:
    """uint64 constant -> the int64 with the same bits."""
    c &= M64
    return c - (1 << 64) if c >= (1 << 63) else c


def _lsr(z, k: int):
    """Logical right shift of int64 bit patterns (torch's >> is arithmetic)."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def normal_bf16_torch(seed: int, stream: int, rows: int, cols: int, std: float, device,
                      row_start: int = 0, chunk_elems: int = 1 << 27):
    """normal_bf16 evaluated with torch int64 / fp64 ops on `device` (for inputs too large
    to draw with numpy in a test, e.g. a 2.5e9-element W): the same splitmix64 counters,
    Irwin-Hall sum and round-to-nearest-even casts, so the bits equal normal_bf16's
    (tests/test_workload.py checks that on CPU).  Returns a [rows, cols] torch.bfloat16."""
    import torch
    key = _as_i64(int(_key(seed, stream)))
    total = rows * cols
    base = row_start * cols
    out = torch.empty(total, dtype=torch.bfloat16, device=device)
    for s in range(0, total, chunk_elems):
        c = min(chunk_elems, total - s)
        z = torch.arange(base + s, base + s + c, dtype=torch.int64, device=device) + key
        z = z + _as_i64(0x9E3779B97F4A7C15)
        z = (z ^ _lsr(z, 30)) * _as_i64(0xBF58476D1CE4E5B9)
        z = (z ^ _lsr(z, 27)) * _as_i64(0x94D049BB133111EB)
        h = z ^ _lsr(z, 31)
        sm = (h & 0xFFFF) + (_lsr(h, 16) & 0xFFFF) + (_lsr(h, 32) & 0xFFFF) + _lsr(h, 48)
        u = (sm.to(torch.float64) + 2.0) * (1.0 / 65536.0)
        out[s:s + c] = (((u - 2.0) * math.sqrt(3.0)) * std).to(torch.float32).to(torch.bfloat16)
        del z, h, sm, u
    return out.view(rows, cols)


_ZIPF_CACHE: dict = {}


def zipf_cdf(V: int, s: float = 1.1) -> np.ndarray:
    key = (V, s)
    if key not in _ZIPF_CACHE:
        w = [math.pow(k, -s) for k in range(1, V + 1)]
        c = np.cumsum(np.array(w, dtype=np.float64))
        _ZIPF_CACHE[key] = c / c[-1]
    return _ZIPF_CACHE[key]


def zipf_labels(seed: int, n: int, V: int, s: float = 1.1, start: int = 0) -> np.ndarray:
    u = uniform01(seed, S_LABEL, start, n)
    lab = np.searchsorted(zipf_cdf(V, s), u, side="right")
    return np.minimum(lab, V - 1).astype(np.int32)


def packed_valid_mask(seed: int, n_rows: int, row_len: int, ignore_frac: float,
                      prompt=(16, 112), response=(16, 256)) -> np.ndarray:
    """SURVEY 8d "packed padding": each row is greedily filled with samples
    [prompt (ignored), response (valid)] until the next sample does not fit; the
    remainder of the row is an ignored tail pad.  Trim rule for an exact count:
    scan from the last position backwards flipping valid->ignored (too few
    ignored) or ignored->valid (too many) until #ignored == round(frac*N)."""
    N = n_rows * row_len
    valid = np.zeros(N, dtype=bool)
    ctr = 0
    for r in range(n_rows):
        pos = 0
        while True:
            p = int(randint(seed, S_PACK, ctr, 1, *prompt)[0]); ctr += 1
            q = int(randint(seed, S_PACK, ctr, 1, *response)[0]); ctr += 1
            if pos + p + q > row_len:
                break
            valid[r * row_len + pos + p: r * row_len + pos + p + q] = True
            pos += p + q
    target_ignored = int(round(ignore_frac * N))
    n_ign = int(N - valid.sum())
    i = N - 1
    while n_ign != target_ignored and i >= 0:
        if n_ign < target_ignored and valid[i]:
            valid[i] = False; n_ign += 1
        elif n_ign > target_ignored and not valid[i]:
            valid[i] = True; n_ign -= 1
        i -= 1
    return valid


def exact_count_valid_mask(seed: int, N: int, n_ignored: int) -> np.ndarray:
    """Exactly n_ignored positions ignored, chosen by a seeded permutation."""
    keys = hash_u64(seed, S_PERM, 0, N)
    order = np.argsort(keys, kind="stable")
    valid = np.ones(N, dtype=bool)
    valid[order[:n_ignored]] = False
    return valid


def bernoulli_valid_mask(seed: int, N: int, ignore_frac: float) -> np.ndarray:
    return uniform01(seed, S_PERM, 0, N) >= ignore_frac


@dataclass(frozen=True)
class Config:
    name: str
    n_rows: int
    row_len: int
    D: int
    V: int
    ignore: str      # "packed40", "exact6", "none", ...

    @property
    def N(self) -> int:
        return self.n_rows * self.row_len


CONFIGS = {
    "tiny": Config("tiny", 1, 64, 64, 1000, "exact6"),
    "qwen05b": Config("qwen05b", 8, 1024, 896, 151936, "packed40"),
    "mem": Config("mem", 4, 4096, 2048, 151936, "none"),
    "llama8b": Config("llama8b", 4, 4096, 4096, 128256, "none"),
    "qwen7b": Config("qwen7b", 8, 4096, 3584, 152064, "none"),
}


def valid_mask(seed: int, n_rows: int, row_len: int, ignore: str) -> np.ndarray:
    N = n_rows * row_len
    if ignore == "none":
        return np.ones(N, dtype=bool)
    if ignore == "all":
        return np.zeros(N, dtype=bool)
    if ignore.startswith("exact"):
        return exact_count_valid_mask(seed, N, int(ignore[5:]))
    if ignore.startswith("bern"):
        return bernoulli_valid_mask(seed, N, int(ignore[4:]) / 100.0)
    if ignore == "packed30":
        return packed_valid_mask(seed, n_rows, row_len, 0.30, (16, 64), (64, 320))
    if ignore == "packed40":
        return packed_valid_mask(seed, n_rows, row_len, 0.40)
    if ignore == "packed60":
        return packed_valid_mask(seed, n_rows, row_len, 0.60, (48, 208), (32, 224))
    raise ValueError(ignore)


def make_problem(N: int, D: int, V: int, seed: int = 42, valid: np.ndarray | None = None,
                 regime: str = "flat", n_rows: int = 1, ignore: str = "none",
                 label_dist: str = "zipf", w_rows: tuple | None = None):
    """Returns dict(H=[N,D] uint16 bf16 bits, W=[V,D] uint16, labels=[N] int32).
    w_rows=(lo, hi) generates only the vocabulary shard W[lo:hi] (same values).

    regimes: flat (default), peaked (planted targets t~U[6,24]), extreme
    (t~U[16,26]), zero (W = 0), smallv (flat with planted t~U[4,20] for V~20k)."""
    if valid is None:
        valid = valid_mask(seed, n_rows, N // n_rows, ignore)
    assert valid.shape == (N,)
    H = normal_bf16(seed, S_H, N, D, 1.0)
    lo, hi = w_rows if w_rows is not None else (0, V)
    if regime == "zero":
        W = np.zeros((hi - lo, D), dtype=np.uint16)
    else:
        W = normal_bf16(seed, S_W, hi - lo, D, 1.0 / math.sqrt(D), row_start=lo)
    if label_dist == "zipf":
        lab_all = zipf_labels(seed, N, V)
    else:
        lab_all = randint(seed, S_LABEL, 0, N, 0, V - 1).astype(np.int32)
    labels = np.where(valid, lab_all, IGNORE_INDEX).astype(np.int32)
    if regime in ("peaked", "extreme", "smallv"):
        assert w_rows is None, "planted regimes need the full W"
        lo, hi = {"peaked": (6.0, 24.0), "extreme": (16.0, 26.0), "smallv": (4.0, 20.0)}[regime]
        t = lo + (hi - lo) * uniform01(seed, S_PLANT, 0, N)
        Hf = bf16_bits_to_f32(H).astype(np.float64)
        for n in np.nonzero(valid)[0]:
            wy = bf16_bits_to_f32(W[labels[n]]).astype(np.float64)
            nrm2 = float(np.sum(wy * wy))     # exact: squares of bf16 fit in 16 bits
            Hf[n] += t[n] * wy / nrm2
        H = f32_to_bf16_bits(Hf.astype(np.float32))
    return {"H": H, "W": W, "labels": labels}


def make_config(name: str, seed: int = 42, regime: str = "flat", ignore: str | None = None,
                w_rows: tuple | None = None):
    c = CONFIGS[name]
    return make_problem(c.N, c.D, c.V, seed=seed, regime=regime, n_rows=c.n_rows,
                        ignore=ignore if ignore is not None else c.ignore, w_rows=w_rows)


S_ADAM_M, S_ADAM_V = 101, 102


def make_adamw_state(seed: int, shape, g_scale: float):
    """Warm AdamW moments (SURVEY 8(f) NEXT #2 test inputs), float32 arrays of `shape`:
    m ~ 0.5 g_scale N(0,1) and v ~ g_scale^2 U(0.5, 2), i.e. the state after a few steps
    with gradients of rms g_scale (v > 0 keeps the update a smooth function of g)."""
    n = int(np.prod(shape))
    m = (0.5 * g_scale * normal_f64(seed, S_ADAM_M, 0, n)).astype(np.float32).reshape(shape)
    v = ((g_scale * g_scale) * (0.5 + 1.5 * uniform01(seed, S_ADAM_V, 0, n))).astype(np.float32).reshape(shape)
    return m, v


S_NORM_X, S_NORM_G = 103, 104


def make_rmsnorm_inputs(seed: int, N: int, D: int, x_std: float = 2.0, g_std: float = 0.1):
    """Inputs of the RMSNorm prologue: the un-normalised final hidden
    states X ~ x_std N(0,1) and a learned-looking scale gamma ~ 1 + g_std N(0,1), both bf16
    bit patterns (RNE)."""
    X = normal_bf16(seed, S_NORM_X, N, D, x_std)
    g = f32_to_bf16_bits((1.0 + g_std * normal_f64(seed, S_NORM_G, 0, D)).astype(np.float32))
    return X, g
