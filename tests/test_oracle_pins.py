"""Pins for the CPU oracle (SURVEY 8c "What pins each part").

Each test checks the oracle against something other than itself: a closed form,
an invariant, a worked example printed in the paper/SPEC (tests/golden), finite
differences, or a library routine.  The aim is that any plausible mistake in
oracle/cce_oracle.c (dropped term, sign, index, transposed operand, wrong
divisor, missing max-shift) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import workload

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _rand_problem(N, D, V, seed, ignore_n=0, scale_w=1.0):
    rng = np.random.default_rng(seed)
    H = rng.standard_normal((N, D))
    W = rng.standard_normal((V, D)) * scale_w / math.sqrt(D)
    y = rng.integers(0, V, N).astype(np.int32)
    if ignore_n:
        y[rng.permutation(N)[:ignore_n]] = -100
    return H, W, y


# ---------------------------------------------------------------- worked examples
def test_golden_online_softmax_examples():
    """printed LSE values through the online (m,d) recursion."""
    for key in ("online_lse_123", "lse_00", "lse_big"):
        g = GOLD[key]
        assert abs(oracle.online_lse(g["x"]) - g["lse"]) <= g["tol"], key
    # any order ("in any order")
    for perm in ([3.0, 1.0, 2.0], [2.0, 3.0, 1.0]):
        assert abs(oracle.online_lse(perm) - GOLD["online_lse_123"]["lse"]) <= 5e-5


def test_golden_zero_logits_loss():
    """all-zero logits, V=97 -> loss ln 97 for any target; P:236 Qwen vocab."""
    for key in ("zero_logits_V97",):
        g = GOLD[key]
        V = g["V"]
        H = np.ones((3, 8))
        W = np.zeros((V, 8))
        y = np.array([0, 5, V - 1], np.int32)
        r = oracle.cce(H, W, y)
        assert abs(r["loss"] - g["loss"]) <= g["tol"]


def test_golden_paper_arithmetic():
    """P:487-490 (4.97 GB of fp32 logits) and P:583 (37x) -- the quantities the
    bench's memory report uses to show no N x V buffer is allocated."""
    g = GOLD["logit_memory_bytes"]
    assert abs(g["B"] * g["N"] * g["V"] * 4 / 1e9 - g["GB"]) <= g["tol"]
    g = GOLD["cce_reduction_factor"]
    assert abs(g["V"] / g["C"] - g["factor"]) <= 0.1


# ---------------------------------------------------------------- pin 1: W = 0
@pytest.mark.parametrize("V", [1000, 151936])
def test_pin1_W_zero(V):
    N, D = 6, 16
    rng = np.random.default_rng(1)
    H = rng.standard_normal((N, D))
    W = np.zeros((V, D))
    y = np.array([0, 3, -100, 3, V - 1, 7], np.int32)
    r = oracle.cce(H, W, y, dloss=1.0, grads=(V <= 1000))
    lnV = math.log(V)
    valid = y != -100
    assert r["n_valid"] == 5
    assert abs(r["loss"] - lnV) <= 1e-12
    assert np.all(np.abs(r["lse"][valid] - lnV) <= 1e-12)
    assert np.all(r["lse"][~valid] == 0.0)
    if V == 151936:
        assert abs(r["loss"] - GOLD["zero_logits_qwen_vocab"]["loss"]) <= 5e-10
        return
    assert np.all(r["dH"] == 0.0)
    # closed form dW[v] = s * ((1/V) sum_valid h_n - sum_{valid n: y_n = v} h_n)
    s = 1.0 / 5
    ref = np.tile(H[valid].sum(0) / V, (V, 1))
    for n in np.nonzero(valid)[0]:
        ref[y[n]] -= H[n]
    ref *= s
    np.testing.assert_allclose(r["dW"], ref, rtol=0, atol=1e-13)


# ---------------------------------------------------------------- pin 2: H = 0
def test_pin2_H_zero():
    N, D, V = 5, 12, 300
    rng = np.random.default_rng(2)
    H = np.zeros((N, D))
    W = rng.standard_normal((V, D))
    y = np.array([4, -100, 299, 0, 4], np.int32)
    r = oracle.cce(H, W, y, dloss=0.5)
    assert abs(r["loss"] - math.log(V)) <= 1e-12
    assert np.all(r["dW"] == 0.0)
    s = 0.5 / 4
    for n in range(N):
        if y[n] == -100:
            assert np.all(r["dH"][n] == 0.0)
        else:
            np.testing.assert_allclose(r["dH"][n], s * (W.mean(0) - W[y[n]]), atol=1e-13)


# ---------------------------------------------------------------- pins 3,4,5: G
def test_pin3_gradient_is_softmax_minus_onehot_fd():
    """dL/dz = softmax - onehot, checked by central differences of the
    per-row loss with respect to the logits (independent computation)."""
    N, D, V = 3, 5, 11
    H, W, y = _rand_problem(N, D, V, 3)
    G = oracle.dlogits(H, W, y, dloss=1.0)
    z = H @ W.T
    eps = 1e-6
    for n in range(N):
        for v in range(V):
            zp = z[n].copy(); zp[v] += eps
            zm = z[n].copy(); zm[v] -= eps
            lp = np.log(np.sum(np.exp(zp))) - zp[y[n]]
            lm = np.log(np.sum(np.exp(zm))) - zm[y[n]]
            fd = (lp - lm) / (2 * eps) / N
            assert abs(G[n, v] - fd) <= 1e-8


def test_pin4_rows_sum_to_zero_and_dW_column_sums():
    N, D, V = 16, 24, 500
    H, W, y = _rand_problem(N, D, V, 4, ignore_n=3)
    G = oracle.dlogits(H, W, y, dloss=1.0)
    assert np.max(np.abs(G.sum(1))) <= 1e-12 * V
    r = oracle.cce(H, W, y)
    assert np.max(np.abs(r["dW"].sum(0))) <= 1e-12 * np.abs(r["dW"]).max() * V


def test_pin5_gradient_bound():
    """||grad_z L||_inf <= 1 per row; with the mean, <= |dloss|/n_valid."""
    N, D, V = 20, 16, 257
    H, W, y = _rand_problem(N, D, V, 5, ignore_n=4, scale_w=8.0)
    dloss = -2.5
    G = oracle.dlogits(H, W, y, dloss=dloss)
    assert np.max(np.abs(G)) <= abs(dloss) / 16 + 1e-15


# ---------------------------------------------------------------- pin 6: all ignored
def test_pin6_all_ignored():
    H, W, _ = _rand_problem(8, 8, 50, 6)
    y = np.full(8, -100, np.int32)
    r = oracle.cce(H, W, y)
    assert r["n_valid"] == 0 and r["loss"] == 0.0
    assert np.all(r["dH"] == 0.0) and np.all(r["dW"] == 0.0) and np.all(r["lse"] == 0.0)


# ---------------------------------------------------------------- pin 7: online merge
def _merge(parts):
    """The (m, d) merge of P:1157-1163 / P:521-541, written out for the test."""
    m = -np.inf
    d = 0.0
    for mi, di in parts:
        if di == 0.0:
            continue
        mn = max(m, mi)
        d = (d * math.exp(m - mn) if d > 0 else 0.0) + di * math.exp(mi - mn)
        m = mn
    return m + math.log(d)


@pytest.mark.parametrize("width", [1, 7, 64, 128, 1005])
def test_pin7_online_equals_two_pass(width):
    rng = np.random.default_rng(width)
    for _ in range(50):
        x = rng.standard_normal(1000) * 5
        x[rng.integers(0, 1000, 3)] = x.max()           # duplicated maxima
        two_pass = x.max() + math.log(np.sum(np.exp(x - x.max())))
        assert abs(oracle.online_lse(x) - two_pass) <= 1e-12 * abs(two_pass) + 1e-12
        assert abs(oracle.online_lse(rng.permutation(x)) - two_pass) <= 1e-12 * abs(two_pass) + 1e-12
        parts = []
        for s in range(0, len(x), width):
            c = x[s:s + width]
            parts.append((c.max(), float(np.sum(np.exp(c - c.max())))))
        assert abs(_merge(parts) - two_pass) <= 1e-12 * abs(two_pass) + 1e-12


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_pin7_sharded_partial_stats_merge(P):
    """Vocabulary shards: per-shard (m, d, z_y) merged in rank order
    equal the unsharded oracle (lse and loss), including uneven and empty shards."""
    N, D, V = 12, 16, 1000
    H, W, y = _rand_problem(N, D, V, 70 + P, ignore_n=2)
    full = oracle.cce(H, W, y, grads=False)
    bounds = np.linspace(0, V, P + 1).astype(int)
    if P == 3:
        bounds = np.array([0, 0, 517, V])      # an empty shard and an uneven split
    stats = [oracle.partial_stats(H, W[bounds[r]:bounds[r + 1]], y, bounds[r]) for r in range(len(bounds) - 1)]
    for n in range(N):
        if y[n] == -100:
            continue
        lse = _merge([(s[0][n], s[1][n]) for s in stats])
        zy = sum(s[2][n] for s in stats)
        assert abs(lse - full["lse"][n]) <= 1e-12 * abs(lse)
        assert abs(zy - (H[n] @ W[y[n]])) <= 1e-12


# ---------------------------------------------------------------- pin 8: finite differences
@pytest.mark.parametrize("shape", [(4, 8, 50), (7, 16, 333)])
def test_pin8_finite_differences(shape):
    N, D, V = shape
    H, W, y = _rand_problem(N, D, V, 8 + N, ignore_n=1)
    r = oracle.cce(H, W, y, dloss=1.0)
    eps = 1e-6

    def loss(Hx, Wx):
        return oracle.cce(Hx, Wx, y, grads=False)["loss"]

    rng = np.random.default_rng(0)
    fdH = np.zeros_like(H)
    for n in range(N):
        for d in range(D):
            Hp = H.copy(); Hp[n, d] += eps
            Hm = H.copy(); Hm[n, d] -= eps
            fdH[n, d] = (loss(Hp, W) - loss(Hm, W)) / (2 * eps)
    assert np.linalg.norm(fdH - r["dH"]) <= 1e-6 * np.linalg.norm(r["dH"])
    vs = list(rng.choice(V, 12, replace=False)) + [int(y[0]) if y[0] >= 0 else int(y[1])]
    for v in vs:
        fd = np.zeros(D)
        for d in range(D):
            Wp = W.copy(); Wp[v, d] += eps
            Wm = W.copy(); Wm[v, d] -= eps
            fd[d] = (loss(H, Wp) - loss(H, Wm)) / (2 * eps)
        assert np.linalg.norm(fd - r["dW"][v]) <= 1e-6 * max(np.linalg.norm(r["dW"][v]), 1e-3)


# ---------------------------------------------------------------- pin 9: shift invariance
def test_pin9_shift_invariance():
    """Append a constant column: H' = [H, 1], W' = [W, c] (c = 80, exact in bf16):
    lse' = lse + c; loss, dH[:, :D], dW[:, :D] unchanged (exercises the max shift)."""
    N, D, V = 10, 15, 400
    H, W, y = _rand_problem(N, D, V, 9, ignore_n=2)
    c = 80.0
    H2 = np.concatenate([H, np.ones((N, 1))], 1)
    W2 = np.concatenate([W, np.full((V, 1), c)], 1)
    a = oracle.cce(H, W, y)
    b = oracle.cce(H2, W2, y)
    valid = y != -100
    np.testing.assert_allclose(b["lse"][valid], a["lse"][valid] + c, rtol=1e-13)
    assert abs(a["loss"] - b["loss"]) <= 1e-11
    np.testing.assert_allclose(b["dH"][:, :D], a["dH"], atol=1e-12)
    np.testing.assert_allclose(b["dW"][:, :D], a["dW"], atol=1e-12)


# ---------------------------------------------------------------- pin 10: V = 2
def test_pin10_two_classes_softplus():
    N, D = 9, 6
    H, W, y = _rand_problem(N, D, 2, 10)
    r = oracle.cce(H, W, y, grads=False)
    z = H @ W.T
    ref = np.mean([np.logaddexp(0.0, z[n, 1 - y[n]] - z[n, y[n]]) for n in range(N)])
    assert abs(r["loss"] - ref) <= 1e-13


# ---------------------------------------------------------------- pin 11: linearity in dloss
def test_pin11_linear_in_dloss():
    H, W, y = _rand_problem(6, 8, 90, 11, ignore_n=1)
    a = oracle.cce(H, W, y, dloss=1.0)
    b = oracle.cce(H, W, y, dloss=0.37)
    z = oracle.cce(H, W, y, dloss=0.0)
    np.testing.assert_allclose(b["dH"], 0.37 * a["dH"], rtol=1e-12, atol=1e-16)
    np.testing.assert_allclose(b["dW"], 0.37 * a["dW"], rtol=1e-12, atol=1e-16)
    assert np.all(z["dH"] == 0) and np.all(z["dW"] == 0)
    assert a["loss"] == b["loss"]


# ---------------------------------------------------------------- pin 12: library routine
@pytest.mark.parametrize("seed", [0, 1])
def test_pin12_matches_torch_fp64(seed):
    torch = pytest.importorskip("torch")
    N, D, V = 24, 32, 777
    H, W, y = _rand_problem(N, D, V, 120 + seed, ignore_n=5)
    Ht = torch.tensor(H, requires_grad=True)
    Wt = torch.tensor(W, requires_grad=True)
    lt = torch.nn.functional.cross_entropy(Ht @ Wt.T, torch.tensor(y, dtype=torch.long), ignore_index=-100)
    lt.backward()
    r = oracle.cce(H, W, y)
    assert abs(r["loss"] - lt.item()) <= 1e-12
    np.testing.assert_allclose(r["dH"], Ht.grad.numpy(), rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(r["dW"], Wt.grad.numpy(), rtol=1e-10, atol=1e-14)


# ---------------------------------------------------------------- pin 13: sanity bounds
def test_pin13_bounds_on_workload_inputs():
    p = workload.make_config("tiny", seed=3)
    r = oracle.cce(p["H"], p["W"], p["labels"])
    Hf = oracle._bits(p["H"]); Wf = oracle._bits(p["W"])
    z = Hf @ Wf.T
    valid = p["labels"] != -100
    for n in np.nonzero(valid)[0]:
        zy = z[n, p["labels"][n]]
        assert zy <= r["lse"][n] + 1e-12
        assert z[n].max() <= r["lse"][n] <= z[n].max() + math.log(z.shape[1]) + 1e-12
    assert r["loss"] >= 0


# ---------------------------------------------------------------- errors, sampled entry points
def test_label_range_error():
    H, W, y = _rand_problem(4, 4, 10, 12)
    y[2] = 10
    with pytest.raises(oracle.OracleError):
        oracle.cce(H, W, y)
    y[2] = -1
    with pytest.raises(oracle.OracleError):
        oracle.cce(H, W, y)


def test_rows_and_dW_rows_agree_with_full():
    p = workload.make_config("tiny", seed=4)
    full = oracle.cce(p["H"], p["W"], p["labels"], dloss=1.0)
    valid_rows = np.nonzero(p["labels"] != -100)[0]
    s = 1.0 / len(valid_rows)
    lse, zy, dH = oracle.rows(p["H"], p["W"], p["labels"], valid_rows[:9], scale=s)
    np.testing.assert_allclose(lse, full["lse"][valid_rows[:9]], rtol=1e-14)
    np.testing.assert_allclose(dH, full["dH"][valid_rows[:9]], rtol=1e-12, atol=1e-15)
    vr = np.array([0, 1, 17, 999])
    dW = oracle.dW_rows(p["H"], p["W"], p["labels"], full["lse"], s, vr)
    np.testing.assert_allclose(dW, full["dW"][vr], rtol=1e-12, atol=1e-15)


# ---------------------------------------------------------------- the generator
def test_workload_packed_padding_recipe():
    for seed in range(3):
        m = workload.valid_mask(seed, 8, 1024, "packed40")
        assert m.sum() == 4915 and (~m).sum() == 3277
    m = workload.valid_mask(0, 1, 64, "exact6")
    assert (~m).sum() == 6
    x = workload.normal_f64(7, 1, 0, 200000)
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1) < 0.01
    a = workload.normal_bf16(1, 2, 3, 5, 1.0)
    b = workload.normal_bf16(1, 2, 3, 5, 1.0, chunk_elems=4)
    assert np.array_equal(a, b)


# ---------------------------------------------------------------- regularised loss (NEXT #1)
# Label smoothing (Def. Smoothed CE) and z-loss (Def. Z-Loss, P:281-287;
# gradient Prop. P:2686-2691); readings R11 / R12.
def test_golden_zloss_zero_logits():
    """all-zero logits, lambda_z = 1e-4, V = 97 -> the z-loss adds 1e-4 (ln 97)^2 =
    2.093e-3; with W = 0 label smoothing leaves the loss at ln V (z_y = mean z = 0)."""
    g = GOLD["zloss_zero_logits_V97"]
    V = g["V"]
    H = np.ones((4, 8))
    W = np.zeros((V, 8))
    y = np.array([0, 5, V - 1, 40], np.int32)
    base = oracle.cce(H, W, y)["loss"]
    r = oracle.cce(H, W, y, z_loss=g["z_weight"])
    assert abs((r["loss"] - base) - g["extra"]) <= g["tol"]
    for eps in (0.1, 0.5):
        r2 = oracle.cce(H, W, y, z_loss=g["z_weight"], label_smoothing=eps)
        assert abs(r2["loss"] - r["loss"]) <= 1e-14
        # W = 0: p = 1/V, so G = s [(1 + 2 lam ln V)/V - (1-eps) 1[y] - eps/V]
        s = 1.0 / len(y)
        G = oracle.dlogits(H, W, y, label_smoothing=eps, z_loss=g["z_weight"])
        want = s * ((1 + 2 * g["z_weight"] * math.log(V)) / V - eps / V)
        assert abs(G[0, 1] - want) <= 1e-15
        assert abs(G[0, 0] - (want - s * (1 - eps))) <= 1e-15


@pytest.mark.parametrize("eps,lam", [(0.1, 0.0), (0.0, 1e-2), (0.1, 1e-4), (0.3, 5e-2)])
def test_regularised_matches_torch_fp64(eps, lam):
    """Library routine: torch fp64 cross_entropy(label_smoothing=eps) -- its definition
    (1-eps) nll + eps (lse - mean z) is P:272-276 -- plus lam * mean_valid(lse^2),
    autograd for the gradients."""
    torch = pytest.importorskip("torch")
    N, D, V = 20, 24, 531
    H, W, y = _rand_problem(N, D, V, 300 + int(eps * 10) + int(lam * 1e4), ignore_n=4)
    Ht = torch.tensor(H, requires_grad=True)
    Wt = torch.tensor(W, requires_grad=True)
    yt = torch.tensor(y, dtype=torch.long)
    z = Ht @ Wt.T
    ce = torch.nn.functional.cross_entropy(z, yt, ignore_index=-100, label_smoothing=eps)
    valid = yt != -100
    lse = torch.logsumexp(z[valid], dim=1)
    lt = ce + lam * (lse * lse).mean()
    lt.backward()
    r = oracle.cce(H, W, y, label_smoothing=eps, z_loss=lam)
    assert abs(r["loss"] - lt.item()) <= 1e-12
    np.testing.assert_allclose(r["dH"], Ht.grad.numpy(), rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(r["dW"], Wt.grad.numpy(), rtol=1e-10, atol=1e-14)


def test_regularised_finite_differences():
    N, D, V = 5, 7, 60
    H, W, y = _rand_problem(N, D, V, 31, ignore_n=1)
    eps_ls, lam = 0.2, 3e-2
    r = oracle.cce(H, W, y, label_smoothing=eps_ls, z_loss=lam)
    h = 1e-6

    def loss(Hx, Wx):
        return oracle.cce(Hx, Wx, y, grads=False, label_smoothing=eps_ls, z_loss=lam)["loss"]

    fdH = np.zeros_like(H)
    for n in range(N):
        for d in range(D):
            Hp = H.copy(); Hp[n, d] += h
            Hm = H.copy(); Hm[n, d] -= h
            fdH[n, d] = (loss(Hp, W) - loss(Hm, W)) / (2 * h)
    assert np.linalg.norm(fdH - r["dH"]) <= 1e-6 * np.linalg.norm(r["dH"])
    for v in (0, 7, int(y[0]) if y[0] >= 0 else int(y[1]), V - 1):
        fd = np.zeros(D)
        for d in range(D):
            Wp = W.copy(); Wp[v, d] += h
            Wm = W.copy(); Wm[v, d] -= h
            fd[d] = (loss(H, Wp) - loss(H, Wm)) / (2 * h)
        assert np.linalg.norm(fd - r["dW"][v]) <= 1e-6 * max(np.linalg.norm(r["dW"][v]), 1e-3)


def test_regularised_row_sums_and_limits():
    """Row sums of the regularised dlogits: (1-eps)*0 + eps*(1 - 1) + 2 lam lse * 1, so
    sum_v G[n,v] = s 2 lam lse_n (label smoothing drops out); eps = lam = 0 is the
    plain loss bit for bit."""
    N, D, V = 9, 12, 300
    H, W, y = _rand_problem(N, D, V, 41, ignore_n=2)
    eps, lam = 0.15, 7e-3
    G = oracle.dlogits(H, W, y, label_smoothing=eps, z_loss=lam)
    r = oracle.cce(H, W, y, label_smoothing=eps, z_loss=lam, grads=False)
    s = 1.0 / int((y != -100).sum())
    for n in range(N):
        want = 0.0 if y[n] == -100 else s * 2 * lam * r["lse"][n]
        assert abs(G[n].sum() - want) <= 1e-14
    a = oracle.cce(H, W, y)
    b = oracle.cce(H, W, y, label_smoothing=0.0, z_loss=0.0)
    assert a["loss"] == b["loss"] and np.array_equal(a["dH"], b["dH"]) and np.array_equal(a["dW"], b["dW"])


# ---------------------------------------------------------------- reductions (NEXT #3)
@pytest.mark.parametrize("reduction,eps,lam", [("sum", 0.0, 0.0), ("none", 0.0, 0.0), ("sum", 0.1, 1e-3),
                                               ("none", 0.2, 5e-3)])
def test_reductions_match_torch_fp64(reduction, eps, lam):
    """Library routine: torch fp64 cross_entropy(reduction='sum'/'none', label_smoothing)
    + lam lse^2 per valid row, autograd with per-row upstream gradients for 'none'."""
    torch = pytest.importorskip("torch")
    N, D, V = 18, 20, 401
    H, W, y = _rand_problem(N, D, V, 500 + len(reduction) + int(eps * 10), ignore_n=4)
    Ht = torch.tensor(H, requires_grad=True)
    Wt = torch.tensor(W, requires_grad=True)
    yt = torch.tensor(y, dtype=torch.long)
    z = Ht @ Wt.T
    valid = (yt != -100).double()
    ce = torch.nn.functional.cross_entropy(z, yt, ignore_index=-100, label_smoothing=eps, reduction="none")
    lse = torch.logsumexp(z, dim=1)
    rows = (ce + lam * lse * lse) * valid
    rng = np.random.default_rng(7)
    if reduction == "sum":
        lt = rows.sum()
        lt.backward(torch.tensor(0.6, dtype=torch.float64))
        r = oracle.cce(H, W, y, dloss=0.6, label_smoothing=eps, z_loss=lam, reduction="sum")
        assert abs(r["loss"] - lt.item()) <= 1e-12
    else:
        g = rng.standard_normal(N)
        rows.backward(torch.tensor(g))
        r = oracle.cce(H, W, y, dloss=g, label_smoothing=eps, z_loss=lam, reduction="none")
        np.testing.assert_allclose(r["loss"], rows.detach().numpy(), rtol=1e-12, atol=1e-14)
        assert np.all(r["loss"][y == -100] == 0.0)
    np.testing.assert_allclose(r["dH"], Ht.grad.numpy(), rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(r["dW"], Wt.grad.numpy(), rtol=1e-10, atol=1e-14)


# ---------------------------------------------------------------- fused AdamW (NEXT #2)
def test_adamw_spec_worked_examples():
    """theta=1, g=1, lr=0.1, wd=0, t=1 -> 0.9000; g=0, wd=0.01, lr=0.1 -> theta*0.999."""
    th, m, v = oracle.adamw_step([1.0], [1.0], [0.0], [0.0], lr=0.1, weight_decay=0.0, step=1)
    assert abs(th[0] - 0.9000) <= 5e-5 and abs(th[0] - (1 - 0.1 / (1 + 1e-8))) <= 1e-15
    th, m, v = oracle.adamw_step([2.0, -3.0], [0.0, 0.0], [0.0, 0.0], [0.0, 0.0], lr=0.1, weight_decay=0.01)
    np.testing.assert_allclose(th, [2.0 * 0.999, -3.0 * 0.999], rtol=0, atol=1e-15)


@pytest.mark.parametrize("step,clip", [(1, 1.0), (5, 0.5)])
def test_adamw_matches_torch_fp64(step, clip):
    """Library routine: torch.optim.AdamW (fp64) after `step - 1` warm-up steps, with the
    clipping coefficient applied to the gradient first."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(step)
    n = 257
    th0 = rng.standard_normal(n)
    grads = [rng.standard_normal(n) * 10.0 ** rng.uniform(-8, 0, n) for _ in range(step)]
    p = torch.nn.Parameter(torch.tensor(th0))
    opt = torch.optim.AdamW([p], lr=3e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
    th, m, v = th0.copy(), np.zeros(n), np.zeros(n)
    for t, g in enumerate(grads, start=1):
        p.grad = torch.tensor(g * clip)
        opt.step()
        th, m, v = oracle.adamw_step(th, g, m, v, lr=3e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1,
                                     clip_coef=clip, step=t)
    np.testing.assert_allclose(th, p.detach().numpy(), rtol=1e-13, atol=1e-15)
    st = opt.state[p]
    # torch forms m with lerp (m + (1 - b1)(g - m)): same value, different rounding
    np.testing.assert_allclose(m, st["exp_avg"].numpy(), rtol=1e-12, atol=1e-30)
    np.testing.assert_allclose(v, st["exp_avg_sq"].numpy(), rtol=1e-12, atol=1e-30)


# ---------------------------------------------------------------- RMSNorm prologue (NEXT #4)
def test_rmsnorm_spec_worked_examples():
    """x=[1,1,1,1], gamma=1, eps=0 -> y=x, rstd=1; x=[3,4] -> rstd=1/3.5355,
    y=[0.8485, 1.1314] (mean square 12.5); scale invariance for eps=0."""
    y, r = oracle.rmsnorm_fwd(np.ones((1, 4)), np.ones(4), 0.0)
    assert np.all(y == 1.0) and r[0] == 1.0
    y, r = oracle.rmsnorm_fwd(np.array([[3.0, 4.0]]), np.ones(2), 0.0)
    assert abs(1.0 / r[0] - 3.5355) <= 5e-5 and abs(1.0 / r[0] - math.sqrt(12.5)) <= 1e-15
    np.testing.assert_allclose(y[0], [0.8485, 1.1314], atol=5e-5)
    x = np.random.default_rng(0).standard_normal((3, 16))
    g = np.random.default_rng(1).standard_normal(16)
    np.testing.assert_allclose(oracle.rmsnorm_fwd(7.5 * x, g, 0.0)[0], oracle.rmsnorm_fwd(x, g, 0.0)[0],
                               rtol=1e-14, atol=1e-15)


def test_rmsnorm_backward_special_cases():
    """dy = 0 -> dx = 0, dgamma = 0; D = 1, eps = 0, gamma = 1: y = sign(x) is
    constant, so dx = 0 exactly (up to rounding of x rstd = +-1)."""
    x = np.array([[2.5], [-0.7]])
    y, r = oracle.rmsnorm_fwd(x, np.ones(1), 0.0)
    np.testing.assert_array_equal(y[:, 0], [1.0, -1.0])
    dx, dg = oracle.rmsnorm_bwd(np.array([[0.3], [1.1]]), x, np.ones(1), r)
    assert np.all(np.abs(dx) <= 1e-16)
    dx, dg = oracle.rmsnorm_bwd(np.zeros((2, 1)), x, np.ones(1), r)
    assert np.all(dx == 0) and np.all(dg == 0)


@pytest.mark.parametrize("N,D,eps", [(5, 8, 1e-6), (3, 64, 1e-5), (4, 7, 0.3)])
def test_rmsnorm_matches_torch_autograd_fp64(N, D, eps):
    """Library routine: torch fp64 autograd of y = x rsqrt(mean(x^2) + eps) gamma, gamma != 1
    (so a gamma applied to the wrong term, as in the paper's garbled Prop., fails)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(N * D)
    x = rng.standard_normal((N, D)) * 3.0
    g = 1.0 + rng.standard_normal(D)
    dy = rng.standard_normal((N, D))
    xt = torch.tensor(x, requires_grad=True)
    gt = torch.tensor(g, requires_grad=True)
    yt = xt * torch.rsqrt((xt * xt).mean(dim=1, keepdim=True) + eps) * gt
    yt.backward(torch.tensor(dy))
    y, r = oracle.rmsnorm_fwd(x, g, eps)
    np.testing.assert_allclose(y, yt.detach().numpy(), rtol=1e-13, atol=1e-14)
    dx, dg = oracle.rmsnorm_bwd(dy, x, g, r)
    np.testing.assert_allclose(dx, xt.grad.numpy(), rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(dg, gt.grad.numpy(), rtol=1e-11, atol=1e-13)


def test_rmsnorm_finite_differences():
    """random (x, gamma, dy), D = 8: dx and dgamma match central finite differences
    of <dy, rmsnorm(x)> within 1e-6 relative."""
    rng = np.random.default_rng(3)
    N, D, eps = 3, 8, 1e-3
    x = rng.standard_normal((N, D))
    g = rng.standard_normal(D)
    dy = rng.standard_normal((N, D))
    f = lambda xx, gg: float(np.sum(dy * oracle.rmsnorm_fwd(xx, gg, eps)[0]))  # noqa: E731
    dx, dg = oracle.rmsnorm_bwd(dy, x, g, oracle.rmsnorm_fwd(x, g, eps)[1])
    h = 1e-6
    fx = np.zeros_like(x)
    for i in range(N):
        for j in range(D):
            e = np.zeros_like(x)
            e[i, j] = h
            fx[i, j] = (f(x + e, g) - f(x - e, g)) / (2 * h)
    fg = np.array([(f(x, g + h * np.eye(D)[j]) - f(x, g - h * np.eye(D)[j])) / (2 * h) for j in range(D)])
    assert np.linalg.norm(dx - fx) / np.linalg.norm(fx) <= 1e-6
    assert np.linalg.norm(dg - fg) / np.linalg.norm(fg) <= 1e-6


def test_rmsnorm_skipped_rows_and_composite():
    """Ignored rows (never read by the CE path) get dx = 0 and add nothing to dgamma; the
    composite oracle (bf16 H = RMSNorm(X), CE, RMSNorm backward) equals torch fp64 autograd
    through the same bf16 rounding of H (straight-through: rounding treated as identity in
    the gradient, which is what consuming a bf16 activation means)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(7)
    N, D, V = 12, 16, 40
    X = workload.f32_to_bf16_bits((rng.standard_normal((N, D)) * 2.0).astype(np.float32))
    G = workload.f32_to_bf16_bits((1.0 + 0.3 * rng.standard_normal(D)).astype(np.float32))
    W = workload.f32_to_bf16_bits((rng.standard_normal((V, D)) / 4.0).astype(np.float32))
    y = rng.integers(0, V, N).astype(np.int32)
    y[[1, 5, 6]] = -100
    r = oracle.cce_rmsnorm(X, G, W, y, eps=1e-6)
    assert np.all(r["dX"][[1, 5, 6]] == 0.0)
    f = lambda b: (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)  # noqa: E731
    xt = torch.tensor(f(X), requires_grad=True)
    gt = torch.tensor(f(G), requires_grad=True)
    Wt = torch.tensor(f(W))
    yn = xt * torch.rsqrt((xt * xt).mean(dim=1, keepdim=True) + 1e-6) * gt
    Hq = torch.tensor(f(r["H_bits"]))
    Hst = yn + (Hq - yn).detach()          # forward value = bf16 H, gradient straight through
    loss = torch.nn.functional.cross_entropy(Hst @ Wt.T, torch.tensor(y, dtype=torch.long), ignore_index=-100)
    loss.backward()
    assert abs(float(loss) - r["loss"]) <= 1e-12
    np.testing.assert_allclose(r["dX"], xt.grad.numpy(), rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(r["dgamma"], gt.grad.numpy(), rtol=1e-10, atol=1e-14)


# ---------------------------------------------------------------- bf16 rounding (oracle_to_bf16)
def _bf16_exact(x32):
    """Round a float32 value to bf16 with exact rationals: the nearest multiple of the bf16
    spacing at x's binade, ties to the even significand, overflow past the largest finite
    bf16 (plus half its spacing) to inf.  Independent of the oracle's bit manipulation."""
    from fractions import Fraction
    if math.isnan(x32):
        return None
    if math.isinf(x32):
        return x32
    q = Fraction(float(x32))
    if q == 0:
        return math.copysign(0.0, x32)
    a = abs(q)
    e = max(math.floor(math.log2(a)), -126)          # bf16 shares fp32's exponent range
    while Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a and e >= -126:
        e += 1
    e = max(e, -126)
    ulp = Fraction(2) ** (e - 7)                    # 8 significand bits (7 stored)
    k, r = divmod(a, ulp)
    if r > ulp / 2 or (r == ulp / 2 and k % 2 == 1):
        k += 1
    v = k * ulp
    bf_max = (2 - Fraction(1, 2 ** 7)) * Fraction(2) ** 127
    out = math.inf if v > bf_max else float(v)
    return -out if q < 0 else out


def _bits_to_f64(b):
    return (np.asarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _f32(bits):
    return np.array(bits, dtype=np.uint32).view(np.float32)


def _bf16_cases():
    """float32 inputs at every place a rounding mistake shows: exact ties with an even and
    an odd bf16 significand, one fp32 ulp either side of each tie, negatives, fp32 and bf16
    subnormals, the largest finite bf16 and the tie above it (-> inf), zeros, infinities."""
    base = []
    for hi in (0x3F80, 0x3F81, 0x4049, 0x404A, 0x0001, 0x0002, 0x007F, 0x0080, 0x7F7E, 0x7F7F, 0x1234, 0x1235):
        t = (hi << 16) | 0x8000                     # exact tie between hi and hi + 1
        base += [t, t - 1, t + 1, (hi << 16), (hi << 16) | 0x7FFF, (hi << 16) | 0xFFFF]
    base += [0x00000001, 0x00000002, 0x00008000, 0x00007FFF, 0x00018000, 0x7F7FFFFF,
             0x00000000, 0x7F800000]
    base = np.array(base, dtype=np.uint32)
    return np.concatenate([base, base | np.uint32(0x80000000)])


def test_to_bf16_exact_rounding():
    """oracle.to_bf16 on float32-representable inputs equals exact round-to-nearest-even."""
    x = _f32(_bf16_cases()).astype(np.float64)
    got = _bits_to_f64(oracle.to_bf16(x))
    for xi, gi in zip(x, got):
        want = _bf16_exact(np.float32(xi))
        assert (gi == want and math.copysign(1, gi) == math.copysign(1, want)), (float(xi), gi, want)


def test_to_bf16_matches_torch_cast():
    """... and torch's float32 -> bfloat16 cast, bit for bit (including inf on overflow);
    fp64 inputs go through fp32 first, as the oracle's reading R18 states."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(11)
    x = np.concatenate([_f32(_bf16_cases()).astype(np.float64),
                        rng.standard_normal(20000) * 10.0 ** rng.uniform(-40, 38, 20000)])
    ours = oracle.to_bf16(x)
    ref = torch.tensor(x.astype(np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)


def test_to_bf16_double_rounding_and_nan():
    """fp64 -> fp32 -> bf16: a double just above a bf16 tie that rounds onto the tie in fp32
    then ties to even (the two-step definition); NaN stays NaN with its sign."""
    tie = np.float64(_f32([0x3F808000])[0])               # 1 + 2^-8: tie, even neighbour 0x3F80
    just_above = tie + 2.0 ** -40                         # fp32 rounds it back onto the tie
    assert np.float32(just_above) == np.float32(tie)
    assert oracle.to_bf16(np.array([just_above]))[0] == 0x3F80
    assert oracle.to_bf16(np.array([tie + 2.0 ** -23]))[0] == 0x3F81   # a whole fp32 ulp above
    nan = oracle.to_bf16(np.array([np.nan, -np.nan, _f32([0x7FFFFFFF])[0].astype(np.float64)]))
    f = _bits_to_f64(nan)
    assert np.isnan(f).all()
    assert (nan[1] & 0x8000) and not (nan[0] & 0x8000)
