"""GPU parity of the RMSNorm prologue: cce_forward_rmsnorm /
cce_backward_rmsnorm against the fp64 oracle (oracle.cce_rmsnorm: H = bf16(RMSNorm(X)),
the plain CE oracle, then the exact RMSNorm backward, reading R18).  Tolerances are the
north_star's (loss abs 2e-3, LSE rel 1e-3, gradients rel Frobenius 1e-2); ignored rows
are bit-exact zeros and are never read."""
import numpy as np
import pytest

import oracle
import workload
from cce_testutil import TOL_GRAD, TOL_LOSS, TOL_LSE, bf16_to_f64, rel_fro

pytestmark = pytest.mark.gpu

EPS = 1e-6


@pytest.fixture(scope="module")
def dev():
    import torch
    import __graft_entry__
    __graft_entry__.build()
    return torch.device("cuda:0")


def _t(bits, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(dev)


def _run(dev, X, g, W, y, flags=0, dX_init=None, dg_init=None):
    import torch
    import paper_2601_02609_b200 as cce
    Xt, gt, Wt = _t(X, dev), _t(g, dev), _t(W, dev)
    yt = torch.from_numpy(y).to(dev)
    h = cce.CCEHandle(vocab_total=W.shape[0], flags=flags)
    loss, lse, nv = h.forward_rmsnorm(Xt, gt, EPS, Wt, yt)
    gdt = torch.float32 if flags & cce.FLAG_GRAD_FP32 else torch.bfloat16
    dX = dX_init if dX_init is not None else torch.full(Xt.shape, float("nan"), dtype=gdt, device=dev)
    dg = dg_init if dg_init is not None else torch.full(gt.shape, float("nan"), dtype=gdt, device=dev)
    dW = torch.empty(Wt.shape, dtype=gdt, device=dev)
    h.backward_rmsnorm(torch.ones((), dtype=torch.float32, device=dev), dX, dg, dW)
    torch.cuda.synchronize()
    h.close()
    f = (lambda t: t.cpu().numpy().astype(np.float64)) if gdt == torch.float32 else bf16_to_f64
    return {"loss": float(loss.item()), "lse": lse.cpu().numpy().astype(np.float64), "n_valid": int(nv.item()),
            "dX": f(dX), "dgamma": f(dg), "dW": f(dW), "dX_bits": dX.view(torch.int16).cpu().numpy()}


def _check(got, ref, y):
    valid = y != -100
    assert got["n_valid"] == int(valid.sum())
    assert abs(got["loss"] - ref["loss"]) <= TOL_LOSS
    if valid.any():
        rel = np.abs(got["lse"][valid] - ref["lse"][valid]) / np.maximum(np.abs(ref["lse"][valid]), 1.0)
        assert rel.max() <= TOL_LSE
    assert np.all(got["lse"][~valid] == 0.0)
    assert np.all(got["dX_bits"][~valid] == 0)
    for k in ("dX", "dgamma", "dW"):
        e = rel_fro(got[k], ref[k])
        assert e <= TOL_GRAD, (k, e)


@pytest.mark.parametrize("N,D,V,ign", [
    (64, 64, 1000, "bern10"),        # configs[0] shape
    (700, 128, 3000, "bern40"),      # ragged rows / vocabulary
    (384, 896, 9000, "bern40"),      # Qwen hidden size, 2 chunks
    (300, 4096, 5000, "bern40"),     # Llama-3-8B hidden size (64 KB of dgamma partials per block)
    (520, 2048, 9000, "none"),       # paper memory example hidden size, 0% ignored
])
def test_rmsnorm_prologue_parity(dev, N, D, V, ign):
    p = workload.make_problem(N, D, V, seed=N + D, ignore=ign)
    X, g = workload.make_rmsnorm_inputs(N + D, N, D)
    ref = oracle.cce_rmsnorm(X, g, p["W"], p["labels"], eps=EPS)
    got = _run(dev, X, g, p["W"], p["labels"])
    _check(got, ref, p["labels"])


def test_rmsnorm_prologue_grad_fp32_and_accumulate(dev):
    import torch
    import paper_2601_02609_b200 as cce
    p = workload.make_problem(700, 128, 3000, seed=3, ignore="bern40")
    X, g = workload.make_rmsnorm_inputs(3, 700, 128)
    ref = oracle.cce_rmsnorm(X, g, p["W"], p["labels"], eps=EPS)
    got = _run(dev, X, g, p["W"], p["labels"], flags=cce.FLAG_GRAD_FP32)
    assert np.all(got["dX"][p["labels"] == -100] == 0.0)
    for k in ("dX", "dgamma", "dW"):
        assert rel_fro(got[k], ref[k]) <= TOL_GRAD, k
    # accumulate into existing fp32 buffers: result = init + gradient, ignored rows untouched
    rng = np.random.default_rng(0)
    x0 = rng.standard_normal((700, 128)).astype(np.float32)
    g0 = rng.standard_normal(128).astype(np.float32)
    got2 = _run(dev, X, g, p["W"], p["labels"], flags=cce.FLAG_GRAD_FP32 | cce.FLAG_ACCUMULATE,
                dX_init=torch.from_numpy(x0.copy()).to(dev), dg_init=torch.from_numpy(g0.copy()).to(dev))
    ign = p["labels"] == -100
    assert np.array_equal(got2["dX"][ign], x0[ign].astype(np.float64))
    assert rel_fro(got2["dX"] - x0, ref["dX"]) <= TOL_GRAD
    assert rel_fro(got2["dgamma"] - g0, ref["dgamma"]) <= TOL_GRAD


def test_rmsnorm_prologue_ignored_rows_never_read(dev):
    """NaN planted in the ignored rows of X leaves every output bit-identical (reading R14)."""
    p = workload.make_problem(700, 128, 3000, seed=8, ignore="bern40")
    X, g = workload.make_rmsnorm_inputs(8, 700, 128)
    a = _run(dev, X, g, p["W"], p["labels"])
    Xn = X.copy()
    Xn[p["labels"] == -100] = 0x7FC0
    b = _run(dev, Xn, g, p["W"], p["labels"])
    for k in ("dX", "dgamma", "dW", "lse"):
        assert np.array_equal(a[k], b[k], equal_nan=False), k
    assert a["loss"] == b["loss"]


def test_rmsnorm_prologue_all_ignored(dev):
    p = workload.make_problem(300, 128, 3000, seed=2, ignore="all")
    X, g = workload.make_rmsnorm_inputs(2, 300, 128)
    got = _run(dev, X, g, p["W"], p["labels"])
    assert got["loss"] == 0.0 and got["n_valid"] == 0
    assert np.all(got["dX"] == 0) and np.all(got["dgamma"] == 0) and np.all(got["dW"] == 0)


def test_rmsnorm_prologue_deterministic(dev):
    p = workload.make_problem(1000, 896, 20000, seed=4, ignore="bern40")
    X, g = workload.make_rmsnorm_inputs(4, 1000, 896)
    a = _run(dev, X, g, p["W"], p["labels"])
    b = _run(dev, X, g, p["W"], p["labels"])
    for k in ("dX", "dgamma", "dW", "lse"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("eps_ls,lam,reduction", [(0.1, 1e-4, "mean"), (0.0, 1e-4, "sum")])
def test_rmsnorm_prologue_with_regularised_loss(dev, eps_ls, lam, reduction):
    """The prologue composes with label smoothing / z-loss and the sum reduction (the
    RMSNorm backward consumes whatever dH the CE path produced)."""
    import torch
    import paper_2601_02609_b200 as cce
    p = workload.make_problem(700, 128, 3000, seed=17, ignore="bern40")
    X, g = workload.make_rmsnorm_inputs(17, 700, 128)
    ref = oracle.cce_rmsnorm(X, g, p["W"], p["labels"], eps=EPS, label_smoothing=eps_ls, z_loss=lam,
                             reduction=reduction)
    Xt, gt, Wt = _t(X, dev), _t(g, dev), _t(p["W"], dev)
    yt = torch.from_numpy(p["labels"]).to(dev)
    h = cce.CCEHandle(vocab_total=3000, label_smoothing=eps_ls, z_loss=lam, reduction=reduction)
    loss, lse, nv = h.forward_rmsnorm(Xt, gt, EPS, Wt, yt)
    dX, dg, dW = torch.empty_like(Xt), torch.empty_like(gt), torch.empty_like(Wt)
    h.backward_rmsnorm(torch.ones((), dtype=torch.float32, device=dev), dX, dg, dW)
    torch.cuda.synchronize()
    h.close()
    assert abs(float(loss.item()) - float(ref["loss"])) <= TOL_LOSS * max(1.0, abs(float(ref["loss"])) * 1e-3)
    assert rel_fro(bf16_to_f64(dX), ref["dX"]) <= TOL_GRAD
    assert rel_fro(bf16_to_f64(dg), ref["dgamma"]) <= TOL_GRAD
    assert rel_fro(bf16_to_f64(dW), ref["dW"]) <= TOL_GRAD
