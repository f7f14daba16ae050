"""GPU parity of the fused optimizer step: AdamW applied in the
dW epilogue of the backward (cce_backward_adamw) and the standalone fused AdamW kernel
(cce_adamw_step), against the fp64 oracle: oracle.cce's dW fed to oracle.adamw_step
(Alg. Fused AdamW P:2003-2046, Def. AdamW).

Tolerances.  The GPU gradient is the fp32 accumulator of bf16 dlogits x bf16 H, so it
carries the same ~3e-3 relative Frobenius error as dW itself (north_star bar 1e-2);
m is linear in g and v quadratic, so both stay within 1e-2.  The parameter update
lr * m_hat / (sqrt(v_hat) + eps) is a smooth function of g when v is warm (v > 0 from
earlier steps), so the update (theta_new - theta_decayed) is held to the same 1e-2 relative
Frobenius bar.  At step 1 (m = v = 0) the update is lr * sign(g) for |g| >> eps, which a
1e-3 relative gradient error flips for gradients near 0: there the test checks the sign
on every element whose reference gradient is resolved (|g| > 5% of the rms) and the
magnitude lr everywhere.  The standalone kernel gets the gradient exactly, so it is held
element-wise to fp32 rounding (rtol 1e-5)."""
import numpy as np
import pytest

import oracle
import workload
from cce_testutil import TOL_GRAD, bf16_to_f64, rel_fro, to_dev

pytestmark = pytest.mark.gpu

LR, B1, B2, EPS, WD = 1e-2, 0.9, 0.95, 1e-8, 0.1


@pytest.fixture(scope="module")
def dev():
    import torch
    import __graft_entry__
    __graft_entry__.build()
    return torch.device("cuda:0")


def _oracle_grad(p, dloss=1.0):
    return oracle.cce(p["H"], p["W"], p["labels"], dloss=dloss)


def _run_fused(p, dev, step, m0, v0, use_master=True, clip=None, grad_in=None, dloss=1.0, w_out=False):
    import torch
    import paper_2601_02609_b200 as cce
    H, W, y = to_dev(p, dev)
    W = W.clone()
    W_in = W.clone()
    V, D = W.shape
    Wo = torch.full_like(W, float("nan")) if w_out else None
    master = W.float().clone() if use_master else None
    m = torch.from_numpy(m0).to(dev)
    v = torch.from_numpy(v0).to(dev)
    clip_t = None if clip is None else torch.tensor(clip, dtype=torch.float32, device=dev)
    gin = None if grad_in is None else torch.from_numpy(grad_in.astype(np.float32)).to(dev)
    h = cce.CCEHandle(vocab_total=V)
    loss, lse, nv = h.forward(H, W, y)
    dH = torch.empty_like(H)
    dl = torch.tensor(dloss, dtype=torch.float32, device=dev)
    opt = cce.adamw_params(m, v, lr=LR, step=step, beta1=B1, beta2=B2, eps=EPS, weight_decay=WD, clip_coef=clip_t,
                           master=master, grad_in=gin, W_out=Wo)
    h.backward_adamw(dl, dH, opt)
    torch.cuda.synchronize()
    h.close()
    if w_out:
        assert torch.equal(W.view(torch.int16), W_in.view(torch.int16))   # the forward's W is only read
        W = Wo
    out = {"W": bf16_to_f64(W), "W_bits": W.view(torch.int16).cpu().numpy(), "m": m.cpu().numpy().astype(np.float64),
           "v": v.cpu().numpy().astype(np.float64), "dH": bf16_to_f64(dH), "loss": float(loss.item())}
    if master is not None:
        out["master"] = master.cpu().numpy().astype(np.float64)
        out["master_f32"] = master.cpu().numpy()
    return out


def _theta0(p):
    return workload.bf16_bits_to_f32(p["W"]).astype(np.float64)


def _check_update(got_theta, ref_theta, theta0, tol=TOL_GRAD):
    decayed = theta0 * (1.0 - LR * WD)
    e = rel_fro(got_theta - decayed, ref_theta - decayed)
    assert e <= tol, ("update", e)


@pytest.mark.parametrize("w_out", [False, True], ids=["in_place", "W_out"])
@pytest.mark.parametrize("N,D,V,ign", [
    (64, 64, 1000, "bern10"),        # configs[0] shape
    (700, 128, 3000, "bern40"),      # ragged rows / vocabulary
    (1000, 128, 41000, "bern40"),    # 6 chunks: every chunk's dW tiles wait on that chunk's dH tiles
    (384, 896, 9000, "bern40"),      # Qwen hidden size (256,256,256,128 hidden tiles), 2 chunks
])
def test_fused_adamw_warm_state(dev, N, D, V, ign, w_out):
    p = workload.make_problem(N, D, V, seed=N + V + 7, ignore=ign)
    ref = _oracle_grad(p)
    g = ref["dW"]
    gs = float(np.sqrt(np.mean(g * g)))
    m0, v0 = workload.make_adamw_state(N + V, g.shape, gs)
    th0 = _theta0(p)
    rth, rm, rv = oracle.adamw_step(th0, g, m0, v0, lr=LR, beta1=B1, beta2=B2, eps=EPS, weight_decay=WD, step=10)
    got = _run_fused(p, dev, 10, m0, v0, w_out=w_out)
    # the loss / dH of the same backward are unchanged by the fused step
    assert abs(got["loss"] - ref["loss"]) <= 2e-3
    assert rel_fro(got["dH"], ref["dH"]) <= TOL_GRAD
    assert rel_fro(got["m"], rm) <= TOL_GRAD
    assert rel_fro(got["v"], rv) <= TOL_GRAD
    _check_update(got["master"], rth, th0)
    # the bf16 weights are exactly the RNE rounding of the fp32 master
    assert np.array_equal(got["W_bits"].view(np.uint16), workload.f32_to_bf16_bits(got["master_f32"]))


def test_fused_adamw_step1_sign(dev):
    """Step 1, zero moments: update = lr * g / (|g| + eps) = lr * sign(g)."""
    p = workload.make_problem(700, 128, 3000, seed=5, ignore="bern40")
    ref = _oracle_grad(p)
    g = ref["dW"]
    z = np.zeros(g.shape, np.float32)
    got = _run_fused(p, dev, 1, z, z)
    th0 = _theta0(p)
    upd = got["master"] - th0 * (1.0 - LR * WD)
    # the dW scale varies by orders of magnitude between vocabulary rows (rows that are some
    # token's target carry the -1 of the one-hot): resolve against each row's own rms
    row_rms = np.sqrt(np.mean(g * g, axis=1, keepdims=True))
    resolved = np.abs(g) > 0.05 * row_rms
    assert resolved.mean() > 0.9
    assert np.all(np.sign(upd[resolved]) == -np.sign(g[resolved]))
    # |update| = lr |g| / (|g| + eps) on the resolved elements (fp32 rounding of theta aside)
    want = LR * np.abs(g[resolved]) / (np.abs(g[resolved]) + EPS)
    assert np.max(np.abs(np.abs(upd[resolved]) - want)) <= 1e-3 * LR
    assert np.all(np.abs(upd) <= LR * (1 + 1e-5))


def test_fused_adamw_clip_and_accumulated_grad(dev):
    """clip_coef (device scalar) and a gradient from earlier micro-batches
     enter as g = (grad_in + dW) * clip."""
    p = workload.make_problem(1000, 128, 41000, seed=11, ignore="bern40")
    ref = _oracle_grad(p)
    g = ref["dW"]
    gs = float(np.sqrt(np.mean(g * g)))
    gin = workload.make_adamw_state(3, g.shape, gs)[0].astype(np.float64)   # any seeded fp32 field
    m0, v0 = workload.make_adamw_state(4, g.shape, gs)
    th0 = _theta0(p)
    rth, rm, rv = oracle.adamw_step(th0, g + gin, m0, v0, lr=LR, beta1=B1, beta2=B2, eps=EPS, weight_decay=WD,
                                    clip_coef=0.5, step=3)
    got = _run_fused(p, dev, 3, m0, v0, clip=0.5, grad_in=gin)
    assert rel_fro(got["m"], rm) <= TOL_GRAD
    assert rel_fro(got["v"], rv) <= TOL_GRAD
    _check_update(got["master"], rth, th0)


@pytest.mark.parametrize("w_out", [False, True], ids=["in_place", "W_out"])
def test_fused_adamw_bf16_weights_only(dev, w_out):
    """No master copy: theta is the bf16 W itself, updated in fp32 and rounded back (RNE)."""
    p = workload.make_problem(700, 128, 3000, seed=9, ignore="bern40")
    ref = _oracle_grad(p)
    g = ref["dW"]
    gs = float(np.sqrt(np.mean(g * g)))
    m0, v0 = workload.make_adamw_state(9, g.shape, gs)
    th0 = _theta0(p)
    rth, rm, rv = oracle.adamw_step(th0, g, m0, v0, lr=LR, beta1=B1, beta2=B2, eps=EPS, weight_decay=WD, step=10)
    got = _run_fused(p, dev, 10, m0, v0, use_master=False, w_out=w_out)
    assert rel_fro(got["m"], rm) <= TOL_GRAD
    assert rel_fro(got["v"], rv) <= TOL_GRAD
    # bf16 result within one bf16 ulp of the exact update plus the gradient-driven error
    ulp = np.abs(rth) * 2.0 ** -7
    err = np.abs(got["W"] - rth)
    assert np.mean(err <= ulp + 1e-3 * LR) > 0.99
    assert rel_fro(got["W"] - th0, rth - th0) <= 5e-2   # update after bf16 rounding (ulp ~ 1e-4 vs lr 1e-2)


def test_fused_adamw_all_ignored(dev):
    """n_valid = 0: zero gradient, the step still decays theta and the moments (Def. AdamW)."""
    p = workload.make_problem(300, 128, 3000, seed=2, ignore="all")
    g = np.zeros((3000, 128))
    m0, v0 = workload.make_adamw_state(2, g.shape, 1e-4)
    th0 = _theta0(p)
    rth, rm, rv = oracle.adamw_step(th0, g, m0, v0, lr=LR, beta1=B1, beta2=B2, eps=EPS, weight_decay=WD, step=4)
    got = _run_fused(p, dev, 4, m0, v0)
    assert np.all(got["dH"] == 0)
    np.testing.assert_allclose(got["m"], rm, rtol=1e-5, atol=1e-12)
    np.testing.assert_allclose(got["v"], rv, rtol=1e-5, atol=1e-16)
    np.testing.assert_allclose(got["master"], rth, rtol=1e-5, atol=1e-7)


def test_fused_equals_unfused(dev):
    """The fused epilogue and the unfused pair (fp32 dW from cce_backward, then the standalone
    cce_adamw_step) run the same fp32 arithmetic on the same accumulator: bit-identical."""
    import torch
    import paper_2601_02609_b200 as cce
    p = workload.make_problem(1000, 896, 20000, seed=21, ignore="bern40")
    H, W, y = to_dev(p, dev)
    V, D = W.shape
    gs = 1e-5
    m0, v0 = workload.make_adamw_state(21, (V, D), gs)
    res = []
    for fused in ("in_place", "W_out", False):
        Wc = W.clone()
        master = Wc.float().clone()
        m, v = torch.from_numpy(m0).to(dev), torch.from_numpy(v0).to(dev)
        opt = cce.adamw_params(m, v, lr=LR, step=7, beta1=B1, beta2=B2, eps=EPS, weight_decay=WD, master=master)
        h = cce.CCEHandle(vocab_total=V, flags=0 if fused else cce.FLAG_GRAD_FP32)
        h.forward(H, Wc, y)
        dl = torch.ones((), dtype=torch.float32, device=dev)
        if fused == "W_out":
            Wo = torch.empty_like(Wc)
            opt = cce.adamw_params(m, v, lr=LR, step=7, beta1=B1, beta2=B2, eps=EPS, weight_decay=WD, master=master,
                                   W_out=Wo)
            h.backward_adamw(dl, torch.empty_like(H), opt)
            Wc = Wo
        elif fused:
            h.backward_adamw(dl, torch.empty_like(H), opt)
        else:
            dW = torch.empty((V, D), dtype=torch.float32, device=dev)
            h.backward(dl, torch.empty(H.shape, dtype=torch.float32, device=dev), dW)
            cce.cce_adamw_step(opt, dW, V * D, Wc)
        torch.cuda.synchronize()
        h.close()
        res.append((Wc.view(torch.int16).cpu(), master.cpu(), m.cpu(), v.cpu()))
    for r in res[1:]:
        for a, b in zip(res[0], r):
            assert torch.equal(a, b)


@pytest.mark.parametrize("n,grad_dtype,use_master", [(1 << 20, "bf16", True), ((1 << 20) + 5, "f32", True),
                                                      (4099, "bf16", False), (7, "f32", True)])
def test_standalone_adamw(dev, n, grad_dtype, use_master):
    """cce_adamw_step vs oracle_adamw_step element-wise (exact gradient input; fp32 rounding only)."""
    import torch
    import paper_2601_02609_b200 as cce
    th_bits = workload.normal_bf16(n, 1, 1, n, 0.03)[0]
    th0 = workload.bf16_bits_to_f32(th_bits)
    g32 = (workload.normal_f64(n, 2, 0, n) * 1e-3).astype(np.float32)
    if grad_dtype == "bf16":
        g_bits = workload.f32_to_bf16_bits(g32)
        g_np = workload.bf16_bits_to_f32(g_bits).astype(np.float64)
        g_t = torch.from_numpy(g_bits.view(np.int16)).view(torch.bfloat16).to(dev)
    else:
        g_np = g32.astype(np.float64)
        g_t = torch.from_numpy(g32).to(dev)
    m0, v0 = workload.make_adamw_state(n, (n,), 1e-3)
    W = torch.from_numpy(th_bits.view(np.int16)).view(torch.bfloat16).to(dev)
    master = torch.from_numpy(th0.copy()).to(dev) if use_master else None
    m, v = torch.from_numpy(m0).to(dev), torch.from_numpy(v0).to(dev)
    clip = torch.tensor(0.8, dtype=torch.float32, device=dev)
    opt = cce.adamw_params(m, v, lr=1e-3, step=5, beta1=B1, beta2=0.999, eps=EPS, weight_decay=WD, clip_coef=clip,
                           master=master)
    cce.cce_adamw_step(opt, g_t, n, W)
    torch.cuda.synchronize()
    rth, rm, rv = oracle.adamw_step(th0.astype(np.float64), g_np, m0, v0, lr=1e-3, beta1=B1, beta2=0.999, eps=EPS,
                                    weight_decay=WD, clip_coef=0.8, step=5)
    # atol: a few fp32 ulps of the operands (m ~ 1e-3, v ~ 1e-6) where b1 m + (1 - b1) g cancels
    np.testing.assert_allclose(m.cpu().numpy(), rm, rtol=1e-5, atol=1e-9)
    np.testing.assert_allclose(v.cpu().numpy(), rv, rtol=1e-5, atol=1e-12)
    if use_master:
        np.testing.assert_allclose(master.cpu().numpy(), rth, rtol=1e-5, atol=1e-8)
        assert np.array_equal(W.view(torch.int16).cpu().numpy().view(np.uint16),
                              workload.f32_to_bf16_bits(master.cpu().numpy()))
    else:
        # theta read from and rounded back to bf16: within one bf16 rounding of the exact result
        got = bf16_to_f64(W)
        assert np.all(np.abs(got - rth) <= np.abs(rth) * 2.0 ** -8 + 1e-12)


def test_fused_adamw_with_regularised_loss(dev):
    """The fused step consumes the regularised dW (label smoothing + z-loss, NEXT #1)."""
    import torch
    import paper_2601_02609_b200 as cce
    p = workload.make_problem(1000, 128, 41000, seed=23, ignore="bern40")
    ref = oracle.cce(p["H"], p["W"], p["labels"], label_smoothing=0.1, z_loss=1e-4)
    g = ref["dW"]
    gs = float(np.sqrt(np.mean(g * g)))
    m0, v0 = workload.make_adamw_state(23, g.shape, gs)
    th0 = _theta0(p)
    rth, rm, rv = oracle.adamw_step(th0, g, m0, v0, lr=LR, beta1=B1, beta2=B2, eps=EPS, weight_decay=WD, step=6)
    H, W, y = to_dev(p, dev)
    master = W.float()
    m, v = torch.from_numpy(m0).to(dev), torch.from_numpy(v0).to(dev)
    Wo = torch.empty_like(W)
    h = cce.CCEHandle(vocab_total=W.shape[0], label_smoothing=0.1, z_loss=1e-4)
    loss, _, _ = h.forward(H, W, y)
    opt = cce.adamw_params(m, v, lr=LR, step=6, beta1=B1, beta2=B2, eps=EPS, weight_decay=WD, master=master, W_out=Wo)
    h.backward_adamw(torch.ones((), dtype=torch.float32, device=dev), torch.empty_like(H), opt)
    torch.cuda.synchronize()
    h.close()
    assert abs(float(loss.item()) - ref["loss"]) <= 2e-3
    assert rel_fro(m.cpu().numpy().astype(np.float64), rm) <= TOL_GRAD
    assert rel_fro(v.cpu().numpy().astype(np.float64), rv) <= TOL_GRAD
    _check_update(master.cpu().numpy().astype(np.float64), rth, th0)
