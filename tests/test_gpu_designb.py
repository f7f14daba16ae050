"""Design B (CCE_FLAG_DESIGN_B): the dH numerator U = E_p[W] - W_y
accumulated in the forward (target excluded, online-rescaled O' like the FlashAttention output,
P:1220-1226) and the backward's dlogits kept in shared memory.  Same oracle and tolerances as
the default path, plus the per-row check on confident tokens that design B's target exclusion
exists for, and cases that force the lazy rescale of O' in the middle of a sweep."""
import os

import numpy as np
import pytest

import oracle
import workload
from cce_testutil import TOL_GRAD, assert_parity, rel_fro, run_gpu, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import torch
    import __graft_entry__
    __graft_entry__.build()
    return torch.device("cuda:0")


def _flags(extra=0):
    import paper_2601_02609_b200 as cce
    return cce.FLAG_DESIGN_B | extra


def _check(p, dev, dloss=1.0, flags=0, reduction="mean"):
    H, W, y = to_dev(p, dev)
    got = run_gpu(H, W, y, dloss=dloss, flags=_flags(flags), reduction=reduction)
    ref = oracle.cce(p["H"], p["W"], p["labels"], dloss=dloss, reduction=reduction)
    assert_parity(got, ref, p["labels"])
    return got, ref


@pytest.mark.parametrize("seed", [0, 42])
def test_tiny_config(dev, seed):
    _check(workload.make_config("tiny", seed=seed), dev)


@pytest.mark.parametrize("N,D,V,ign", [
    (700, 128, 3000, "bern40"),      # ragged token tiles (64) and vocabulary steps (128)
    (129, 64, 257, "none"),          # one vocabulary row past a step; 3 token tiles
    (384, 896, 9000, "bern40"),      # Qwen hidden size: 7 hidden blocks, 512 TMEM columns
    (1000, 832, 41000, "bern40"),    # D = 13 x 64: the last hidden block half empty (TMA zero fill)
    (300, 192, 20000, "bern30"),     # several partial segments per token tile across CTAs
])
def test_shapes(dev, N, D, V, ign):
    _check(workload.make_problem(N, D, V, seed=N + V + 7, ignore=ign), dev)


@pytest.mark.parametrize("regime", ["peaked", "zero"])
def test_regimes(dev, regime):
    _check(workload.make_problem(300, 256, 5000, seed=11, ignore="bern40", regime=regime), dev)


def test_confident_rows_per_row_dh(dev):
    """with p_y -> 1 - 1e-6 ("extreme" regime) dH_n = s (E_p[W] - W_y) is a tiny
    difference; design B forms U = (O' - d_nt W_y) / d with the target excluded from the bf16
    P', so every row -- not only the Frobenius norm -- stays accurate."""
    p = workload.make_problem(300, 256, 5000, seed=12, ignore="bern40", regime="extreme")
    got, ref = _check(p, dev)
    valid = np.nonzero(p["labels"] != -100)[0]
    errs = [rel_fro(got["dH"][n], ref["dH"][n]) for n in valid]
    assert max(errs) <= 2e-2, max(errs)


def test_midsweep_rescale(dev):
    """Logits jump by +40 (58 in log2 units, past the 2^16 headroom) half way through the
    vocabulary: the reference maxima move in the middle of every unit's sweep, so O' in TMEM
    and d_nt are rescaled before later GEMM2 steps (the lazy-rescale path)."""
    p = workload.make_problem(256, 256, 6000, seed=13, ignore="bern40")
    H = p["H"].copy(); W = p["W"].copy()
    H[:, -1] = 0x3F80                       # 1.0
    W[:, -1] = 0
    W[3000:, -1] = 0x4220                   # 40.0 for the second half of the vocabulary
    q = {"H": H, "W": W, "labels": p["labels"]}
    _check(q, dev)


def test_bigshift(dev):
    p = workload.make_problem(256, 896, 3000, seed=10, ignore="bern40")
    H = p["H"].copy(); W = p["W"].copy()
    H[:, -1] = 0x3F80
    W[:, -1] = 0x42A0                       # every logit + 80
    q = {"H": H, "W": W, "labels": p["labels"]}
    H_, W_, y_ = to_dev(q, dev)
    got = run_gpu(H_, W_, y_, flags=_flags())
    ref = oracle.cce(q["H"], q["W"], q["labels"])
    assert_parity(got, ref, q["labels"], check_grads=False)
    assert rel_fro(got["dH"][:, :-1], ref["dH"][:, :-1]) <= TOL_GRAD
    assert rel_fro(got["dW"], ref["dW"]) <= TOL_GRAD


@pytest.mark.parametrize("reduction", ["sum", "none"])
def test_reductions(dev, reduction):
    p = workload.make_problem(500, 256, 7000, seed=21, ignore="bern40")
    dloss = (np.random.default_rng(3).standard_normal(500).astype(np.float32).astype(np.float64) / 500
             if reduction == "none" else 0.5 / 300)
    _check(p, dev, dloss=dloss, reduction=reduction)


@pytest.mark.parametrize("extra", [64, 192], ids=["fp32", "accumulate_fp32"])
def test_grad_modes(dev, extra):
    import torch
    p = workload.make_problem(400, 192, 5000, seed=22, ignore="bern40")
    H, W, y = to_dev(p, dev)
    g = torch.Generator(device="cpu").manual_seed(5)
    dH0 = (torch.randn(H.shape, generator=g) * 1e-3).float().to(dev)
    dW0 = (torch.randn(W.shape, generator=g) * 1e-3).float().to(dev)
    got = run_gpu(H, W, y, flags=_flags(extra), dH_init=dH0.clone(), dW_init=dW0.clone())
    ref = oracle.cce(p["H"], p["W"], p["labels"])
    acc = bool(extra & 128)
    dH = got["dH"] - (dH0.double().cpu().numpy() if acc else 0.0)
    dW = got["dW"] - (dW0.double().cpu().numpy() if acc else 0.0)
    assert rel_fro(dH, ref["dH"]) <= TOL_GRAD
    assert rel_fro(dW, ref["dW"]) <= TOL_GRAD


def test_all_ignored_and_single_valid(dev):
    p = workload.make_problem(130, 64, 1500, seed=7, ignore="all")
    _check(p, dev)
    p["labels"][77] = 1234
    _check(p, dev)


def test_nan_in_ignored_rows_does_not_leak(dev):
    p = workload.make_problem(300, 128, 2500, seed=8, ignore="bern40")
    H, W, y = to_dev(p, dev)
    a = run_gpu(H, W, y, flags=_flags())
    Hn = p["H"].copy()
    Hn[p["labels"] == -100] = 0x7FC0
    H2, _, _ = to_dev({"H": Hn, "W": p["W"], "labels": p["labels"]}, dev)
    b = run_gpu(H2, W, y, flags=_flags())
    assert a["loss"] == b["loss"]
    for k in ("lse_bits", "dH_bits", "dW_bits"):
        assert np.array_equal(a[k], b[k]), k


def test_deterministic_and_agrees_with_default_path(dev):
    p = workload.make_problem(500, 256, 9000, seed=9, ignore="bern40")
    H, W, y = to_dev(p, dev)
    a = run_gpu(H, W, y, flags=_flags())
    b = run_gpu(H, W, y, flags=_flags())
    for k in ("lse_bits", "dH_bits", "dW_bits"):
        assert np.array_equal(a[k], b[k]), k
    c = run_gpu(H, W, y)
    assert abs(a["loss"] - c["loss"]) <= 1e-4
    assert rel_fro(a["dH"], c["dH"]) <= TOL_GRAD and rel_fro(a["dW"], c["dW"]) <= TOL_GRAD


def test_unsupported_configurations(dev):
    import torch
    import paper_2601_02609_b200 as cce
    with pytest.raises(cce.CCEError) as ei:
        cce.CCEHandle(vocab_total=500, flags=_flags(), label_smoothing=0.1)
    assert ei.value.status == 2
    p = workload.make_problem(64, 1024, 500, seed=1)
    H, W, y = to_dev(p, dev)
    h = cce.CCEHandle(vocab_total=500, flags=_flags())
    with pytest.raises(cce.CCEError) as ei:
        h.forward(H, W, y)                   # D = 1024 > 896
    assert ei.value.status == 2
    h.close()


def test_full_size_qwen05b(dev):
    """configs[1] at full size through design B: every valid row's LSE and the loss against
    the oracle golden, sampled dH rows (oracle.rows) and dW rows (oracle.dW_rows)."""
    import torch
    import paper_2601_02609_b200 as cce
    p = workload.make_config("qwen05b", seed=42)
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "qwen05b_seed42.npz"))
    H, W, y = to_dev(p, dev)
    h = cce.CCEHandle(vocab_total=W.shape[0], flags=_flags())
    loss, lse, nv = h.forward(H, W, y)
    dH = torch.empty(H.shape, dtype=torch.bfloat16, device=dev)
    dW = torch.empty(W.shape, dtype=torch.bfloat16, device=dev)
    h.backward(torch.ones((), dtype=torch.float32, device=dev), dH, dW)
    torch.cuda.synchronize()
    rows = g["valid_rows"].astype(np.int64)
    assert int(nv.item()) == len(rows)
    lse_g = lse.double().cpu().numpy()
    assert (np.abs(lse_g[rows] - g["lse"]) / np.maximum(np.abs(g["lse"]), 1.0)).max() <= 1e-3
    assert abs(float(loss.item()) - float(np.mean(g["lse"] - g["zy"]))) <= 2e-3
    s = 1.0 / len(rows)
    pick = rows[np.linspace(0, len(rows) - 1, 12).astype(int)]
    _, _, dH_ref = oracle.rows(p["H"], p["W"], p["labels"], pick, scale=s)
    assert rel_fro(dH[torch.from_numpy(pick).to(dev)].double().cpu().numpy(), dH_ref) <= TOL_GRAD
    lse_full = np.zeros(len(p["labels"]))
    lse_full[rows] = g["lse"]
    vr = np.array([0, 1, 17, 1000, 50000, 151935])
    dW_ref = oracle.dW_rows(p["H"], p["W"], p["labels"], lse_full, s, vr)
    assert rel_fro(dW[torch.from_numpy(vr).to(dev)].double().cpu().numpy(), dW_ref) <= TOL_GRAD
    h.close()
