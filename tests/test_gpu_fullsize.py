"""Full-size parity at the bench configuration (Qwen2.5-0.5B head: N=8192, D=896,
V=151936, 40% packed padding, seed 42), in the launch configuration bench.py times.

The oracle cannot afford the whole fp64 problem on the test box, so:
  * every valid row's LSE and the loss are compared with the ORACLE's per-row LSE
    stored in tests/golden/qwen05b_seed42.npz (written by scripts/make_golden.py,
    which calls only oracle/ and workload/; content hashes of H and W guard against
    generator drift);
  * dH rows and dW rows are compared on samples the oracle computes one by one;
  * properties that hold at any size are checked on the whole output."""
import hashlib
import os

import numpy as np
import pytest

import oracle
import workload
from cce_testutil import TOL_GRAD, TOL_LOSS, TOL_LSE, bf16_to_f64, rel_fro, to_dev

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "qwen05b_seed42.npz")


@pytest.fixture(scope="module")
def full():
    import torch
    import __graft_entry__
    import paper_2601_02609_b200 as cce
    __graft_entry__.build()
    if not os.path.exists(GOLD):
        pytest.skip("golden file missing (scripts/make_golden.py)")
    g = np.load(GOLD)
    p = workload.make_config("qwen05b", seed=42)
    assert hashlib.sha256(p["H"].tobytes()).hexdigest() == str(g["H_sha256"]), "input generator drift (H)"
    assert hashlib.sha256(p["W"].tobytes()).hexdigest() == str(g["W_sha256"]), "input generator drift (W)"
    assert np.array_equal(p["labels"], g["labels"])
    dev = torch.device("cuda:0")
    H, W, y = to_dev(p, dev)
    h = cce.CCEHandle(vocab_total=W.shape[0])
    outs = []
    for _ in range(2):
        loss, lse, nv = h.forward(H, W, y)
        dH = torch.empty(H.shape, dtype=torch.bfloat16, device=dev)
        dW = torch.empty(W.shape, dtype=torch.bfloat16, device=dev)
        h.backward(torch.ones((), dtype=torch.float32, device=dev), dH, dW)
        torch.cuda.synchronize()
        outs.append({"loss": loss.item(), "lse": lse.cpu().numpy(), "n_valid": int(nv.item()),
                     "dH": dH.view(torch.int16).cpu().numpy(), "dW": dW.view(torch.int16).cpu().numpy()})
    h.close()
    return p, g, outs


def test_counts_masks_loss_and_every_lse(full):
    p, g, outs = full
    o = outs[0]
    valid = p["labels"] != -100
    assert o["n_valid"] == int(valid.sum()) == len(g["valid_rows"]) == 4915
    ref_loss = float(np.mean(g["lse"] - g["zy"]))
    assert abs(o["loss"] - ref_loss) <= TOL_LOSS
    rel = np.abs(o["lse"][valid] - g["lse"]) / np.maximum(np.abs(g["lse"]), 1.0)
    assert rel.max() <= TOL_LSE, rel.max()
    assert np.all(o["lse"][~valid].view(np.int32) == 0)
    assert np.all(o["dH"][~valid] == 0)


def test_deterministic_bits(full):
    _, _, outs = full
    a, b = outs
    assert a["loss"] == b["loss"]
    assert np.array_equal(a["lse"].view(np.int32), b["lse"].view(np.int32))
    assert np.array_equal(a["dH"], b["dH"]) and np.array_equal(a["dW"], b["dW"])


def test_sampled_dH_rows(full):
    p, g, outs = full
    rows = g["valid_rows"]
    pick = np.unique(np.concatenate([rows[:4], rows[-4:], rows[np.linspace(0, len(rows) - 1, 16).astype(int)]]))
    s = 1.0 / len(rows)
    _, _, dH_ref = oracle.rows(p["H"], p["W"], p["labels"], pick, scale=s)
    got = (outs[0]["dH"][pick].astype(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    assert rel_fro(got, dH_ref) <= TOL_GRAD


def test_sampled_dW_rows(full):
    p, g, outs = full
    V = p["W"].shape[0]
    lab = p["labels"][p["labels"] != -100]
    common = np.bincount(lab, minlength=V).argsort()[-6:]      # most frequent targets (Zipf head)
    pick = np.unique(np.concatenate([[0, 1, 2, 8191, 8192, 8193, 65535, 65536, V - 257, V - 256, V - 1],
                                     common, np.random.default_rng(0).choice(V, 10, replace=False)]))
    lse_all = np.zeros(len(p["labels"]))
    lse_all[g["valid_rows"]] = g["lse"]
    ref = oracle.dW_rows(p["H"], p["W"], p["labels"], lse_all, 1.0 / len(g["valid_rows"]), pick)
    got = (outs[0]["dW"][pick].astype(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    assert rel_fro(got, ref) <= TOL_GRAD


def test_full_size_invariants(full):
    """sum_v dW[v,:] = 0 (rows of dlogits sum to 0) within the bf16
    rounding budget of G (1.9e-3 simulated); finite, non-zero grads."""
    _, _, outs = full
    dW = (outs[0]["dW"].astype(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    assert np.isfinite(dW).all() and np.abs(dW).sum() > 0
    assert np.linalg.norm(dW.sum(0)) <= 1e-2 * np.linalg.norm(dW)
    dH = (outs[0]["dH"].astype(np.uint16).astype(np.uint32) << 16).view(np.float32)
    assert np.isfinite(dH).all()


def test_memory_no_nxv_buffer():
    """SURVEY 8(d) memory report at the bench configuration: the library allocates nothing
    (caller-owned workspace: device free memory and the torch allocator peak do not move
    during a forward + backward) and no buffer is N x V sized (the workspace, the largest
    buffer, is compared with one bf16 copy of the logits, N V 2 bytes = 2.49 GB)."""
    import torch
    import __graft_entry__
    import paper_2601_02609_b200 as cce
    __graft_entry__.build()
    dev = torch.device("cuda:0")
    c = workload.CONFIGS["qwen05b"]
    p = workload.make_config("qwen05b", seed=42)
    H, W, y = to_dev(p, dev)
    h = cce.CCEHandle(vocab_total=c.V)
    ws = h.workspace(c.N, c.D, c.V, dev)
    assert ws.numel() < c.N * c.V * 2 // 4
    dH = torch.empty_like(H)
    dW = torch.empty_like(W)
    one = torch.ones((), dtype=torch.float32, device=dev)
    h.forward(H, W, y)          # warm: the handle's small outputs are allocated here
    h.backward(one, dH, dW)
    loss = torch.empty((), dtype=torch.float32, device=dev)
    lse = torch.empty(c.N, dtype=torch.float32, device=dev)
    nvt = torch.empty((), dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info(dev)[0]
    torch.cuda.reset_peak_memory_stats(dev)
    a0 = torch.cuda.memory_allocated(dev)
    cce.cce_forward(h.h, H, W, y, loss, lse, nvt, ws)
    cce.cce_backward(h.h, one, dH, dW)
    torch.cuda.synchronize()
    assert torch.cuda.max_memory_allocated(dev) == a0
    assert torch.cuda.mem_get_info(dev)[0] == free0
    assert np.isfinite(loss.item())
    h.close()


def test_rmsnorm_prologue_full_size_sampled_rows():
    """The RMSNorm prologue at the bench configuration: per-row LSE
    and dX of sampled valid rows against the oracle (H = bf16(RMSNorm(X)) for all rows,
    then the row-local CE and RMSNorm backward of the picked rows), plus the whole-output
    properties (ignored rows of dX bit-zero, finite gradients)."""
    import torch
    import __graft_entry__
    import paper_2601_02609_b200 as cce
    __graft_entry__.build()
    dev = torch.device("cuda:0")
    c = workload.CONFIGS["qwen05b"]
    p = workload.make_config("qwen05b", seed=42)
    X, g = workload.make_rmsnorm_inputs(42, c.N, c.D)
    t = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).to(dev)  # noqa: E731
    Xt, gt, Wt = t(X), t(g), t(p["W"])
    y = torch.from_numpy(p["labels"]).to(dev)
    h = cce.CCEHandle(vocab_total=c.V)
    loss, lse, nv = h.forward_rmsnorm(Xt, gt, 1e-6, Wt, y)
    dX = torch.empty_like(Xt)
    dg = torch.empty_like(gt)
    dW = torch.empty_like(Wt)
    h.backward_rmsnorm(torch.ones((), dtype=torch.float32, device=dev), dX, dg, dW)
    torch.cuda.synchronize()
    h.close()
    valid = p["labels"] != -100
    rows = np.nonzero(valid)[0]
    pick = np.unique(np.concatenate([rows[:3], rows[-3:], rows[np.linspace(0, len(rows) - 1, 10).astype(int)]]))
    y_ref, rstd = oracle.rmsnorm_fwd(X, g, 1e-6)
    H_bits = oracle.to_bf16(y_ref)
    lse_ref, _, dH_ref = oracle.rows(H_bits, p["W"], p["labels"], pick, scale=1.0 / len(rows))
    got_lse = lse.cpu().numpy().astype(np.float64)[pick]
    assert np.max(np.abs(got_lse - lse_ref) / np.maximum(np.abs(lse_ref), 1.0)) <= TOL_LSE
    dX_ref, _ = oracle.rmsnorm_bwd(dH_ref, X[pick], g, rstd[pick])
    got = bf16_to_f64(dX)
    assert rel_fro(got[pick], dX_ref) <= TOL_GRAD
    assert np.all(dX.view(torch.int16).cpu().numpy()[~valid] == 0)
    assert np.isfinite(got).all() and np.isfinite(bf16_to_f64(dg)).all() and np.isfinite(loss.item())


def test_fused_adamw_full_size_sampled_rows():
    """The fused optimizer step at the bench configuration, in the
    default launch (pair kernel, W_out double buffer): sampled vocabulary rows of the new
    master weights / moments against oracle.dW_rows (golden LSE) fed to oracle.adamw_step,
    with warm moments (step 10)."""
    import torch
    import __graft_entry__
    import paper_2601_02609_b200 as cce
    __graft_entry__.build()
    if not os.path.exists(GOLD):
        pytest.skip("golden file missing (scripts/make_golden.py)")
    g = np.load(GOLD)
    dev = torch.device("cuda:0")
    p = workload.make_config("qwen05b", seed=42)
    H, W, y = to_dev(p, dev)
    V, D = W.shape
    lab = p["labels"][p["labels"] != -100]
    common = np.bincount(lab, minlength=V).argsort()[-4:]
    pick = np.unique(np.concatenate([[0, 8191, 8192, V - 1], common,
                                     np.random.default_rng(1).choice(V, 8, replace=False)]))
    lse_all = np.zeros(len(p["labels"]))
    lse_all[g["valid_rows"]] = g["lse"]
    dW_ref = oracle.dW_rows(p["H"], p["W"], p["labels"], lse_all, 1.0 / len(g["valid_rows"]), pick)
    gs = float(np.sqrt(np.mean(dW_ref * dW_ref)))
    m0, v0 = workload.make_adamw_state(5, (V, D), gs)
    master = W.float()
    m, v = torch.from_numpy(m0).to(dev), torch.from_numpy(v0).to(dev)
    Wo = torch.empty_like(W)
    h = cce.CCEHandle(vocab_total=V)
    h.forward(H, W, y)
    opt = cce.adamw_params(m, v, lr=1e-3, step=10, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1,
                           master=master, W_out=Wo)
    h.backward_adamw(torch.ones((), dtype=torch.float32, device=dev), torch.empty_like(H), opt)
    torch.cuda.synchronize()
    h.close()
    th0 = workload.bf16_bits_to_f32(p["W"][pick]).astype(np.float64)
    rth, rm, rv = oracle.adamw_step(th0, dW_ref, m0[pick], v0[pick], lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8,
                                    weight_decay=0.1, step=10)
    got_m = m.cpu().numpy()[pick].astype(np.float64)
    got_v = v.cpu().numpy()[pick].astype(np.float64)
    got_t = master.cpu().numpy()[pick].astype(np.float64)
    assert rel_fro(got_m, rm) <= TOL_GRAD
    assert rel_fro(got_v, rv) <= TOL_GRAD
    dec = th0 * (1 - 1e-3 * 0.1)
    assert rel_fro(got_t - dec, rth - dec) <= TOL_GRAD
    assert np.array_equal(Wo.view(torch.int16).cpu().numpy()[pick].view(np.uint16),
                          workload.f32_to_bf16_bits(master.cpu().numpy()[pick]))
