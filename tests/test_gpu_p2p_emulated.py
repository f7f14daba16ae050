"""The vocabulary-sharded exchange over peer memory (CCE_FLAG_P2P_COMBINE, SURVEY 8(f)
NEXT #4; rows a9 / a10) on ONE GPU: `world` ranks as handles of one process, attached with
cce_p2p_attach_group.  The forward's merge kernel pushes each rank's stats into every rank's
all-ranks array (a9 fused into the kernel that produces them); the backward runs as ONE
launch in which each rank's queue owns its own CTA pairs, so the RED items reduce every dH
tile across the co-resident rank groups (a10 fused into the backward kernel) -- the same
kernels and flags as across GPUs, without time-slicing ranks that wait on one another.

Every rank must match the unsharded fp64 oracle (north_star tolerances) and every other rank
bit for bit, over consecutive steps (per-step flag epochs, double-buffered stats)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2601_02609_b200 as cce
import workload
from cce_testutil import TOL_GRAD, TOL_LOSS, TOL_LSE, rel_fro, to_dev

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _bf(b):
    return (b.astype(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _group(V, world, N, D, W, **kw):
    hs, wss, Ws = [], [], []
    for r in range(world):
        lo, hi = cce.shard_range(V, r, world)
        h = cce.CCEHandle(vocab_total=V, vocab_offset=lo, rank=r, world=world, flags=cce.FLAG_P2P_COMBINE, **kw)
        hs.append(h)
        wss.append(h.workspace(N, D, hi - lo, DEV))
        Ws.append(W[lo:hi].contiguous())
    cce.cce_p2p_attach_group([h.h for h in hs], wss, N, D)
    return hs, Ws


def _step(hs, Ws, H, y, dloss=None):
    one = torch.ones((), dtype=torch.float32, device=DEV) if dloss is None else dloss
    fw = [h.forward(H, Wr, y) for h, Wr in zip(hs, Ws)]
    dHs = [torch.empty_like(H) for _ in hs]
    dWs = [torch.empty_like(Wr) for Wr in Ws]
    for h, dH, dW in zip(hs, dHs, dWs):
        h.backward(one, dH, dW)
    torch.cuda.synchronize()
    for h in hs:
        assert cce.cce_get_error(h.h) == 0
    return fw, dHs, dWs


def _check(p, fw, dHs, dWs, ref, dref=None):
    valid = p["labels"] != -100
    loss0, lse0 = fw[0][0].item(), fw[0][1].cpu().numpy()
    dH0 = dHs[0].view(torch.int16).cpu().numpy()
    for (loss, lse, nv), dH in zip(fw, dHs):
        assert loss.item() == loss0
        assert np.array_equal(lse.cpu().numpy().view(np.int32), lse0.view(np.int32))
        assert np.array_equal(dH.view(torch.int16).cpu().numpy(), dH0)
        assert int(nv.item()) == int(valid.sum())
    assert abs(loss0 - ref["loss"]) <= TOL_LOSS
    rel = np.abs(lse0[valid] - ref["lse"][valid]) / np.maximum(np.abs(ref["lse"][valid]), 1.0)
    assert rel.max() <= TOL_LSE
    assert np.all(lse0[~valid] == 0.0)
    assert np.all(dH0[~valid] == 0)
    assert rel_fro(_bf(dH0), ref["dH"] if dref is None else dref) <= TOL_GRAD
    dW = np.concatenate([_bf(d.view(torch.int16).cpu().numpy()) for d in dWs])
    assert rel_fro(dW, ref["dW"]) <= TOL_GRAD


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_p2p_group_matches_oracle(world):
    """2-8 ranks, a ragged vocabulary split (3000 / world) and a ragged row count: several dH
    tiles and chunks per rank; two consecutive steps (epochs 1, 2)."""
    p = workload.make_problem(700, 128, 3000, seed=606, ignore="bern40")
    H, W, y = to_dev(p, DEV)
    hs, Ws = _group(3000, world, 700, 128, W)
    ref = oracle.cce(p["H"], p["W"], p["labels"])
    for _ in range(2):
        fw, dHs, dWs = _step(hs, Ws, H, y)
        _check(p, fw, dHs, dWs, ref)
    for h in hs:
        h.close()


def test_p2p_group_multi_chunk_and_tiles():
    """A vocabulary shard larger than one backward chunk (8192) on every rank and 2 x 4 dH
    tiles: the RED items start while other rank groups still run their last chunk's dW items."""
    p = workload.make_problem(600, 896, 20000, seed=11, ignore="bern40")
    H, W, y = to_dev(p, DEV)
    hs, Ws = _group(20000, 2, 600, 896, W)
    ref = oracle.cce(p["H"], p["W"], p["labels"])
    fw, dHs, dWs = _step(hs, Ws, H, y)
    _check(p, fw, dHs, dWs, ref)
    for h in hs:
        h.close()


@pytest.mark.parametrize("mode", ["ls", "rms"])
def test_p2p_group_regularised_loss_and_rmsnorm(mode):
    """The exchange carries the label-smoothing logit sums (4th stat) and feeds the RMSNorm
    prologue's backward (dH reduced across ranks before dX / dgamma)."""
    p = workload.make_problem(700, 128, 3000, seed=606, ignore="bern40")
    H, W, y = to_dev(p, DEV)
    kw = dict(label_smoothing=0.1, z_loss=1e-4) if mode == "ls" else {}
    hs, Ws = _group(3000, 2, 700, 128, W, **kw)
    one = torch.ones((), dtype=torch.float32, device=DEV)
    if mode == "ls":
        ref = oracle.cce(p["H"], p["W"], p["labels"], label_smoothing=0.1, z_loss=1e-4)
        fw, dHs, dWs = _step(hs, Ws, H, y)
        _check(p, fw, dHs, dWs, ref)
    else:
        Xb, gb = workload.make_rmsnorm_inputs(606, 700, 128)
        X = torch.from_numpy(Xb.view(np.int16)).view(torch.bfloat16).to(DEV)
        g = torch.from_numpy(gb.view(np.int16)).view(torch.bfloat16).to(DEV)
        ref = oracle.cce_rmsnorm(Xb, gb, p["W"], p["labels"], eps=1e-6)
        fw = [h.forward_rmsnorm(X, g, 1e-6, Wr, y) for h, Wr in zip(hs, Ws)]
        dXs = [torch.empty_like(X) for _ in hs]
        dgs = [torch.empty_like(g) for _ in hs]
        dWs = [torch.empty_like(Wr) for Wr in Ws]
        for h, dX, dg, dW in zip(hs, dXs, dgs, dWs):
            h.backward_rmsnorm(one, dX, dg, dW)
        torch.cuda.synchronize()
        for h in hs:
            assert cce.cce_get_error(h.h) == 0
        assert abs(fw[0][0].item() - ref["loss"]) <= TOL_LOSS
        for dX in dXs:
            assert torch.equal(dX.view(torch.int16), dXs[0].view(torch.int16))
        assert rel_fro(_bf(dXs[0].view(torch.int16).cpu().numpy()), ref["dX"]) <= TOL_GRAD
        assert rel_fro(np.concatenate([_bf(d.view(torch.int16).cpu().numpy()) for d in dWs]), ref["dW"]) <= TOL_GRAD
    for h in hs:
        h.close()


def test_p2p_group_forward_only_loop():
    """Back-to-back forwards without a backward (evaluation): the double-buffered stats
    exchange keeps step e + 1 from overwriting what a rank still reads for step e."""
    p = workload.make_problem(700, 128, 3000, seed=606, ignore="bern40")
    H, W, y = to_dev(p, DEV)
    hs, Ws = _group(3000, 3, 700, 128, W)
    losses = []
    for step in range(4):
        yr = torch.roll(y, step)
        fw = [h.forward(H, Wr, yr) for h, Wr in zip(hs, Ws)]
        losses.append([f[0] for f in fw])
    torch.cuda.synchronize()
    for step in range(4):
        ref = oracle.cce(p["H"], p["W"], np.roll(p["labels"], step))
        for l in losses[step]:
            assert abs(l.item() - ref["loss"]) <= TOL_LOSS
    for h in hs:
        assert cce.cce_get_error(h.h) == 0
        h.close()


def test_p2p_group_out_of_order_calls_are_refused():
    """The group defers each rank's tail to the last rank's call: a backward before the
    group's forward is complete is refused, and a group with a foreign handle is rejected."""
    p = workload.make_problem(300, 64, 1000, seed=3, ignore="bern40")
    H, W, y = to_dev(p, DEV)
    hs, Ws = _group(1000, 2, 300, 64, W)
    hs[0].forward(H, Ws[0], y)     # rank 1 has not run its forward: nothing is finalised yet
    with pytest.raises(cce.CCEError):
        hs[0].backward(torch.ones((), device=DEV), torch.empty_like(H), torch.empty_like(Ws[0]))
    hs[1].forward(H, Ws[1], y)
    fw, dHs, dWs = _step(hs, Ws, H, y)
    _check(p, fw, dHs, dWs, oracle.cce(p["H"], p["W"], p["labels"]))
    lone = cce.CCEHandle(vocab_total=1000, rank=0, world=2, flags=cce.FLAG_P2P_COMBINE)
    with pytest.raises(cce.CCEError):
        cce.cce_p2p_attach_group([lone.h, hs[1].h], [lone.workspace(300, 64, 500, DEV), hs[1]._ws], 300, 64)
    hs[0].close()                   # a destroyed member: the others refuse further steps
    with pytest.raises(cce.CCEError):
        hs[1].forward(H, Ws[1], y)
    for h in hs + [lone]:
        h.close()


@pytest.mark.parametrize("world", [2, 8])
def test_p2p_group_full_size_bench_config(world):
    """The bench configuration (Qwen2.5-0.5B head, N = 8192, V = 151,936 split `world` ways,
    40% packed padding): every rank's loss and every valid row's LSE against the fp64 oracle
    golden, sampled dW rows of every shard against the oracle, bit-identical ranks."""
    import hashlib
    import os
    gold = os.path.join(os.path.dirname(__file__), "golden", "qwen05b_seed42.npz")
    if not os.path.exists(gold):
        pytest.skip("golden file missing (scripts/make_golden.py)")
    g = np.load(gold)
    p = workload.make_config("qwen05b", seed=42)
    assert hashlib.sha256(p["W"].tobytes()).hexdigest() == str(g["W_sha256"])
    H, W, y = to_dev(p, DEV)
    N, D = H.shape
    V = W.shape[0]
    hs, Ws = _group(V, world, N, D, W)
    fw, dHs, dWs = _step(hs, Ws, H, y)
    valid = p["labels"] != -100
    ref_loss = float(np.mean(g["lse"] - g["zy"]))
    lse0 = fw[0][1].cpu().numpy()
    for (loss, lse, nv), dH in zip(fw, dHs):
        assert abs(loss.item() - ref_loss) <= TOL_LOSS
        assert np.array_equal(lse.cpu().numpy().view(np.int32), lse0.view(np.int32))
        assert torch.equal(dH.view(torch.int16), dHs[0].view(torch.int16))
    rel = np.abs(lse0[valid] - g["lse"]) / np.maximum(np.abs(g["lse"]), 1.0)
    assert rel.max() <= TOL_LSE
    lse_all = np.zeros(N)
    lse_all[g["valid_rows"]] = g["lse"]
    for r in range(world):
        lo, hi = cce.shard_range(V, r, world)
        pick = np.unique(np.array([lo, lo + 1, (lo + hi) // 2, hi - 1]))
        ref = oracle.dW_rows(p["H"], p["W"], p["labels"], lse_all, 1.0 / len(g["valid_rows"]), pick)
        got = _bf(dWs[r].view(torch.int16).cpu().numpy()[pick - lo])
        assert rel_fro(got, ref) <= TOL_GRAD, r
    rows = g["valid_rows"]
    pick = rows[np.linspace(0, len(rows) - 1, 8).astype(int)]
    _, _, dH_ref = oracle.rows(p["H"], p["W"], p["labels"], pick, scale=1.0 / len(rows))
    assert rel_fro(_bf(dHs[0].view(torch.int16).cpu().numpy()[pick]), dH_ref) <= TOL_GRAD
    for h in hs:
        h.close()


@pytest.mark.parametrize("mode", ["sum", "none", "fp32", "fp32_accumulate"])
def test_p2p_group_reductions_and_gradient_modes(mode):
    """The exchange under the other reductions (sum; none with per-row upstream gradients, the
    per-token losses identical on every rank) and gradient modes (float32 dH / dW, accumulated
    into existing buffers: the reduced dH is added once, on every rank)."""
    p = workload.make_problem(700, 256, 9000, seed=21, ignore="bern40")
    H, W, y = to_dev(p, DEV)
    world = 3
    reduction = mode if mode in ("sum", "none") else "mean"
    flags = cce.FLAG_GRAD_FP32 | (cce.FLAG_ACCUMULATE if mode == "fp32_accumulate" else 0) if mode.startswith("fp32") else 0
    hs, Ws, wss = [], [], []
    for r in range(world):
        lo, hi = cce.shard_range(9000, r, world)
        h = cce.CCEHandle(vocab_total=9000, vocab_offset=lo, rank=r, world=world, flags=cce.FLAG_P2P_COMBINE | flags,
                          reduction=reduction)
        hs.append(h)
        wss.append(h.workspace(700, 256, hi - lo, DEV))
        Ws.append(W[lo:hi].contiguous())
    cce.cce_p2p_attach_group([h.h for h in hs], wss, 700, 256)
    if reduction == "none":
        dl_np = np.random.default_rng(3).standard_normal(700).astype(np.float32).astype(np.float64) / 700
        dloss = torch.tensor(dl_np, dtype=torch.float32, device=DEV)
    else:
        dl_np = 0.5 / 420
        dloss = torch.tensor(dl_np, dtype=torch.float32, device=DEV)
    ref = oracle.cce(p["H"], p["W"], p["labels"], dloss=dl_np, reduction=reduction)
    gdt = torch.float32 if flags & cce.FLAG_GRAD_FP32 else torch.bfloat16
    init = mode == "fp32_accumulate"
    g0 = torch.Generator(device="cpu").manual_seed(5)
    dH0 = torch.randn(H.shape, generator=g0).to(DEV) * 1e-3 if init else None
    dHs = [dH0.clone() if init else torch.empty(H.shape, dtype=gdt, device=DEV) for _ in hs]
    dW0 = [torch.randn(Wr.shape, generator=g0).to(DEV) * 1e-3 if init else None for Wr in Ws]
    dWs = [dW0[r].clone() if init else torch.empty(Wr.shape, dtype=gdt, device=DEV) for r, Wr in enumerate(Ws)]
    fw = [h.forward(H, Wr, y) for h, Wr in zip(hs, Ws)]
    for h, dH, dW in zip(hs, dHs, dWs):
        h.backward(dloss, dH, dW)
    torch.cuda.synchronize()
    valid = p["labels"] != -100
    for h, (loss, lse, nv), dH in zip(hs, fw, dHs):
        assert cce.cce_get_error(h.h) == 0
        assert torch.equal(loss, fw[0][0]) and torch.equal(dH, dHs[0])
    l0 = fw[0][0].cpu().numpy().astype(np.float64)
    assert np.max(np.abs(l0 - np.asarray(ref["loss"]))) <= TOL_LOSS
    f64 = (lambda t: t.cpu().numpy().astype(np.float64)) if gdt == torch.float32 else (
        lambda t: _bf(t.view(torch.int16).cpu().numpy()))
    dH_ref = ref["dH"] + (dH0.cpu().numpy().astype(np.float64) if init else 0.0)
    assert rel_fro(f64(dHs[0]), dH_ref) <= TOL_GRAD
    dW_ref = ref["dW"] + (np.concatenate([d.cpu().numpy() for d in dW0]).astype(np.float64) if init else 0.0)
    assert rel_fro(np.concatenate([f64(d) for d in dWs]), dW_ref) <= TOL_GRAD
    if not init:
        assert np.all(f64(dHs[0])[~valid] == 0)
    for h in hs:
        h.close()
