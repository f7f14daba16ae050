"""Vocabulary-sharded path (rows a9 stats exchange, a10 dH sum) on ONE GPU:
several shard handles driven by one process with the split-phase combine
(CCE_FLAG_EXTERNAL_COMBINE), the exchange done with torch ops in rank order -- the same
data flow as the NCCL path (allgather of per-row (m, d, z_y, sum z), rank-order merge in
k_finalize, sum of partial dH).  Compared with the unsharded fp64 oracle; every rank must
produce the same loss / LSE / dH bit for bit, and the concatenated dW shards the global dW."""
import numpy as np
import pytest

import oracle
import workload
from cce_testutil import TOL_GRAD, TOL_LOSS, TOL_LSE, bf16_to_f64, rel_fro, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import torch
    import __graft_entry__
    __graft_entry__.build()
    return torch.device("cuda:0")


def _sharded(dev, p, world, eps=0.0, lam=0.0):
    import torch
    import paper_2601_02609_b200 as cce
    H, W, y = to_dev(p, dev)
    N, D = H.shape
    V = W.shape[0]
    hs, outs = [], []
    for r in range(world):
        lo, hi = cce.shard_range(V, r, world)
        Wr = W[lo:hi].contiguous()
        h = cce.CCEHandle(vocab_total=V, vocab_offset=lo, rank=r, world=world, flags=cce.FLAG_EXTERNAL_COMBINE,
                          label_smoothing=eps, z_loss=lam)
        loss, lse, nv = h.forward(H, Wr, y)
        hs.append((h, Wr, loss, lse, nv, cce.cce_combine_offsets(h.h, N, D, hi - lo)))
    # a9: allgather the per-rank stats (rank-major) into every rank's all-ranks array
    parts = []
    for h, Wr, _, _, _, (so, sao, dho, npad) in hs:
        parts.append(h._ws[so:so + npad * 16].view(torch.float32).clone())
    allstats = torch.cat(parts)
    for h, Wr, _, _, _, (so, sao, dho, npad) in hs:
        h._ws[sao:sao + world * npad * 16].view(torch.float32).copy_(allstats)
        cce.cce_forward_finish(h.h)
    one = torch.ones((), dtype=torch.float32, device=dev)
    dWs, dHs = [], []
    for h, Wr, *_ in hs:
        dH = torch.empty_like(H)
        dW = torch.empty_like(Wr)
        h.backward(one, dH, dW)
        dHs.append(dH)
        dWs.append(dW)
    # a10: sum of the partial dH (fixed rank order), written back to every rank
    tot = None
    for h, Wr, _, _, _, (so, sao, dho, npad) in hs:
        part = h._ws[dho:dho + npad * D * 4].view(torch.float32)
        tot = part.clone() if tot is None else tot + part
    for (h, Wr, _, _, _, (so, sao, dho, npad)), dH in zip(hs, dHs):
        h._ws[dho:dho + npad * D * 4].view(torch.float32).copy_(tot)
        cce.cce_backward_finish(h.h)
    torch.cuda.synchronize()
    res = []
    for (h, Wr, loss, lse, nv, _), dH in zip(hs, dHs):
        res.append({"loss": float(loss.item()), "lse": lse.cpu().numpy(), "n_valid": int(nv.item()),
                     "dH_bits": dH.view(torch.int16).cpu().numpy(), "dH": bf16_to_f64(dH)})
        h.close()
    dW = np.concatenate([bf16_to_f64(d) for d in dWs]) if dWs else None
    return res, dW


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("N,D,V,ign", [
    (700, 128, 3000, "bern40"),      # ragged shards (3000 / 3, / 8 not multiples of 256)
    (384, 896, 20000, "bern40"),     # Qwen hidden size, several chunks per shard at world 2
])
def test_sharded_matches_oracle(dev, world, N, D, V, ign):
    p = workload.make_problem(N, D, V, seed=N + V + world, ignore=ign)
    res, dW = _sharded(dev, p, world)
    ref = oracle.cce(p["H"], p["W"], p["labels"])
    valid = p["labels"] != -100
    for r in res:   # identical on every rank
        assert r["loss"] == res[0]["loss"]
        assert np.array_equal(r["lse"].view(np.int32), res[0]["lse"].view(np.int32))
        assert np.array_equal(r["dH_bits"], res[0]["dH_bits"])
    o = res[0]
    assert o["n_valid"] == int(valid.sum())
    assert abs(o["loss"] - ref["loss"]) <= TOL_LOSS
    rel = np.abs(o["lse"][valid] - ref["lse"][valid]) / np.maximum(np.abs(ref["lse"][valid]), 1.0)
    assert rel.max() <= TOL_LSE
    assert np.all(o["lse"][~valid].view(np.int32) == 0) and np.all(o["dH_bits"][~valid] == 0)
    assert rel_fro(o["dH"], ref["dH"]) <= TOL_GRAD
    assert rel_fro(dW, ref["dW"]) <= TOL_GRAD


def test_sharded_regularised_loss(dev):
    """Label smoothing needs the sum of the logits over the GLOBAL vocabulary (4th stat,
    summed across ranks, reading R12); z-loss the global LSE."""
    p = workload.make_problem(700, 128, 3000, seed=77, ignore="bern40")
    res, dW = _sharded(dev, p, 3, eps=0.1, lam=1e-4)
    ref = oracle.cce(p["H"], p["W"], p["labels"], label_smoothing=0.1, z_loss=1e-4)
    assert abs(res[0]["loss"] - ref["loss"]) <= TOL_LOSS
    assert rel_fro(res[0]["dH"], ref["dH"]) <= TOL_GRAD
    assert rel_fro(dW, ref["dW"]) <= TOL_GRAD


def test_sharded_with_empty_shard(dev):
    """More ranks than some shards have rows: V = 2, world = 3 (rank 0 owns nothing and
    contributes (m = -inf, d = 0, z_y = 0), reading R17)."""
    p = workload.make_problem(64, 64, 2, seed=5, ignore="bern10")
    res, dW = _sharded(dev, p, 3)
    ref = oracle.cce(p["H"], p["W"], p["labels"])
    assert abs(res[0]["loss"] - ref["loss"]) <= TOL_LOSS
    assert rel_fro(res[0]["dH"], ref["dH"]) <= TOL_GRAD
    assert rel_fro(dW, ref["dW"]) <= TOL_GRAD


@pytest.mark.parametrize("world", [2, 3])
def test_labels_in_a_shards_padded_tail(dev, world):
    """Regression: a label owned by rank r+1 whose local id on rank r falls in rank r's padded
    tail tile (V_local .. next multiple of 256) must not be captured as rank r's target logit
    (it read the masked -inf logit: loss = inf).  Uniform labels over V = 600 put many labels
    in [300, 512) for world 2 (rank 0 owns [0, 300))."""
    p = workload.make_problem(256, 64, 600, seed=3 + world, ignore="bern10", label_dist="uniform")
    res, dW = _sharded(dev, p, world)
    ref = oracle.cce(p["H"], p["W"], p["labels"])
    assert np.isfinite(res[0]["loss"]) and abs(res[0]["loss"] - ref["loss"]) <= TOL_LOSS
    assert rel_fro(res[0]["dH"], ref["dH"]) <= TOL_GRAD
    assert rel_fro(dW, ref["dW"]) <= TOL_GRAD


def _sharded_seq(dev, p, world):
    """CCE_FLAG_DH_SEQ_SHARD with the split-phase combine: the stats allgather as above,
    then each rank's partial dH in original row order is reduce-scattered (torch sum in rank
    order; rank r's slice placed at row r*S of its own array) and cce_backward_finish writes
    that rank's [n_r, D] rows."""
    import torch
    import paper_2601_02609_b200 as cce
    H, W, y = to_dev(p, dev)
    N, D = H.shape
    V = W.shape[0]
    S = (N + world - 1) // world
    hs = []
    for r in range(world):
        lo, hi = cce.shard_range(V, r, world)
        Wr = W[lo:hi].contiguous()
        h = cce.CCEHandle(vocab_total=V, vocab_offset=lo, rank=r, world=world,
                          flags=cce.FLAG_EXTERNAL_COMBINE | cce.FLAG_DH_SEQ_SHARD)
        loss, lse, nv = h.forward(H, Wr, y)
        hs.append((h, Wr, loss, cce.cce_combine_offsets(h.h, N, D, hi - lo)))
    allstats = torch.cat([h._ws[so:so + npad * 16].view(torch.float32).clone()
                          for h, _, _, (so, sao, dho, npad) in hs])
    for h, _, _, (so, sao, dho, npad) in hs:
        h._ws[sao:sao + world * npad * 16].view(torch.float32).copy_(allstats)
        cce.cce_forward_finish(h.h)
    one = torch.ones((), dtype=torch.float32, device=dev)
    dHs, dWs = [], []
    for r, (h, Wr, _, _) in enumerate(hs):
        n_r = max(0, min(S, N - r * S))
        dH = torch.full((max(n_r, 1), D), float("nan"), dtype=torch.bfloat16, device=dev)
        dW = torch.empty_like(Wr)
        h.backward(one, dH, dW)
        dHs.append((dH, n_r))
        dWs.append(dW)
    tot = None
    for h, _, _, (so, sao, dho, npad) in hs:
        part = h._ws[dho:dho + world * S * D * 4].view(torch.float32)
        tot = part.clone() if tot is None else tot + part
    for r, (h, _, _, (so, sao, dho, npad)) in enumerate(hs):
        h._ws[dho + r * S * D * 4:dho + (r + 1) * S * D * 4].view(torch.float32).copy_(tot[r * S * D:(r + 1) * S * D])
        cce.cce_backward_finish(h.h)
    torch.cuda.synchronize()
    dH = np.concatenate([bf16_to_f64(d)[:n] for d, n in dHs])
    loss = hs[0][2].item()
    for h, *_ in hs:
        h.close()
    return loss, dH, np.concatenate([bf16_to_f64(d) for d in dWs])


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_sequence_sharded_dH(dev, world):
    """CCE_FLAG_DH_SEQ_SHARD (NEXT #4): every rank gets its own ceil(N/P) original rows of dH
    (N = 700 is not a multiple of 3: ragged last slice)."""
    p = workload.make_problem(700, 128, 3000, seed=91 + world, ignore="bern40")
    loss, dH, dW = _sharded_seq(dev, p, world)
    ref = oracle.cce(p["H"], p["W"], p["labels"])
    assert abs(loss - ref["loss"]) <= TOL_LOSS
    assert dH.shape == ref["dH"].shape
    assert np.all(dH[p["labels"] == -100] == 0)
    assert rel_fro(dH, ref["dH"]) <= TOL_GRAD
    assert rel_fro(dW, ref["dW"]) <= TOL_GRAD


def test_sequence_sharded_dH_nccl_one_rank(dev):
    """The NCCL reduce-scatter on a 1-rank communicator is the identity: dH bit-identical to
    the plain path."""
    import torch
    import paper_2601_02609_b200 as cce
    p = workload.make_problem(700, 256, 9000, seed=29, ignore="bern40")
    H, W, y = to_dev(p, dev)
    one = torch.ones((), dtype=torch.float32, device=dev)
    outs = []
    comm = cce.cce_nccl_comm_init(1, cce.cce_nccl_unique_id(), 0)
    try:
        for flags, c in ((0, None), (cce.FLAG_DH_SEQ_SHARD, comm)):
            h = cce.CCEHandle(vocab_total=9000, nccl_comm=c, flags=flags)
            h.forward(H, W, y)
            dH = torch.empty_like(H)
            dW = torch.empty_like(W)
            h.backward(one, dH, dW)
            torch.cuda.synchronize()
            outs.append((dH.view(torch.int16).cpu(), dW.view(torch.int16).cpu()))
            h.close()
    finally:
        cce.cce_nccl_comm_destroy(comm)
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
