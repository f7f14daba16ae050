"""A classifier whose element count passes 2^31: V = 151,936 (the Qwen vocabulary) x
D = 16,384 (405B-class hidden size) = 2.49e9 elements, 4.98 GB bf16.  From vocabulary row
131,072 on, element offsets of W / dW pass 2^31 and byte offsets pass 2^32, so any 32-bit
index arithmetic in the kernels, the tensor maps or the epilogues shows up here.

W is drawn on the GPU by workload.normal_bf16_torch (bit-identical to the numpy generator,
tests/test_workload.py) and copied to the host for the oracle.  The oracle's per-row LSE
comes from oracle.partial_stats over 8192-row vocabulary slices (fp64 copies of one slice
at a time), merged by the (m, d) rule of P:1157-1163 written out below (pin 7 checks that
merge against the unsharded oracle); dW rows around and past the boundary come from
oracle.dW_rows on those rows.  N is small (one 256-row tile, 40% ignored), so the oracle
finishes in about a minute."""
import math

import numpy as np
import pytest

import oracle
import workload
from cce_testutil import TOL_GRAD, TOL_LOSS, TOL_LSE, rel_fro

pytestmark = pytest.mark.gpu

N, D, V = 96, 16384, 151936
SEED = 11


def _merge(parts):
    """lse of a union of slices from per-slice (max, sum exp(z - max))."""
    m = max(mi for mi, di in parts if di > 0)
    return m + math.log(sum(di * math.exp(mi - m) for mi, di in parts if di > 0))


def test_lse_loss_and_dW_rows_past_2_pow_31_elements():
    import torch
    import __graft_entry__
    import paper_2601_02609_b200 as cce
    __graft_entry__.build()
    dev = torch.device("cuda:0")
    valid = workload.bernoulli_valid_mask(SEED, N, 0.4)
    lab = workload.randint(SEED, workload.S_LABEL, 0, N, 0, V - 1).astype(np.int32)   # uniform: many in the tail
    lab[:4] = [131071, 131072, V - 1, 140000]
    valid[:4] = True
    labels = np.where(valid, lab, workload.IGNORE_INDEX).astype(np.int32)
    H = workload.normal_bf16(SEED, workload.S_H, N, D, 1.0)
    Wd = workload.normal_bf16_torch(SEED, workload.S_W, V, D, 1.0 / math.sqrt(D), dev)
    Hd = torch.from_numpy(H.view(np.int16)).view(torch.bfloat16).to(dev)
    yd = torch.from_numpy(labels).to(dev)

    h = cce.CCEHandle(vocab_total=V)
    loss, lse, nv = h.forward(Hd, Wd, yd)
    dH = torch.empty((N, D), dtype=torch.bfloat16, device=dev)
    dW = torch.empty((V, D), dtype=torch.bfloat16, device=dev)
    h.backward(torch.ones((), dtype=torch.float32, device=dev), dH, dW)
    torch.cuda.synchronize()
    h.close()
    nvalid = int(valid.sum())
    assert int(nv.item()) == nvalid
    lse_g = lse.cpu().numpy().astype(np.float64)

    # whole-output properties (every vocabulary row, incl. the 20,864 past the boundary):
    # rows of dlogits sum to zero, so sum_v dW[v, :] = 0 up to the bf16 rounding of G
    dWf = dW.float()
    assert bool(torch.isfinite(dWf).all())
    colsum = dWf.sum(0).norm().item()
    assert colsum <= 1e-2 * dWf.norm().item()
    tail_norm = dWf[131072:].norm().item()
    assert tail_norm > 0
    del dWf
    assert bool(torch.isfinite(dH.float()).all())
    assert bool((dH[torch.from_numpy(~valid).to(dev)] == 0).all())

    W = Wd.view(torch.int16).cpu().numpy().view(np.uint16)      # 4.98 GB of host memory
    del Wd
    pick = np.array([0, 131071, 131072, 131073, 140000, 150000, V - 257, V - 256, V - 1], np.int64)
    dW_got = (dW[torch.from_numpy(pick).to(dev)].view(torch.int16).cpu().numpy().astype(np.uint16)
              .astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    del dW
    torch.cuda.empty_cache()

    # oracle LSE / target logits over 8192-row vocabulary slices
    stats = [oracle.partial_stats(H, W[lo:min(lo + 8192, V)], labels, lo) for lo in range(0, V, 8192)]
    lse_ref = np.zeros(N)
    zy_ref = np.zeros(N)
    for n in np.nonzero(valid)[0]:
        lse_ref[n] = _merge([(s[0][n], s[1][n]) for s in stats])
        zy_ref[n] = sum(s[2][n] for s in stats)
    rel = np.abs(lse_g[valid] - lse_ref[valid]) / np.maximum(np.abs(lse_ref[valid]), 1.0)
    assert rel.max() <= TOL_LSE, rel.max()
    assert abs(loss.item() - float(np.mean(lse_ref[valid] - zy_ref[valid]))) <= TOL_LOSS

    # dW rows around and past the 2^31-element boundary: the picked rows as their own
    # small W, labels renumbered to positions in `pick` (others point past it)
    pos = {int(v): i for i, v in enumerate(pick)}
    lab_sub = np.array([pos.get(int(y), len(pick)) if y != workload.IGNORE_INDEX else y for y in labels], np.int32)
    ref = oracle.dW_rows(H, W[pick], lab_sub, lse_ref, 1.0 / nvalid, np.arange(len(pick)))
    for i in range(len(pick)):
        assert rel_fro(dW_got[i], ref[i]) <= TOL_GRAD, (int(pick[i]), rel_fro(dW_got[i], ref[i]))


def test_lse_and_dH_rows_past_2_pow_31_token_elements():
    """The token side: N = 163,840 x D = 16,384 (H 5.4 GB, 10% ignored, so the compacted
    rows pass 2^31 elements too, from compact row 131,072 on) against a small vocabulary
    (V = 4,000, ragged tail tile).  LSE and dH are compared on rows before and past the
    boundary, computed by oracle.rows one by one; dW by the zero-column-sum property."""
    import torch
    import __graft_entry__
    import paper_2601_02609_b200 as cce
    __graft_entry__.build()
    dev = torch.device("cuda:0")
    Nt, Dt, Vt = 163840, 16384, 4000
    valid = workload.bernoulli_valid_mask(SEED, Nt, 0.1)
    labels = np.where(valid, workload.randint(SEED, workload.S_LABEL, 0, Nt, 0, Vt - 1),
                      workload.IGNORE_INDEX).astype(np.int32)
    W = workload.normal_bf16(SEED, workload.S_W, Vt, Dt, 1.0 / math.sqrt(Dt))
    Hd = workload.normal_bf16_torch(SEED, workload.S_H, Nt, Dt, 1.0, dev)
    Wd = torch.from_numpy(W.view(np.int16)).view(torch.bfloat16).to(dev)
    yd = torch.from_numpy(labels).to(dev)
    h = cce.CCEHandle(vocab_total=Vt)
    loss, lse, nv = h.forward(Hd, Wd, yd)
    dH = torch.empty((Nt, Dt), dtype=torch.bfloat16, device=dev)
    dW = torch.empty((Vt, Dt), dtype=torch.bfloat16, device=dev)
    h.backward(torch.ones((), dtype=torch.float32, device=dev), dH, dW)
    torch.cuda.synchronize()
    h.close()
    vrows = np.nonzero(valid)[0]
    nvalid = len(vrows)
    assert int(nv.item()) == nvalid and nvalid * Dt > (1 << 31)
    assert bool(torch.isfinite(dH.float()).all()) and bool(torch.isfinite(dW.float()).all())
    assert bool((dH[torch.from_numpy(~valid).to(dev)] == 0).all())
    dWf = dW.float()
    assert dWf.sum(0).norm().item() <= 1e-2 * dWf.norm().item()

    # valid rows around compact row 131,072 (the 2^31-element boundary of the compact copy),
    # around original row 131,072, and the last rows
    pick = np.unique(np.concatenate([vrows[[0, 1, 131070, 131071, 131072, 131073, nvalid - 2, nvalid - 1]],
                                     vrows[np.searchsorted(vrows, [131071, 131072, 140000])]]))
    pick_d = torch.from_numpy(pick).to(dev)
    H_pick = Hd[pick_d].view(torch.int16).cpu().numpy().view(np.uint16)
    dH_pick = (dH[pick_d].view(torch.int16).cpu().numpy().astype(np.uint16).astype(np.uint32) << 16) \
        .view(np.float32).astype(np.float64)
    lse_ref, _, dH_ref = oracle.rows(H_pick, W, labels[pick], np.arange(len(pick)), scale=1.0 / nvalid)
    lse_g = lse.cpu().numpy().astype(np.float64)[pick]
    rel = np.abs(lse_g - lse_ref) / np.maximum(np.abs(lse_ref), 1.0)
    assert rel.max() <= TOL_LSE, rel.max()
    for i in range(len(pick)):
        assert rel_fro(dH_pick[i], dH_ref[i]) <= TOL_GRAD, (int(pick[i]), rel_fro(dH_pick[i], dH_ref[i]))
