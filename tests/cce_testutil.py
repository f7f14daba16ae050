"""Shared helpers for the GPU parity tests (marshalling only; no method arithmetic)."""
import numpy as np

TOL_LOSS = 2e-3          # north_star: loss absolute error
TOL_LSE = 1e-3           # per-token LSE relative error (floor 1 on |lse|)
TOL_GRAD = 1e-2          # dH, dW relative Frobenius error


def to_dev(p, dev):
    import torch
    H = torch.from_numpy(p["H"].view(np.int16)).view(torch.bfloat16).to(dev)
    W = torch.from_numpy(p["W"].view(np.int16)).view(torch.bfloat16).to(dev)
    y = torch.from_numpy(p["labels"]).to(dev)
    return H, W, y


def bf16_to_f64(t):
    import torch
    return t.detach().to(torch.float32).cpu().numpy().astype(np.float64)


def rel_fro(got, want):
    nw = np.linalg.norm(want)
    if nw == 0:
        return 0.0 if np.all(got == 0) else np.inf
    return float(np.linalg.norm(got - want) / nw)


def run_gpu(H, W, y, dloss=1.0, handle=None, vocab_total=None, flags=0, label_smoothing=0.0, z_loss=0.0,
            reduction="mean", dH_init=None, dW_init=None):
    """Forward + backward through the C ABI. Returns numpy results.  With reduction
    "none", dloss is an [N] array and "loss" the [N] per-token losses.  dH_init / dW_init
    (torch tensors, bf16 or fp32) are the buffers the backward writes / accumulates into."""
    import torch
    import paper_2601_02609_b200 as cce
    dev = H.device
    h = handle or cce.CCEHandle(vocab_total=vocab_total or W.shape[0], flags=flags, label_smoothing=label_smoothing,
                                z_loss=z_loss, reduction=reduction)
    loss, lse, nv = h.forward(H, W, y)
    gdt = torch.float32 if flags & cce.FLAG_GRAD_FP32 else torch.bfloat16
    dH = dH_init if dH_init is not None else torch.empty(H.shape, dtype=gdt, device=dev)
    dW = dW_init if dW_init is not None else torch.empty(W.shape, dtype=gdt, device=dev)
    dl = torch.tensor(np.asarray(dloss, dtype=np.float32), dtype=torch.float32, device=dev)
    h.backward(dl, dH, dW)
    torch.cuda.synchronize()
    lv = loss.cpu().numpy().astype(np.float64)
    if gdt == torch.float32:
        out_g = {"dH": dH.cpu().numpy().astype(np.float64), "dW": dW.cpu().numpy().astype(np.float64),
                 "dH_bits": dH.view(torch.int32).cpu().numpy(), "dW_bits": dW.view(torch.int32).cpu().numpy()}
    else:
        out_g = {"dH": bf16_to_f64(dH), "dW": bf16_to_f64(dW),
                 "dH_bits": dH.view(torch.int16).cpu().numpy(), "dW_bits": dW.view(torch.int16).cpu().numpy()}
    out = {"loss": lv if lv.ndim else float(lv), "lse": lse.cpu().numpy().astype(np.float64), "n_valid": int(nv.item()),
           "lse_bits": lse.view(torch.int32).cpu().numpy(), **out_g}
    if handle is None:
        h.close()
    return out


def assert_parity(got, ref, labels, check_grads=True):
    valid = labels != -100
    assert got["n_valid"] == ref["n_valid"] == int(valid.sum())
    assert np.max(np.abs(np.asarray(got["loss"]) - np.asarray(ref["loss"]))) <= TOL_LOSS, (got["loss"], ref["loss"])
    if valid.any():
        rel = np.abs(got["lse"][valid] - ref["lse"][valid]) / np.maximum(np.abs(ref["lse"][valid]), 1.0)
        assert rel.max() <= TOL_LSE, rel.max()
    assert np.all(got["lse_bits"][~valid] == 0)          # ignored rows: exactly 0.0f
    if check_grads:
        assert np.all(got["dH_bits"][~valid] == 0)       # ignored rows: bit-zero
        e = rel_fro(got["dH"], ref["dH"])
        assert e <= TOL_GRAD, ("dH", e)
        e = rel_fro(got["dW"], ref["dW"])
        assert e <= TOL_GRAD, ("dW", e)
