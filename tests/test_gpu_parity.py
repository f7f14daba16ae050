"""GPU parity: the CUDA path (through the C ABI) vs the fp64 CPU oracle, element
by element on the same seeded inputs.  Tolerances are north_star's (loss abs
2e-3, LSE rel 1e-3, dH/dW rel Frobenius 1e-2; n_valid and ignore masks exact)."""
import numpy as np
import pytest

import oracle
import workload
from cce_testutil import assert_parity, run_gpu, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import torch
    import __graft_entry__
    __graft_entry__.build()
    return torch.device("cuda:0")


def _check(p, dev, dloss=1.0, flags=0, label_smoothing=0.0, z_loss=0.0, reduction="mean"):
    H, W, y = to_dev(p, dev)
    got = run_gpu(H, W, y, dloss=dloss, flags=flags, label_smoothing=label_smoothing, z_loss=z_loss,
                  reduction=reduction)
    ref = oracle.cce(p["H"], p["W"], p["labels"], dloss=dloss, label_smoothing=label_smoothing, z_loss=z_loss,
                     reduction=reduction)
    assert_parity(got, ref, p["labels"])
    return got, ref


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4, 42])
def test_tiny_config(dev, seed):
    """configs[0]: N=64, D=64, V=1000 (tail tile of 232), 10% ignored."""
    _check(workload.make_config("tiny", seed=seed), dev)


@pytest.mark.parametrize("N,D,V,ign", [
    (700, 128, 3000, "bern40"),        # ragged rows (5.5 tiles), ragged vocab (11.7 tiles)
    (257, 64, 256, "none"),             # exactly one vocab tile, one ragged row
    (129, 192, 20000, "bern30"),        # 3 backward chunks, ragged last chunk
    (384, 896, 9000, "bern40"),         # Qwen hidden size, 2 chunks
    (1000, 128, 41000, "bern40"),       # 6 chunks: Gbuf ring slots reused, dH accumulated 6x
])
def test_multi_tile_shapes(dev, N, D, V, ign):
    p = workload.make_problem(N, D, V, seed=N + V, ignore=ign)
    _check(p, dev)


@pytest.mark.parametrize("N,D,V,ign", [
    (520, 2048, 9000, "none"),     # configs[2] hidden size (paper memory example), 0% ignored
    (300, 4096, 5000, "bern40"),   # configs[3] hidden size (Llama-3-8B head), ragged rows / vocabulary
    (700, 3584, 6100, "bern40"),   # configs[4] hidden size (Qwen2.5-7B head), 14 x 256 hidden tiles
    (260, 8192, 2300, "bern40"),   # Llama-3-70B-class hidden size: 128 k-blocks per logit tile, 32 hidden tiles
    (333, 5120, 4100, "none"),     # 5120 = 20 hidden tiles, ragged rows / vocabulary
    # L2 row groups (cce_pair.cuh l2_group_rows, 32 MB of Hc per group): 8 row tiles per group
    # at D = 8192 -> 13 tiles = 8 + 5; 4 per group at D = 16384 -> 9 tiles = 4 + 4 + a ragged ONE
    (3300, 8192, 1000, "none"),
    (2100, 16384, 700, "none"),
])
def test_large_hidden_sizes(dev, N, D, V, ign):
    """The wide-hidden configurations: D = 2048 / 3584 / 4096 (8 / 14 / 16 hidden tiles
    of 256, i.e. 4 / 7 / 8 quad items per dW / dH row or vocabulary tile)."""
    p = workload.make_problem(N, D, V, seed=D + V, ignore=ign)
    _check(p, dev)


@pytest.mark.parametrize("eps,lam", [(0.1, 0.0), (0.0, 1e-4), (0.1, 1e-4), (0.3, 1e-2)])
@pytest.mark.parametrize("N,D,V,ign,flags", [
    (700, 128, 3000, "bern40", 0),       # ragged rows / vocabulary
    (384, 896, 9000, "bern40", 0),       # Qwen hidden size, 2 chunks
    (1000, 128, 41000, "bern40", 0),     # 6 chunks
])
def test_label_smoothing_and_z_loss(dev, N, D, V, ign, flags, eps, lam):
    """the regularised loss (Def. Smoothed CE P:266-276, Def. Z-Loss
    P:281-287) against oracle_cce_reg, same tolerances as the plain loss."""
    p = workload.make_problem(N, D, V, seed=N + V + 1, ignore=ign)
    _check(p, dev, flags=flags, label_smoothing=eps, z_loss=lam)


@pytest.mark.parametrize("reduction,eps,lam,flags", [
    ("sum", 0.0, 0.0, 0), ("none", 0.0, 0.0, 0), ("sum", 0.1, 1e-4, 0), ("none", 0.1, 1e-3, 0),
])
def test_reductions(dev, reduction, eps, lam, flags):
    """sum and per-token ("none", per-row upstream gradients) losses."""
    p = workload.make_problem(700, 256, 9000, seed=21, ignore="bern40")
    if reduction == "none":
        dloss = np.random.default_rng(3).standard_normal(700).astype(np.float32).astype(np.float64) / 700
    else:
        dloss = 0.5 / 420
    _check(p, dev, dloss=dloss, flags=flags, label_smoothing=eps, z_loss=lam, reduction=reduction)


@pytest.mark.parametrize("flags", [64, 128, 192], ids=["fp32", "accumulate_bf16", "accumulate_fp32"])
def test_grad_dtype_and_accumulation(dev, flags):
    """NEXT #3: float32 gradients and accumulation into existing .grad buffers (the
    result minus the initial buffer is the gradient; ignored rows of dH untouched)."""
    import torch
    import paper_2601_02609_b200 as cce
    from cce_testutil import rel_fro
    p = workload.make_problem(600, 192, 7000, seed=22, ignore="bern40")
    H, W, y = to_dev(p, dev)
    gdt = torch.float32 if flags & cce.FLAG_GRAD_FP32 else torch.bfloat16
    g = torch.Generator(device="cpu").manual_seed(5)
    dH0 = (torch.randn(H.shape, generator=g) * 1e-3).to(gdt).to(dev)
    dW0 = (torch.randn(W.shape, generator=g) * 1e-3).to(gdt).to(dev)
    init_H = dH0.double().cpu().numpy(); init_W = dW0.double().cpu().numpy()
    got = run_gpu(H, W, y, flags=flags, dH_init=dH0.clone(), dW_init=dW0.clone())
    ref = oracle.cce(p["H"], p["W"], p["labels"])
    acc = bool(flags & cce.FLAG_ACCUMULATE)
    dH = got["dH"] - (init_H if acc else 0.0)
    dW = got["dW"] - (init_W if acc else 0.0)
    tol = 1e-2 if gdt == torch.bfloat16 and not acc else 2e-2   # bf16 accumulation rounds once more
    assert rel_fro(dH, ref["dH"]) <= tol and rel_fro(dW, ref["dW"]) <= tol
    ign = p["labels"] == -100
    if acc:
        assert np.array_equal(got["dH"][ign], init_H[ign])      # ignored rows untouched
    else:
        assert np.all(got["dH"][ign] == 0)


@pytest.mark.parametrize("regime", ["peaked", "zero"])
def test_label_smoothing_and_z_loss_regimes(dev, regime):
    """W = 0 (loss = ln V + lam ln^2 V exactly) and confident targets."""
    p = workload.make_problem(300, 128, 5000, seed=17, ignore="bern40", regime=regime)
    _check(p, dev, label_smoothing=0.1, z_loss=1e-3)


@pytest.mark.parametrize("regime", ["peaked", "extreme", "zero"])
def test_value_regimes(dev, regime):
    p = workload.make_problem(300, 128, 5000, seed=11, ignore="bern40", regime=regime)
    _check(p, dev)


@pytest.mark.parametrize("dloss", [0.37, -1.5, 0.0])
def test_upstream_gradient_scaling(dev, dloss):
    p = workload.make_problem(200, 64, 2000, seed=5, ignore="bern20")
    if dloss == 0.0:
        H, W, y = to_dev(p, dev)
        got = run_gpu(H, W, y, dloss=0.0)
        assert np.all(got["dH_bits"] == 0) and np.all(np.abs(got["dW"]) == 0)
        return
    _check(p, dev, dloss=dloss)


def test_all_ignored(dev):
    p = workload.make_problem(150, 64, 700, seed=6, ignore="all")
    H, W, y = to_dev(p, dev)
    got = run_gpu(H, W, y)
    assert got["n_valid"] == 0 and got["loss"] == 0.0
    assert np.all(got["dH_bits"] == 0) and np.all(got["dW_bits"] == 0) and np.all(got["lse_bits"] == 0)


def test_single_valid_token(dev):
    p = workload.make_problem(130, 64, 1500, seed=7, ignore="all")
    p["labels"][77] = 1234
    _check(p, dev)


def test_nan_in_ignored_rows_does_not_leak(dev):
    """Reading R14: ignored rows are never read -- NaN there leaves outputs bit-identical."""
    p = workload.make_problem(300, 128, 2500, seed=8, ignore="bern40")
    H, W, y = to_dev(p, dev)
    a = run_gpu(H, W, y)
    q = dict(p)
    Hn = p["H"].copy()
    Hn[p["labels"] == -100] = 0x7FC0          # bf16 NaN
    q["H"] = Hn
    H2, _, _ = to_dev(q, dev)
    b = run_gpu(H2, W, y)
    assert a["loss"] == b["loss"]
    for k in ("lse_bits", "dH_bits", "dW_bits"):
        assert np.array_equal(a[k], b[k]), k


def test_deterministic(dev):
    p = workload.make_problem(500, 128, 9000, seed=9, ignore="bern40")
    H, W, y = to_dev(p, dev)
    a = run_gpu(H, W, y)
    b = run_gpu(H, W, y)
    assert a["loss"] == b["loss"]
    for k in ("lse_bits", "dH_bits", "dW_bits"):
        assert np.array_equal(a[k], b[k]), k


def test_shift_invariance_bigshift(dev):
    """SURVEY pin 9 on the GPU: D = 895 + 1 constant column, c = 80, so every
    logit is shifted by +80 (exercises the max shift in the online softmax).
    Loss, LSE and the first 895 columns of dH / all of dW are held to the usual
    tolerances.  The appended dH column is 80 * sum_v G[n,v], exactly 0 in fp64
    but bf16-rounded G (the MMA operand) leaves
    80 x rounding noise there, so it is only bounded, not compared."""
    from cce_testutil import rel_fro
    p = workload.make_problem(256, 896, 3000, seed=10, ignore="bern40")
    H = p["H"].copy(); W = p["W"].copy()
    H[:, -1] = 0x3F80          # 1.0
    W[:, -1] = 0x42A0          # 80.0
    q = {"H": H, "W": W, "labels": p["labels"]}
    H_, W_, y_ = to_dev(q, dev)
    got = run_gpu(H_, W_, y_)
    ref = oracle.cce(q["H"], q["W"], q["labels"])
    assert_parity(got, ref, q["labels"], check_grads=False)
    assert rel_fro(got["dH"][:, :-1], ref["dH"][:, :-1]) <= 1e-2
    assert rel_fro(got["dW"], ref["dW"]) <= 1e-2
    # |dH[n,-1]| = 80 |sum_v G_bf16[n,v]| <= 80 * 2^-9 * sum_v |G[n,v]| <= 80 * 2^-8 * s  (s = 1/n_valid)
    s = 1.0 / ref["n_valid"]
    assert np.abs(got["dH"][:, -1]).max() <= 80.0 * 2.0 ** -8 * s * 2.0


def test_label_out_of_range_reports_error(dev):
    import torch
    import paper_2601_02609_b200 as cce
    p = workload.make_problem(100, 64, 500, seed=12, ignore="bern10")
    p["labels"][3] = 500
    H, W, y = to_dev(p, dev)
    h = cce.CCEHandle(vocab_total=500)
    loss, lse, nv = h.forward(H, W, y)
    assert cce.cce_get_error(h.h) == 3          # CCE_ERR_LABEL_RANGE
    assert np.isnan(loss.item())
    assert cce.cce_get_error(h.h) == 0          # cleared
    h.close()


def test_autograd_entry_point(dev):
    import torch
    import paper_2601_02609_b200 as cce
    p = workload.make_problem(200, 128, 3000, seed=13, ignore="bern40")
    H, W, y = to_dev(p, dev)
    H.requires_grad_(True); W.requires_grad_(True)
    loss = cce.linear_cross_entropy(H, W, y)
    (2.0 * loss).backward()
    ref = oracle.cce(p["H"], p["W"], p["labels"], dloss=2.0)
    from cce_testutil import bf16_to_f64, rel_fro
    assert abs(loss.item() - ref["loss"]) <= 2e-3
    assert rel_fro(bf16_to_f64(H.grad), ref["dH"]) <= 1e-2
    assert rel_fro(bf16_to_f64(W.grad), ref["dW"]) <= 1e-2


def test_step_host_matches_device_path(dev):
    import torch
    import paper_2601_02609_b200 as cce
    p = workload.make_problem(300, 128, 4000, seed=14, ignore="bern40")
    _, W, _ = to_dev(p, dev)
    Hh = torch.from_numpy(p["H"].view(np.int16)).view(torch.bfloat16).pin_memory()
    yh = torch.from_numpy(p["labels"]).pin_memory()
    h = cce.CCEHandle(vocab_total=4000)
    ws = h.workspace(300, 128, 4000, dev)
    st = torch.empty(cce.cce_host_staging_bytes(300, 128), dtype=torch.uint8, device=dev)
    dH = torch.empty((300, 128), dtype=torch.bfloat16, device=dev)
    dW = torch.empty((4000, 128), dtype=torch.bfloat16, device=dev)
    loss = cce.cce_step_host(h.h, Hh, yh, W, dH, dW, st, ws)
    ref = oracle.cce(p["H"], p["W"], p["labels"])
    assert abs(loss - ref["loss"]) <= 2e-3
    from cce_testutil import bf16_to_f64, rel_fro
    assert rel_fro(bf16_to_f64(dH), ref["dH"]) <= 1e-2
    assert rel_fro(bf16_to_f64(dW), ref["dW"]) <= 1e-2
    h.close()


def test_step_host_async_pipeline(dev):
    """cce_step_host_async with two staging buffers rotated on a copy stream: different
    batches per step, each step's loss / gradients equal the synchronous path's bits."""
    import torch
    import paper_2601_02609_b200 as cce
    probs = [workload.make_problem(300, 128, 4000, seed=40 + i, ignore="bern40") for i in range(4)]
    _, W, _ = to_dev(probs[0], dev)
    Hs = [torch.from_numpy(p["H"].view(np.int16)).view(torch.bfloat16).pin_memory() for p in probs]
    ys = [torch.from_numpy(p["labels"]).pin_memory() for p in probs]
    h = cce.CCEHandle(vocab_total=4000)
    ws = h.workspace(300, 128, 4000, dev)
    nb = cce.cce_host_staging_bytes(300, 128)
    stages = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(2)]
    dHs = [torch.empty((300, 128), dtype=torch.bfloat16, device=dev) for _ in range(4)]
    dWs = [torch.empty((4000, 128), dtype=torch.bfloat16, device=dev) for _ in range(4)]
    losses = torch.empty(4, dtype=torch.float32).pin_memory()
    copy = torch.cuda.Stream()
    for i in range(4):
        cce.cce_step_host_async(h.h, Hs[i], ys[i], W, dHs[i], dWs[i], stages[i % 2], ws, losses[i], None, copy)
    torch.cuda.synchronize()
    for i in range(4):
        dH = torch.empty_like(dHs[i])
        dW = torch.empty_like(dWs[i])
        l_sync = cce.cce_step_host(h.h, Hs[i], ys[i], W, dH, dW, stages[0], ws)
        assert losses[i].item() == l_sync
        assert torch.equal(dH.view(torch.int16), dHs[i].view(torch.int16))
        assert torch.equal(dW.view(torch.int16), dWs[i].view(torch.int16))
        ref = oracle.cce(probs[i]["H"], probs[0]["W"], probs[i]["labels"])   # W is shared by the steps
        assert abs(l_sync - ref["loss"]) <= 2e-3
    h.close()


def test_nccl_path_on_one_rank(dev):
    """The vocabulary-sharded combine (a9 stats allgather, a10 dH all-reduce) through a
    real 1-rank NCCL communicator: the collectives are identities, so every output must
    be bit-identical to the plain path.  (More ranks need more GPUs: bench.py --gpus N.)"""
    import paper_2601_02609_b200 as cce
    p = workload.make_problem(700, 256, 9000, seed=23, ignore="bern40")
    H, W, y = to_dev(p, dev)
    comm = cce.cce_nccl_comm_init(1, cce.cce_nccl_unique_id(), 0)
    try:
        h1 = cce.CCEHandle(vocab_total=9000, nccl_comm=comm)
        a = run_gpu(H, W, y, handle=h1)
        h1.close()
    finally:
        cce.cce_nccl_comm_destroy(comm)
    b = run_gpu(H, W, y)
    assert a["loss"] == b["loss"]
    for k in ("lse_bits", "dH_bits", "dW_bits"):
        assert np.array_equal(a[k], b[k]), k


def test_unsupported_flag_combinations(dev):
    """Host-side validation on a real device: combinations the library does not implement
    are refused with CCE_ERR_UNSUPPORTED (2) before anything is enqueued."""
    import ctypes
    import paper_2601_02609_b200 as cce
    L = cce.lib()
    cfg = cce.cce_config()
    L.cce_config_default(ctypes.byref(cfg))
    cfg.vocab_total = 1000
    h = ctypes.c_void_p()
    for flags in (cce.FLAG_P2P_COMBINE | cce.FLAG_DH_SEQ_SHARD, cce.FLAG_P2P_COMBINE | cce.FLAG_EXTERNAL_COMBINE):
        cfg.flags = flags
        assert L.cce_create(ctypes.byref(h), ctypes.byref(cfg)) == 2, flags
    # world > 1 needs a communicator, the split-phase flag or the peer-memory flag
    cfg.flags = 0
    cfg.world, cfg.rank = 2, 0
    assert L.cce_create(ctypes.byref(h), ctypes.byref(cfg)) == 1
    cfg.flags = cce.FLAG_EXTERNAL_COMBINE
    assert L.cce_create(ctypes.byref(h), ctypes.byref(cfg)) == 0
    L.cce_destroy(h)


def test_split_phase_finish_without_pending_phase(dev):
    import torch
    import paper_2601_02609_b200 as cce
    h = cce.CCEHandle(vocab_total=1000, world=2, rank=0, vocab_offset=0, flags=cce.FLAG_EXTERNAL_COMBINE)
    with pytest.raises(cce.CCEError):
        cce.cce_forward_finish(h.h)
    with pytest.raises(cce.CCEError):
        cce.cce_backward_finish(h.h)
    h.close()


def test_autograd_refuses_a_stale_handle(dev):
    """the library keeps the forward state in the handle; two forwards on one
    handle before the first backward must fail loudly, not return the second's gradients."""
    import torch
    import paper_2601_02609_b200 as cce
    p = workload.make_problem(100, 64, 500, seed=31, ignore="bern10")
    H, W, y = to_dev(p, dev)
    Hr = H.clone().requires_grad_(True)
    h = cce.CCEHandle(vocab_total=500)
    l1 = cce.linear_cross_entropy(Hr, W, y, handle=h)
    l2 = cce.linear_cross_entropy(Hr, W, y, handle=h)
    l2.backward(retain_graph=True)              # the latest forward: fine
    with pytest.raises(RuntimeError, match="another forward"):
        l1.backward()
    h.close()


def test_rmsnorm_eps_must_be_positive(dev):
    import torch
    import paper_2601_02609_b200 as cce
    h = cce.CCEHandle(vocab_total=500)
    X = torch.zeros(8, 64, dtype=torch.bfloat16, device=dev)
    g = torch.ones(64, dtype=torch.bfloat16, device=dev)
    W = torch.zeros(500, 64, dtype=torch.bfloat16, device=dev)
    y = torch.zeros(8, dtype=torch.int32, device=dev)
    with pytest.raises(cce.CCEError) as ei:
        h.forward_rmsnorm(X, g, 0.0, W, y)
    assert ei.value.status == 1
    h.close()


@pytest.mark.parametrize("flags", [0, 2048], ids=["default", "design_b"])
def test_row_strided_inputs(dev, flags):
    """H and W as column slices of wider buffers (ldh = D + 64, ldw = D + 128, the padding
    columns NaN): the row strides reach the TMA maps and the padding is never read."""
    import torch
    p = workload.make_problem(500, 192, 7000, seed=51, ignore="bern40")
    H, W, y = to_dev(p, dev)
    Hb = torch.full((500, 192 + 64), float("nan"), dtype=torch.bfloat16, device=dev)
    Wb = torch.full((7000, 192 + 128), float("nan"), dtype=torch.bfloat16, device=dev)
    Hb[:, :192] = H
    Wb[:, :192] = W
    Hs, Ws = Hb[:, :192], Wb[:, :192]
    assert Hs.stride(0) == 256 and Ws.stride(0) == 320
    got = run_gpu(Hs, Ws, y, flags=flags)
    ref = oracle.cce(p["H"], p["W"], p["labels"])
    assert_parity(got, ref, p["labels"])
