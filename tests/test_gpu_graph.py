"""The library is stream-ordered with no host synchronisation in cce_forward / cce_backward,
so a whole training step can be captured in a CUDA graph and replayed; the replay must be
bit-identical to the eager launches (scripts/bench_graph.py times it: no material gain at
P = 1, the eager launch gaps are already ~20 us per 4 ms step)."""
import numpy as np
import pytest

import workload
from cce_testutil import to_dev

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("flags", [0, 2048], ids=["default", "design_b"])
def test_step_captured_in_cuda_graph(flags):
    import torch
    import __graft_entry__
    import paper_2601_02609_b200 as cce
    __graft_entry__.build()
    dev = torch.device("cuda:0")
    p = workload.make_problem(600, 256, 20000, seed=41, ignore="bern40")
    H, W, y = to_dev(p, dev)
    h = cce.CCEHandle(vocab_total=20000, flags=flags)
    ws = h.workspace(600, 256, 20000, dev)
    loss = torch.empty((), dtype=torch.float32, device=dev)
    lse = torch.empty(600, dtype=torch.float32, device=dev)
    nv = torch.empty((), dtype=torch.int32, device=dev)
    dH = torch.empty_like(H)
    dW = torch.empty_like(W)
    one = torch.ones((), dtype=torch.float32, device=dev)
    s = torch.cuda.Stream(device=dev)

    def step():
        cce.cce_forward(h.h, H, W, y, loss, lse, nv, ws, s)
        cce.cce_backward(h.h, one, dH, dW, s)

    with torch.cuda.stream(s):
        step()
    torch.cuda.synchronize()
    ref = [t.view(torch.int32 if t.dtype == torch.float32 else torch.int16).clone() for t in (loss.view(1), lse, dH, dW)]
    for t in (loss, lse, dH, dW):
        t.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    for _ in range(2):
        for t in (loss, lse, dH, dW):
            t.zero_()
        g.replay()
        torch.cuda.synchronize()
        got = [t.view(torch.int32 if t.dtype == torch.float32 else torch.int16) for t in (loss.view(1), lse, dH, dW)]
        for a, b in zip(ref, got):
            assert torch.equal(a, b)
    h.close()
