#!/usr/bin/env python
"""Context (not the product): the same fused linear cross-entropy fwd+bwd done the plain
PyTorch way on the same B200 -- materialised logits (cuBLAS bf16 GEMM, fp32 logits),
F.cross_entropy(ignore_index=-100) and autograd -- at the Qwen2.5-0.5B head shape, next to
the library's step, in one process.  Also the plain cuBLAS GEMM time for the three
contractions (logits, dH, dW) at the same shapes, i.e. what a library GEMM reaches on them
in the same power regime.  CUDA events, L2 flush between steps.  One JSON line."""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import __graft_entry__
    import paper_2601_02609_b200 as cce
    import workload

    __graft_entry__.build()
    dev = torch.device("cuda:0")
    c = workload.CONFIGS["qwen05b"]
    p = workload.make_config("qwen05b", seed=42)
    t = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).to(dev)  # noqa: E731
    H, W = t(p["H"]), t(p["W"])
    y = torch.from_numpy(p["labels"]).to(dev)
    yl = y.long()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def timeit(fn, steps=10, warm=3):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in ev:
            flush.zero_()
            a.record()
            fn()
            b.record()
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in ev)
        return ms[len(ms) // 2]

    res = {}
    # the library
    h = cce.CCEHandle(vocab_total=c.V)
    dH = torch.empty_like(H)
    dW = torch.empty_like(W)
    one = torch.ones((), dtype=torch.float32, device=dev)

    def ours():
        h.forward(H, W, y, want_lse=False)
        h.backward(one, dH, dW)
    res["library_fwd_bwd_ms"] = timeit(ours)
    h.close()

    # PyTorch eager: materialised fp32 logits [N, V] (4.98 GB), cross_entropy, autograd
    Hp = H.clone().requires_grad_(True)
    Wp = W.clone().requires_grad_(True)

    def eager():
        Hp.grad = None
        Wp.grad = None
        logits = (Hp @ Wp.T).float()
        loss = torch.nn.functional.cross_entropy(logits, yl, ignore_index=-100)
        loss.backward()
    torch.cuda.reset_peak_memory_stats(dev)
    res["torch_eager_fwd_bwd_ms"] = timeit(eager, steps=5)
    res["torch_eager_peak_alloc_GB"] = torch.cuda.max_memory_allocated(dev) / 1e9
    del Hp, Wp

    # plain cuBLAS bf16 GEMMs of the three contractions over the valid rows (no epilogue work):
    valid = torch.nonzero(y != -100).squeeze(1)
    Hv = H[valid].contiguous()
    nv = Hv.shape[0]
    G = torch.randn(nv, c.V, device=dev, dtype=torch.bfloat16) * 1e-3
    S = torch.empty(nv, c.V, device=dev, dtype=torch.bfloat16)

    def gemms():
        torch.matmul(Hv, W.T, out=S)        # logits      2 nv V D
        torch.matmul(G, W)                  # dH          2 nv V D
        torch.matmul(G.T, Hv)               # dW          2 nv V D
    ms = timeit(gemms)
    flops = 3 * 2.0 * nv * c.V * c.D
    res["cublas_3_gemms_ms"] = ms
    res["cublas_3_gemms_tflops"] = flops / (ms / 1e3) / 1e12
    res["library_executed_tflops"] = 8.0 * nv * c.V * c.D / (res["library_fwd_bwd_ms"] / 1e3) / 1e12
    res["n_valid"] = int(nv)
    res["note"] = ("library executes 8 nv V D (forward logits + recompute + dW + dH); cuBLAS line is 3 plain GEMMs "
                   "(6 nv V D) with bf16 outputs, no softmax, no ignore handling")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
