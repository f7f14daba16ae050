#!/usr/bin/env python
"""RMSNorm prologue at the Qwen2.5-0.5B head shape on one B200:
device time per step of cce_forward + cce_backward (H given) against
cce_forward_rmsnorm + cce_backward_rmsnorm (X and gamma given; the norm fused into the
row gather and the dH scatter), and the per-kernel times of the prologue's kernels
(cce_profile class "aux").  CUDA events, 256 MB L2 flush between steps.  One JSON line."""
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
    cfg = sys.argv[1] if len(sys.argv) > 1 else "qwen05b"
    c = workload.CONFIGS[cfg]
    p = workload.make_config(cfg, seed=42)
    X, g = workload.make_rmsnorm_inputs(42, c.N, c.D)
    t = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).to(dev)  # noqa: E731
    H, W, Xt, gt = t(p["H"]), t(p["W"]), t(X), t(g)
    y = torch.from_numpy(p["labels"]).to(dev)
    dl = torch.ones((), dtype=torch.float32, device=dev)
    dH = torch.empty_like(H)
    dW = torch.empty_like(W)
    dg = torch.empty_like(gt)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    res = {}
    for mode in ("plain", "rmsnorm"):
        h = cce.CCEHandle(vocab_total=c.V)

        def step():
            if mode == "plain":
                h.forward(H, W, y, want_lse=False)
                h.backward(dl, dH, dW)
            else:
                h.forward_rmsnorm(Xt, gt, 1e-6, W, y, want_lse=False)
                h.backward_rmsnorm(dl, dH, dg, dW)

        for _ in range(5):
            step()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        for a, b in ev:
            flush.zero_()
            a.record()
            step()
            b.record()
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in ev)
        cce.cce_profile_enable(h.h, True)
        cce.cce_profile_read(h.h)
        for _ in range(10):
            step()
        prof = cce.cce_profile_read(h.h)
        cce.cce_profile_enable(h.h, False)
        res[mode] = {"ms_median": ms[len(ms) // 2], "ms_min": ms[0],
                     "aux_ms_per_step": prof["aux"][0] / 10, "aux_launches_per_step": prof["aux"][1] / 10}
        h.close()
    print(json.dumps({"config": cfg, "N": c.N, "D": c.D, "V": c.V, "steps": 20, "ms": res,
                      "prologue_overhead_ms": res["rmsnorm"]["ms_median"] - res["plain"]["ms_median"],
                      "aux_delta_ms": res["rmsnorm"]["aux_ms_per_step"] - res["plain"]["aux_ms_per_step"]}))


if __name__ == "__main__":
    main()
