#!/usr/bin/env python
"""Fused optimizer step at the Qwen2.5-0.5B head shape on one B200:
per-step device time of
  plain    cce_forward + cce_backward (bf16 dW; no optimizer)
  unfused  cce_forward + cce_backward (fp32 dW) + cce_adamw_step (standalone fused AdamW)
  fused    cce_forward + cce_backward_adamw (AdamW in the dW epilogue; dW never in HBM), W in place
  fused_wout  the same with the new bf16 weights written to a second buffer (no dH wait)
with fp32 master weights and moments, CUDA events on the launching stream, a 256 MB L2
flush between steps.  Prints one JSON line."""
from __future__ import annotations

import argparse
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
    if os.environ.get("CCE_LIB"):  # time another build of libcce.so
        cce.LIB_PATH = os.environ["CCE_LIB"]

    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="qwen05b")
    args = ap.parse_args()
    __graft_entry__.build()
    if os.environ.get("CCE_LIB"):  # A/B another build of libcce.so
        cce.LIB_PATH = os.environ["CCE_LIB"]
    dev = torch.device("cuda:0")
    c = workload.CONFIGS[args.config]
    p = workload.make_config(args.config, seed=42)
    H = torch.from_numpy(p["H"].view(np.int16)).view(torch.bfloat16).to(dev)
    W = torch.from_numpy(p["W"].view(np.int16)).view(torch.bfloat16).to(dev)
    y = torch.from_numpy(p["labels"]).to(dev)
    V, D = W.shape
    master = W.float()
    m = torch.zeros(V, D, dtype=torch.float32, device=dev)
    v = torch.zeros(V, D, dtype=torch.float32, device=dev)
    dl = torch.ones((), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    res = {}
    W_alt = torch.empty_like(W)
    for mode in ("plain", "unfused", "fused", "fused_wout"):
        h = cce.CCEHandle(vocab_total=V, flags=cce.FLAG_GRAD_FP32 if mode == "unfused" else 0)
        gdt = torch.float32 if mode == "unfused" else torch.bfloat16
        dH = torch.empty(H.shape, dtype=gdt, device=dev)
        dW = torch.empty(V, D, dtype=gdt, device=dev) if mode != "fused" else None
        step_no = [0]

        def step():
            step_no[0] += 1
            h.forward(H, W, y, want_lse=False)
            if mode == "plain":
                h.backward(dl, dH, dW)
                return
            opt = cce.adamw_params(m, v, lr=1e-6, step=step_no[0], beta1=0.9, beta2=0.999, eps=1e-8,
                                   weight_decay=0.0, master=master, W_out=W_alt if mode == "fused_wout" else None)
            if mode == "unfused":
                h.backward(dl, dH, dW)
                cce.cce_adamw_step(opt, dW, V * D, W)
            else:
                h.backward_adamw(dl, dH, opt)

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record()
            step()
            ev[i][1].record()
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in ev)
        res[mode] = {"ms_median": ms[len(ms) // 2], "ms_mean": sum(ms) / len(ms), "ms_min": ms[0]}
        h.close()
    state_bytes = V * D * (4 + 4 + 4)          # master, m, v read and written once each
    out = {"config": args.config, "N": c.N, "D": D, "V": V, "steps": args.steps, "warmup": args.warmup,
           "l2": "256 MB flush between steps", "ms": res,
           "adamw_overhead_ms": {"unfused": res["unfused"]["ms_median"] - res["plain"]["ms_median"],
                                 "fused": res["fused"]["ms_median"] - res["plain"]["ms_median"],
                                 "fused_wout": res["fused_wout"]["ms_median"] - res["plain"]["ms_median"]},
           "optimizer_state_bytes_rw": 2 * state_bytes + V * D * 2,
           "unfused_extra_bytes": V * D * (4 + 4) - V * D * 2}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
