#!/usr/bin/env python
"""Cost of the fused peer-memory exchange, measured on ONE B200 through the one-launch rank group
(cce_p2p_attach_group): world P ranks of the Qwen2.5-0.5B head (V/P vocabulary rows each) run
their backward queues side by side on 74/P CTA pairs of one launch, so a group step does the
same tensor work as the unsharded step PLUS the exchange (stats pushed by the merge kernel,
dH tiles reduced by the RED items, the finalize / scatter waits) and P-fold the replicated
per-rank kernels (label scan, gather, merge, finalize, scatter).  NOT a scaling number (one GPU
does all ranks' work): the difference to P = 1 is an upper bound on the exchange's cost PLUS
the P-fold replicated per-rank kernels, P forward launches of 1/P of the work each (their ramp
and tail), and P rank queues of 74/P pairs each finishing at the slowest one.
CUDA events around each step, L2 flush between steps, median of `steps`.  One JSON line."""
from __future__ import annotations

import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    import __graft_entry__
    import paper_2601_02609_b200 as cce
    import workload
    from cce_testutil import to_dev

    __graft_entry__.build()
    dev = torch.device("cuda:0")
    c = workload.CONFIGS["qwen05b"]
    p = workload.make_config("qwen05b", seed=42)
    H, W, y = to_dev(p, dev)
    one = torch.ones((), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    out = {"config": "qwen05b", "steps": steps, "note": __doc__.split("\n\n")[0].replace("\n", " ")}
    for world in (1, 2, 4, 8):
        hs, Ws, wss = [], [], []
        for r in range(world):
            lo, hi = cce.shard_range(c.V, r, world)
            flags = cce.FLAG_P2P_COMBINE if world > 1 else 0
            h = cce.CCEHandle(vocab_total=c.V, vocab_offset=lo, rank=r, world=world, flags=flags)
            hs.append(h)
            wss.append(h.workspace(c.N, c.D, hi - lo, dev))
            Ws.append(W[lo:hi].contiguous())
        if world > 1:
            cce.cce_p2p_attach_group([h.h for h in hs], wss, c.N, c.D)
        dHs = [torch.empty_like(H) for _ in hs]
        dWs = [torch.empty_like(Wr) for Wr in Ws]

        def step():
            for h, Wr in zip(hs, Ws):
                h.forward(H, Wr, y, want_lse=False)
            for h, dH, dW in zip(hs, dHs, dWs):
                h.backward(one, dH, dW)

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        ms = []
        for _ in range(steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            step()
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b))
        for h in hs:
            assert cce.cce_get_error(h.h) == 0
            h.close()
        out[f"P{world}"] = {"ms_median": statistics.median(ms), "ms_min": min(ms)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
