#!/usr/bin/env python
"""Per-rank compute of the vocabulary-sharded path, measured on ONE B200 (this run has one
GPU): for world P in 1, 2, 4, 8, each rank's cce_forward + cce_backward on its V/P shard is
run and timed alone (CUDA events, L2 flush between steps), with the split-phase combine
(CCE_FLAG_EXTERNAL_COMBINE) standing in for the NCCL exchange, which is NOT timed.  Reports
max over ranks and t(1) / max_r t(P): the compute-only scaling a P-GPU run could reach
before communication (stats allgather ~3.2 MB, dH all-reduce Npad x D fp32).  One JSON line."""
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
    t = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).to(dev)  # noqa: E731
    H, W = t(p["H"]), t(p["W"])
    y = torch.from_numpy(p["labels"]).to(dev)
    one = torch.ones((), dtype=torch.float32, device=dev)
    dH = torch.empty_like(H)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {"config": cfg, "N": c.N, "D": c.D, "V": c.V, "note": "compute only, one rank at a time on one GPU; "
           "the exchange (split-phase, untimed) replaces NCCL"}
    for world in (1, 2, 4, 8):
        per_rank = []
        for r in range(world):
            lo, hi = cce.shard_range(c.V, r, world)
            Wr = W[lo:hi].contiguous()
            dW = torch.empty_like(Wr)
            flags = cce.FLAG_EXTERNAL_COMBINE if world > 1 else 0
            h = cce.CCEHandle(vocab_total=c.V, vocab_offset=lo, rank=r, world=world, flags=flags)
            so, sao, dho, npad = cce.cce_combine_offsets(h.h, c.N, c.D, hi - lo)

            def step():
                h.forward(H, Wr, y, want_lse=False)
                if world > 1:   # stand-in for the allgather (one copy launch): this rank's stats in every slot
                    st = h._ws[so:so + npad * 16]
                    h._ws[sao:sao + world * npad * 16].view(world, npad * 16).copy_(st.expand(world, -1))
                    cce.cce_forward_finish(h.h)
                h.backward(one, dH, dW)
                if world > 1:
                    cce.cce_backward_finish(h.h)

            for _ in range(3):
                step()
            torch.cuda.synchronize()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
            for a, b in ev:
                flush.zero_()
                a.record()
                step()
                b.record()
            torch.cuda.synchronize()
            ms = sorted(a.elapsed_time(b) for a, b in ev)
            per_rank.append(ms[len(ms) // 2])
            if r == 0:   # per-class kernel time of rank 0 (cce_profile)
                cce.cce_profile_enable(h.h, True)
                cce.cce_profile_read(h.h)
                for _ in range(5):
                    step()
                prof = {k: round(v[0] / 5, 4) for k, v in cce.cce_profile_read(h.h).items() if v[1]}
                cce.cce_profile_enable(h.h, False)
            h.close()
        out[f"P{world}"] = {"max_rank_ms": max(per_rank), "min_rank_ms": min(per_rank), "rank0_kernel_ms": prof,
                             "per_rank_ms": [round(x, 4) for x in per_rank]}
    t1 = out["P1"]["max_rank_ms"]
    for world in (2, 4, 8):
        out[f"P{world}"]["compute_scaling"] = t1 / out[f"P{world}"]["max_rank_ms"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
