#!/usr/bin/env python
"""Is the CCE_DBG_G=1 speed-up (dlogits TMA stores skipped) the energy of the stores, or
the tensor cores multiplying a ring of zeros?  Three variants, interleaved, one handle:

  normal     the real backward
  skip_real  stores skipped, the ring still holding the real dlogits of the last normal step
  skip_zero  stores skipped, the ring zeroed first (what a fresh workspace may hold)

Debug measurement only (results of the skip variants are garbage)."""
from __future__ import annotations

import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_2601_02609_b200 as cce
    import workload
    from bench import ClockSampler
    from paper_2601_02609_b200 import build as cce_build

    cce_build.build()
    dev = torch.device("cuda:0")
    c = workload.CONFIGS["qwen05b"]
    p = workload.make_config("qwen05b", seed=42)
    H = torch.from_numpy(p["H"].view(np.int16)).view(torch.bfloat16).to(dev)
    W = torch.from_numpy(p["W"].view(np.int16)).view(torch.bfloat16).to(dev)
    y = torch.from_numpy(p["labels"]).to(dev)
    loss = torch.empty((), dtype=torch.float32, device=dev)
    lse = torch.empty(c.N, dtype=torch.float32, device=dev)
    nvt = torch.empty((), dtype=torch.int32, device=dev)
    dH = torch.empty((c.N, c.D), dtype=torch.bfloat16, device=dev)
    dW = torch.empty((c.V, c.D), dtype=torch.bfloat16, device=dev)
    one = torch.ones((), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    h = cce.CCEHandle(vocab_total=c.V)
    ws = h.workspace(c.N, c.D, c.V, dev)

    def run(steps, dbg):
        if dbg:
            os.environ["CCE_DBG_G"] = str(dbg)
        else:
            os.environ.pop("CCE_DBG_G", None)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
        for i in range(steps):
            flush.zero_()
            cce.cce_forward(h.h, H, W, y, loss, lse, nvt, ws, stream)
            ev[i][0].record(stream)
            cce.cce_backward(h.h, one, dH, dW, stream)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        os.environ.pop("CCE_DBG_G", None)
        return [a.elapsed_time(b) for a, b in ev]

    res = {k: [] for k in ("normal", "skip_real", "skip_zero")}
    for _ in range(4):
        for name in ("normal", "skip_real", "skip_zero"):
            if name == "skip_zero":
                ws.zero_()
                torch.cuda.synchronize()
            else:
                run(3, 0 if name != "skip_zero" else 1)   # normal warm-up: the ring holds real dlogits
            time.sleep(1.0)
            smp = ClockSampler(0, period_ms=10)
            smp.start()
            time.sleep(0.2)
            t = run(20, 0 if name == "normal" else 1)
            ck = smp.stop()
            res[name].append((statistics.median(t), ck.get("sm_mhz") if ck else None))
    for k, v in res.items():
        print(f"{k:10s} backward median over rounds {statistics.median(x[0] for x in v):.3f} ms   rounds {v}", flush=True)
    h.close()


if __name__ == "__main__":
    main()
