#!/usr/bin/env python
"""Energy per FLOP of the pair kernels against a plain cuBLAS GEMM, on one B200 (Qwen2.5-0.5B
head).  Each workload runs back to back for ~2 s while nvidia-smi samples power and SM clock
every 20 ms; reported: executed TFLOP/s, median power, median SM clock, pJ per executed FLOP.
  forward  cce_forward only              (2 N_valid D V executed FLOPs per call)
  backward cce_backward only (one forward first; every call recomputes: 6 N_valid D V)
  designb_forward / designb_backward  the same with CCE_FLAG_DESIGN_B (4 N_valid D V each)
  cublas   torch.matmul bf16 8192 x 8192 x 8192 (2 M N K)
One JSON line."""
from __future__ import annotations

import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    import __graft_entry__
    import paper_2601_02609_b200 as cce
    import workload
    from bench import ClockSampler
    from cce_testutil import to_dev

    __graft_entry__.build()
    dev = torch.device("cuda:0")
    c = workload.CONFIGS["qwen05b"]
    p = workload.make_config("qwen05b", seed=42)
    H, W, y = to_dev(p, dev)
    nv = int((p["labels"] != -100).sum())
    h = cce.CCEHandle(vocab_total=c.V)
    dH, dW = torch.empty_like(H), torch.empty_like(W)
    one = torch.ones((), dtype=torch.float32, device=dev)
    a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    b = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    nvd = nv * c.D * c.V
    h.forward(H, W, y, want_lse=False)
    h.backward(one, dH, dW)
    hb = cce.CCEHandle(vocab_total=c.V, flags=cce.FLAG_DESIGN_B)
    hb.forward(H, W, y, want_lse=False)
    hb.backward(one, dH, dW)
    work = {
        "forward": (lambda: h.forward(H, W, y, want_lse=False), 2 * nvd),
        "backward": (lambda: h.backward(one, dH, dW), 6 * nvd),
        # design B: the forward also accumulates the dH numerator (4 N_valid D V), the backward
        # recomputes the logits and forms dW (4 N_valid D V)
        "designb_forward": (lambda: hb.forward(H, W, y, want_lse=False), 4 * nvd),
        "designb_backward": (lambda: hb.backward(one, dH, dW), 4 * nvd),
        "cublas": (lambda: torch.matmul(a, b), 2 * 8192 ** 3),
    }
    out = {"config": "qwen05b", "n_valid": nv}
    for name, (fn, flops) in work.items():
        time.sleep(3.0)  # cool down between workloads
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        smp = ClockSampler(0, period_ms=20)
        smp.start()
        smp.wait_first()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 0
        e0.record()
        while time.perf_counter() - t0 < 2.0:
            for _ in range(10):
                fn()
            n += 10
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        smp.stop(window=(t0, t1))
        rows = [r for t, r in smp.stamped if t0 + 0.2 <= t <= t1]  # (skip the first 0.2 s ramp)
        pw = [float(r[3]) for r in rows if len(r) > 3 and r[3].replace(".", "").isdigit()]
        mhz = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        ms = e0.elapsed_time(e1)
        tf = flops * n / (ms * 1e-3) / 1e12
        pmed = statistics.median(pw) if pw else None
        out[name] = {"calls": n, "tflops_executed": round(tf, 1), "power_w_median": pmed,
                     "sm_mhz_median": statistics.median(mhz) if mhz else None,
                     "pj_per_flop": round(pmed / (tf * 1e12) * 1e12, 4) if pmed else None}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
