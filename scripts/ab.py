#!/usr/bin/env python
"""A/B timing of kernel variants on the bench workload, interleaved in one process
so that box-to-box and clock drift affect every variant alike.

  python scripts/ab.py name=flags[@path/to/libcce.so] ... [--rounds 3] [--steps 20] [--config qwen05b]

Each variant gets its own handle, optionally on another build of libcce.so (the library
reads no environment: compile-time variants are separate builds).  Prints per-variant
median step / forward / backward times in ms.
"""
from __future__ import annotations

import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="qwen05b")
    ap.add_argument("--vslice", type=int, default=0, help="time one vocabulary shard: the first n rows of W")
    ap.add_argument("--sample-ms", type=int, default=20)
    ap.add_argument("--rest", type=float, default=1.0, help="idle seconds before each measurement")
    args = ap.parse_args()

    import numpy as np
    import torch

    import paper_2601_02609_b200 as cce
    import workload
    from paper_2601_02609_b200 import build as cce_build

    cce_build.build()
    dev = torch.device("cuda:0")
    c = workload.CONFIGS[args.config]
    p = workload.make_config(args.config, seed=42)
    H = torch.from_numpy(p["H"].view(np.int16)).view(torch.bfloat16).to(dev)
    W = torch.from_numpy(p["W"].view(np.int16)).view(torch.bfloat16).to(dev)
    y = torch.from_numpy(p["labels"]).to(dev)
    V = c.V
    if args.vslice:
        V = args.vslice
        W = W[:V].contiguous()
        y = torch.where(y >= 0, y % V, y)
    loss = torch.empty((), dtype=torch.float32, device=dev)
    lse = torch.empty(c.N, dtype=torch.float32, device=dev)
    nvt = torch.empty((), dtype=torch.int32, device=dev)
    dH = torch.empty((c.N, c.D), dtype=torch.bfloat16, device=dev)
    dW = torch.empty((V, c.D), dtype=torch.bfloat16, device=dev)
    one = torch.ones((), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    vs = []
    libs = {}
    main_lib = cce.lib()
    for spec in args.variants:
        spec, _, libpath = spec.partition("@")   # optional: another build of libcce.so
        name, rest = spec.split("=", 1)
        flags, _, envs = rest.partition(":")
        env = dict(kv.split("=", 1) for kv in envs.split(",") if kv)
        vs.append((name, int(flags), env))
        if libpath:
            saved = cce.LIB_PATH
            cce.LIB_PATH, cce._lib = libpath, None
            libs[name] = cce.lib()
            cce.LIB_PATH, cce._lib = saved, main_lib
        else:
            libs[name] = main_lib

    handles = {}
    for name, flags, env in vs:
        cce._lib = libs[name]
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        h = cce.CCEHandle(vocab_total=V, flags=flags)
        # WSOFF=<bytes>: place the workspace at this offset from a 2 MiB-aligned base
        off = int(env.get("WSOFF", "-1"))
        if off >= 0:
            need = cce.cce_workspace_bytes(h.h, c.N, c.D, V)
            raw = torch.empty(need + off + (4 << 20), dtype=torch.uint8, device=dev)
            base = (-raw.data_ptr()) % (2 << 20)
            ws = raw[base + off: base + off + need]
            h._ws_keep = raw
        else:
            ws = h.workspace(c.N, c.D, V, dev)
        cce.cce_forward(h.h, H, W, y, loss, lse, nvt, ws, stream)
        cce.cce_backward(h.h, one, dH, dW, stream)
        torch.cuda.synchronize()
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        handles[name] = (h, ws)

    from bench import ClockSampler
    import time
    res = {name: {"step": [], "fwd": [], "bwd": [], "mhz": []} for name, _, _ in vs}
    import random
    rng = random.Random(1234)
    for r in range(args.rounds):
        order = list(vs)
        rng.shuffle(order)          # no position bias from the GPU's thermal / power drift
        for name, _, _ in order:
            h, ws = handles[name]
            cce._lib = libs[name]
            time.sleep(args.rest)
            smp = ClockSampler(0, period_ms=args.sample_ms)
            smp.start()
            time.sleep(0.2)
            for _ in range(args.warmup):
                cce.cce_forward(h.h, H, W, y, loss, lse, nvt, ws, stream)
                cce.cce_backward(h.h, one, dH, dW, stream)
            torch.cuda.synchronize()
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
            for i in range(args.steps):
                flush.zero_()
                ev[i][0].record(stream)
                cce.cce_forward(h.h, H, W, y, loss, lse, nvt, ws, stream)
                ev[i][1].record(stream)
                cce.cce_backward(h.h, one, dH, dW, stream)
                ev[i][2].record(stream)
            torch.cuda.synchronize()
            ck = smp.stop()
            if ck and ck["sm_mhz"]:
                res[name]["mhz"].append((ck["sm_mhz"], ck.get("power_w_max"), ck.get("reasons")))
            res[name].setdefault("rounds", []).append(statistics.median([a.elapsed_time(c_) for a, b, c_ in ev]))
            res[name]["step"] += [a.elapsed_time(c_) for a, b, c_ in ev]
            res[name]["fwd"] += [a.elapsed_time(b) for a, b, c_ in ev]
            res[name]["bwd"] += [b.elapsed_time(c_) for a, b, c_ in ev]
    for name, _, _ in vs:
        d = res[name]
        print(f"{name:24s} step {statistics.median(d['step']):7.3f} ms  fwd {statistics.median(d['fwd']):7.3f}"
              f"  bwd {statistics.median(d['bwd']):7.3f}  (min step {min(d['step']):.3f})  per-round medians "
              f"{[round(x, 3) for x in d['rounds']]}  sm MHz {d['mhz']}", flush=True)
    for name, (h, _) in handles.items():
        cce._lib = libs[name]
        h.close()


if __name__ == "__main__":
    main()
