#!/usr/bin/env python
"""Run `steps` forward + backward steps of a workload config on cuda:0 (no timing, no checks):
the target for ncu captures of configs other than the bench's.

  python scripts/run_once.py CONFIG [--vslice n] [--steps k]

--vslice n: one vocabulary shard's kernels -- the first n rows of W (labels taken mod n), i.e.
the per-rank work of a vocabulary-sharded run (e.g. configs[4] on 8 GPUs: n = 19008)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--vslice", type=int, default=0)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_2601_02609_b200 as cce
    import workload
    if os.environ.get("CCE_LIB"):  # another build of libcce.so
        cce.LIB_PATH = os.environ["CCE_LIB"]
    from cce_testutil import to_dev

    dev = torch.device("cuda:0")
    c = workload.CONFIGS[args.config]
    V = args.vslice or c.V
    p = workload.make_config(args.config, seed=42, w_rows=(0, V))
    H, W, y = to_dev(p, dev)
    if args.vslice:
        y = torch.where(y >= 0, y % V, y)
    h = cce.CCEHandle(vocab_total=V)
    dH, dW = torch.empty_like(H), torch.empty_like(W)
    one = torch.ones((), dtype=torch.float32, device=dev)
    for _ in range(args.steps):
        loss, _, _ = h.forward(H, W, y, want_lse=False)
        h.backward(one, dH, dW)
    torch.cuda.synchronize()
    print(f"{args.config} V={V}: loss {loss.item():.6f}")


if __name__ == "__main__":
    main()
