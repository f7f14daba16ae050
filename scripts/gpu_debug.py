"""Quick GPU diagnostics: parity on small shapes with per-output error printout,
then a rough timing of forward/backward at the Qwen2.5-0.5B head shape."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import oracle  # noqa: E402
import paper_2601_02609_b200 as cce  # noqa: E402
import workload  # noqa: E402
from cce_testutil import rel_fro, run_gpu, to_dev  # noqa: E402

dev = torch.device("cuda:0")
print(torch.cuda.get_device_name(0), cce.lib().cce_build_info().decode())

for (N, D, V, ign) in [(64, 64, 1000, "exact6"), (700, 128, 3000, "bern40"), (384, 896, 9000, "bern40")]:
    p = workload.make_problem(N, D, V, seed=1, ignore=ign)
    H, W, y = to_dev(p, dev)
    t = time.time()
    got = run_gpu(H, W, y)
    ref = oracle.cce(p["H"], p["W"], p["labels"])
    valid = p["labels"] != -100
    lse_err = np.max(np.abs(got["lse"][valid] - ref["lse"][valid]))
    print(f"N={N} D={D} V={V}: n_valid {got['n_valid']}/{ref['n_valid']} loss {got['loss']:.6f} vs {ref['loss']:.6f} "
          f"lse_maxabs {lse_err:.3e} dH {rel_fro(got['dH'], ref['dH']):.3e} dW {rel_fro(got['dW'], ref['dW']):.3e} "
          f"({time.time() - t:.1f}s)", flush=True)

if len(sys.argv) > 1 and sys.argv[1] == "perf":
    c = workload.CONFIGS["qwen05b"]
    p = workload.make_config("qwen05b", seed=42)
    H, W, y = to_dev(p, dev)
    h = cce.CCEHandle(vocab_total=c.V)
    dH = torch.empty(H.shape, dtype=torch.bfloat16, device=dev)
    dW = torch.empty(W.shape, dtype=torch.bfloat16, device=dev)
    one = torch.ones((), dtype=torch.float32, device=dev)
    for _ in range(3):
        h.forward(H, W, y)
        h.backward(one, dH, dW)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    fwd, bwd = [], []
    for _ in range(10):
        e[0].record()
        h.forward(H, W, y)
        e[1].record()
        h.backward(one, dH, dW)
        e[2].record()
        torch.cuda.synchronize()
        fwd.append(e[0].elapsed_time(e[1]))
        bwd.append(e[1].elapsed_time(e[2]))
    nv = int((p["labels"] != -100).sum())
    fl = 6.0 * nv * c.D * c.V
    t = np.median(fwd) + np.median(bwd)
    print(f"qwen05b: fwd {np.median(fwd):.3f} ms  bwd {np.median(bwd):.3f} ms  total {t:.3f} ms  "
          f"credited {fl / t / 1e9:.1f} TFLOP/s  tokens/s {c.N / t * 1e3:.0f}")
