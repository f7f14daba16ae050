import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle, workload
from cce_testutil import run_gpu, to_dev, rel_fro
N, D, V, ign = [int(x) if x.isdigit() else x for x in sys.argv[1:5]]
flags = int(sys.argv[5]) if len(sys.argv) > 5 else 0
p = workload.make_problem(N, D, V, seed=N + V, ignore=ign)
H, W, y = to_dev(p, torch.device("cuda:0"))
ref = oracle.cce(p["H"], p["W"], p["labels"])
for trial in range(3):
    got = run_gpu(H, W, y, flags=flags)
    print("trial", trial, "loss", got["loss"], ref["loss"], "dH", rel_fro(got["dH"], ref["dH"]), "dW", rel_fro(got["dW"], ref["dW"]))
    C = 8192  # the library's backward chunk (compile-time CCE_CHUNK)
    for c0 in range(0, V, C):
        sl = slice(c0, min(V, c0 + C))
        print("   chunk", c0 // C, "dW relF", rel_fro(got["dW"][sl], ref["dW"][sl]))
    valid = p["labels"] != -100
    e = np.linalg.norm(got["dH"] - ref["dH"], axis=1) / np.maximum(np.linalg.norm(ref["dH"], axis=1), 1e-30)
    bad = np.nonzero(valid & (e > 0.05))[0]
    print("   dH bad rows", len(bad), bad[:20])
