"""Write tests/golden/<config>_seed42.npz for BASELINE.json configs[2..4] (mem, llama8b,
qwen7b; 0% ignored, seed 42): the ORACLE's fp64 per-row LSE and target logit for EVERY
valid row, plus the labels and content hashes of the generated H and W.

Calls only oracle/ and workload/ (never the CUDA path).  With every row's LSE stored, the
full-size GPU tests (tests/test_gpu_configs.py) can check the mean loss exactly and sampled
dW rows through oracle.dW_rows without re-running ~1e13 fp64 MACs per config on the test box.
Runtime here (8 vCPU, memory-bound row-at-a-time fp64 logits): roughly 0.5 / 1 / 2 hours.

usage: python scripts/make_golden_configs.py [mem llama8b qwen7b]"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import workload  # noqa: E402

names = sys.argv[1:] or ["mem", "llama8b", "qwen7b"]
for name in names:
    p = workload.make_config(name, seed=42)
    valid = np.nonzero(p["labels"] != -100)[0]
    t = time.time()
    lse = np.zeros(len(valid)); zy = np.zeros(len(valid))
    # in slices so progress is visible and a crash loses little
    step = 1024
    for i in range(0, len(valid), step):
        l, z, _ = oracle.rows(p["H"], p["W"], p["labels"], valid[i:i + step])
        lse[i:i + step] = l; zy[i:i + step] = z
        print(f"{name}: {i + len(l)}/{len(valid)} rows, {time.time() - t:.0f} s", flush=True)
    out = os.path.join(ROOT, "tests", "golden", f"{name}_seed42.npz")
    np.savez_compressed(out, valid_rows=valid.astype(np.int32), lse=lse, zy=zy, labels=p["labels"],
                        H_sha256=hashlib.sha256(p["H"].tobytes()).hexdigest(),
                        W_sha256=hashlib.sha256(p["W"].tobytes()).hexdigest(),
                        source=f"oracle.rows (fp64) via scripts/make_golden_configs.py; inputs "
                               f"workload.make_config('{name}', 42)")
    print("wrote", out, os.path.getsize(out), "bytes", flush=True)
