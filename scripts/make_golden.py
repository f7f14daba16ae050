"""Write tests/golden/qwen05b_seed42.npz with the ORACLE's per-row LSE for every valid
row of the Qwen2.5-0.5B bench batch (seed 42), plus the labels and content hashes of
the generated H and W.  Calls only oracle/ and workload/ (never the CUDA path), so
full-size GPU parity tests can check sampled dW rows (which need every row's LSE)
without re-running ~1e12 fp64 MACs on the test box."""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import workload  # noqa: E402

p = workload.make_config("qwen05b", seed=42)
valid = np.nonzero(p["labels"] != -100)[0]
t = time.time()
lse, zy, _ = oracle.rows(p["H"], p["W"], p["labels"], valid)
print(f"oracle rows: {len(valid)} in {time.time() - t:.0f} s ({oracle.num_threads()} threads)")
out = os.path.join(ROOT, "tests", "golden", "qwen05b_seed42.npz")
np.savez_compressed(out, valid_rows=valid.astype(np.int32), lse=lse, zy=zy, labels=p["labels"],
                    H_sha256=hashlib.sha256(p["H"].tobytes()).hexdigest(),
                    W_sha256=hashlib.sha256(p["W"].tobytes()).hexdigest(),
                    source="oracle.rows (fp64) via scripts/make_golden.py; inputs workload.make_config('qwen05b', 42)")
print("wrote", out, os.path.getsize(out), "bytes")
