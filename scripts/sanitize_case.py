"""One forward + backward through the C ABI on a small problem, for compute-sanitizer
(memcheck / racecheck / synccheck).  usage: python scripts/sanitize_case.py N D V [flags] [p2p]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2601_02609_b200 as cce  # noqa: E402
import workload  # noqa: E402
from cce_testutil import assert_parity, run_gpu, to_dev  # noqa: E402

N, D, V = (int(a) for a in sys.argv[1:4])
flags = int(sys.argv[4]) if len(sys.argv) > 4 else 0
p = workload.make_problem(N, D, V, seed=N + V, ignore="bern40")
H, W, y = to_dev(p, torch.device("cuda:0"))
got = run_gpu(H, W, y, flags=flags)
got2 = run_gpu(H, W, y, flags=flags)      # a second step on fresh handles
ref = oracle.cce(p["H"], p["W"], p["labels"])
assert_parity(got, ref, p["labels"])
assert_parity(got2, ref, p["labels"])
print(f"sanitize case N={N} D={D} V={V} flags={flags}: parity ok")
