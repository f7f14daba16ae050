"""Timeline of the persistent backward kernel's work queue (cce_debug_trace)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2601_02609_b200 as cce  # noqa: E402
import workload  # noqa: E402
from cce_testutil import to_dev  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "qwen05b"
out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "trace.npy")
dev = torch.device("cuda:0")
c = workload.CONFIGS[cfg]
p = workload.make_config(cfg, seed=42)
H, W, y = to_dev(p, dev)
h = cce.CCEHandle(vocab_total=c.V)
dH = torch.empty(H.shape, dtype=torch.bfloat16, device=dev)
dW = torch.empty(W.shape, dtype=torch.bfloat16, device=dev)
one = torch.ones((), dtype=torch.float32, device=dev)
for _ in range(3):
    h.forward(H, W, y)
    h.backward(one, dH, dW)
buf = torch.zeros(64 * 200000, dtype=torch.uint8, device=dev)
cce.cce_debug_trace(h.h, buf)
h.forward(H, W, y)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
h.backward(one, dH, dW)
e1.record()
torch.cuda.synchronize()
cce.cce_debug_trace(h.h, None)
rec = buf.view(torch.int64).view(-1, 8).cpu().numpy().astype(np.uint64)
rec = rec[rec[:, 5] > 0]
np.save(out, rec)
q = (rec[:, 0] >> 32).astype(np.int64)
typ = ((rec[:, 0] >> 16) & 0xFFFF).astype(np.int64)
ch = (rec[:, 0] & 0xFFFF).astype(np.int64)
t0 = rec[:, 2].min()
deq, rdy, ep0, ep1 = [(rec[:, i] - t0).astype(np.float64) / 1e3 for i in (2, 3, 4, 5)]
print(f"{cfg}: backward {e0.elapsed_time(e1):.3f} ms (events), items {len(rec)}, span {ep1.max():.1f} us, "
      f"chunk={os.environ.get('CCE_CHUNK', '8192')}")
for t, nm in enumerate(["G", "DW", "DH"]):
    m = typ == t
    if not m.any():
        continue
    print(f"  {nm}: n={m.sum():5d} dep_wait mean {np.mean(rdy[m]-deq[m]):7.2f} us max {np.max(rdy[m]-deq[m]):7.1f} "
          f"sum {np.sum(rdy[m]-deq[m]):9.0f} | epi {np.mean(ep1[m]-ep0[m]):6.2f} us | deq->epi_end {np.mean(ep1[m]-deq[m]):7.2f} us")
for cc in range(0, ch.max() + 1, max(1, (ch.max() + 1) // 6)):
    g = (typ == 0) & (ch == cc)
    w = (typ != 0) & (ch == cc)
    print(f"  chunk {cc:2d}: G [{deq[g].min():8.1f} .. {ep1[g].max():8.1f}]  W [{deq[w].min():8.1f} .. {ep1[w].max():8.1f}]")
