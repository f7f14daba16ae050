"""Per-item timeline of the pair kernels (forward + backward) via cce_debug_trace."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2601_02609_b200 as cce  # noqa: E402

if os.environ.get("CCE_LIB"):  # trace another build of libcce.so
    cce.LIB_PATH = os.environ["CCE_LIB"]
import workload  # noqa: E402
from cce_testutil import to_dev  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "qwen05b"
out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "trace_pair.npz")
dev = torch.device("cuda:0")
c = workload.CONFIGS[cfg]
p = workload.make_config(cfg, seed=42)
H, W, y = to_dev(p, dev)
V = c.V
if os.environ.get("CCE_VSLICE"):  # the kernels of one vocabulary shard: the first n rows of W
    V = int(os.environ["CCE_VSLICE"])
    W = W[:V].contiguous()
    y = torch.where(y >= 0, y % V, y)
h = cce.CCEHandle(vocab_total=V, flags=int(os.environ.get("CCE_FLAGS", "0")))
dH = torch.empty(H.shape, dtype=torch.bfloat16, device=dev)
dW = torch.empty(W.shape, dtype=torch.bfloat16, device=dev)
one = torch.ones((), dtype=torch.float32, device=dev)
ADAMW = os.environ.get("CCE_ADAMW")  # "1": fused AdamW, W in place; "2": W_out double buffer
if ADAMW:
    st = {k: torch.zeros(W.shape, dtype=torch.float32, device=dev) for k in ("m", "v")}
    master = W.float()
    W2 = torch.empty_like(W)
    opt = cce.adamw_params(st["m"], st["v"], lr=1e-6, step=1, master=master, W_out=W2 if ADAMW == "2" else None)


def bwd():
    if ADAMW:
        h.backward_adamw(one, dH, opt)
    else:
        h.backward(one, dH, dW)


for _ in range(3):
    h.forward(H, W, y)
    bwd()
CAP = 60000
buf = torch.zeros(2 * CAP * 128, dtype=torch.uint8, device=dev)
cce.cce_debug_trace(h.h, buf)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ev[0].record()
h.forward(H, W, y)
ev[1].record()
bwd()
ev[2].record()
torch.cuda.synchronize()
cce.cce_debug_trace(h.h, None)
allrec = buf.view(torch.int64).view(2, CAP, 16).cpu().numpy().astype(np.uint64)
np.savez(out, bwd=allrec[0], fwd=allrec[1])
print(f"{cfg}: fwd {ev[0].elapsed_time(ev[1]):.3f} ms, bwd {ev[1].elapsed_time(ev[2]):.3f} ms")
NAMES = {0: "FWD", 1: "G", 2: "DW", 3: "DH", 5: "RED", 6: "OPT"}
for name, rec in (("forward", allrec[1]), ("backward", allrec[0])):
    rec = rec[rec[:, 5] > 0]
    if len(rec) == 0:
        continue
    typ = ((rec[:, 0] >> 16) & 0xFFFF).astype(np.int64)
    t0 = rec[:, 2].min()
    f = lambda i: (rec[:, i].astype(np.float64) - float(t0)) / 1e3  # noqa: E731
    deq, rdy, ep0, ep1, l0, l1, m0, m1 = [f(i) for i in (2, 3, 4, 5, 8, 9, 10, 11)]
    fw = rec[:, 12].astype(np.float64) / 1e3
    kb = rec[:, 7].astype(np.float64)
    cyc = rec[:, 13].astype(np.float64)
    lat = rec[:, 15].astype(np.float64)
    print(f" {name}: items {len(rec)} span {ep1.max():.1f} us; sum of dep-wait {np.sum(rdy-deq):.0f} us")
    # DW / DH items grouped by their hidden tile (column offset n0): a narrow tail tile shows up
    npk = np.where((typ == 2) | (typ == 3), (rec[:, 6] & np.uint64(0xFFFFFFFF)).astype(np.int64), 0)
    for t, npv in sorted(set(zip(typ.tolist(), npk.tolist()))):
        m = (typ == t) & (npk == npv)
        print(f"   {NAMES[t]:3s}{'@' + str(npv) if npv else '':5s} n={m.sum():6d} kb={kb[m].mean():5.1f} | mma window {np.mean(m1[m]-m0[m]):7.2f} us "
              f"(full-wait {np.mean(fw[m]):6.2f}) | load window {np.mean(l1[m]-l0[m]):7.2f} | "
              f"mma_end->epi0 {np.mean(ep0[m]-m1[m]):6.2f} | epi {np.mean(ep1[m]-ep0[m]):6.2f} | dep-wait {np.mean(rdy[m]-deq[m]):6.2f} | "
              f"per-kb {np.mean((m1[m]-m0[m])/np.maximum(kb[m],1)):.3f} us, {np.mean(cyc[m]/np.maximum(kb[m],1)):.0f} cyc"
              f" (clock {np.sum(cyc[m])/np.sum((m1[m]-m0[m])*1e3):.2f} GHz) | issue->full {np.mean(lat[m]/np.maximum(kb[m],1)):.0f} cyc")
    # per CTA pair (leader SM): MMA-window occupancy, idle before the first and after the last item
    sm = rec[:, 1].astype(np.int64)
    busy, head, tail = [], [], []
    for s_ in np.unique(sm):
        m = sm == s_
        busy.append(np.sum(m1[m] - m0[m]) / ep1.max())
        head.append(m0[m].min())
        tail.append(ep1.max() - m1[m].max())
    print(f"   per pair: MMA window {np.mean(busy)*100:.1f}% of the span (min {np.min(busy)*100:.1f}%), "
          f"first MMA at {np.mean(head):.1f} us (max {np.max(head):.1f}), idle after the last MMA {np.mean(tail):.1f} us "
          f"(max {np.max(tail):.1f})")
