"""Analyse a backward trace (scripts/trace_pair.py output): per-cluster producer idle
time split into 'waiting for a dependency' and 'ring empty', and per-chunk timelines."""
import sys
import numpy as np

d = np.load(sys.argv[1])
rec = d["bwd"]
rec = rec[rec[:, 5] > 0]
q = (rec[:, 0] >> 32).astype(np.int64)
typ = ((rec[:, 0] >> 16) & 0xFFFF).astype(np.int64)
ch = (rec[:, 0] & 0xFFFF).astype(np.int64)
sm = rec[:, 1].astype(np.int64)
t0 = rec[:, 2].min()
f = lambda i: (rec[:, i].astype(np.float64) - float(t0)) / 1e3
deq, rdy, ep0, ep1, l0, l1, m0, m1 = [f(i) for i in (2, 3, 4, 5, 8, 9, 10, 11)]
span = ep1.max()
dep_total = 0.0
gap_total = 0.0
for s in np.unique(sm):
    idx = np.nonzero(sm == s)[0]
    idx = idx[np.argsort(q[idx])]
    prev_l1 = 0.0
    for i in idx:
        start = max(prev_l1, deq[i])        # producer could have started this item
        dep_total += max(0.0, rdy[i] - start)
        gap_total += max(0.0, deq[i] - prev_l1)
        prev_l1 = l1[i]
ncl = len(np.unique(sm))
print(f"span {span:.0f} us, clusters {ncl}: producer dependency wait {dep_total / ncl:.0f} us/cluster, "
      f"queue gaps {gap_total / ncl:.0f} us/cluster")
names = {1: "G", 2: "DW", 3: "DH"}
print("chunk |  G first-load .. last-epi-end |  W first-load .. last-epi-end")
for c in range(ch.max() + 1):
    g = (ch == c) & (typ == 1)
    w = (ch == c) & (typ != 1)
    print(f"{c:5d} | {l0[g].min():8.1f} .. {ep1[g].max():8.1f} | {l0[w].min():8.1f} .. {ep1[w].max():8.1f}")
