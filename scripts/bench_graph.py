"""One forward + backward step captured in a CUDA graph vs launched eagerly (same process,
interleaved, L2 flushed between steps): the library is stream-ordered with no host syncs,
so the whole step is capturable; the graph removes the host launch gaps between its ~7
kernels.  Prints one JSON line."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import __graft_entry__
    import paper_2601_02609_b200 as cce
    import workload
    __graft_entry__.build()
    dev = torch.device("cuda:0")
    cfg = sys.argv[1] if len(sys.argv) > 1 else "qwen05b"
    c = workload.CONFIGS[cfg]
    p = workload.make_config(cfg, seed=42)
    H = torch.from_numpy(p["H"].view(np.int16)).view(torch.bfloat16).to(dev)
    W = torch.from_numpy(p["W"].view(np.int16)).view(torch.bfloat16).to(dev)
    y = torch.from_numpy(p["labels"]).to(dev)
    h = cce.CCEHandle(vocab_total=c.V)
    ws = h.workspace(c.N, c.D, c.V, dev)
    loss = torch.empty((), dtype=torch.float32, device=dev)
    lse = torch.empty(c.N, dtype=torch.float32, device=dev)
    nv = torch.empty((), dtype=torch.int32, device=dev)
    dH = torch.empty_like(H)
    dW = torch.empty_like(W)
    one = torch.ones((), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(device=dev)

    def step():
        cce.cce_forward(h.h, H, W, y, loss, lse, nv, ws, s)
        cce.cce_backward(h.h, one, dH, dW, s)

    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.synchronize()
    ref = (loss.item(), dW.view(torch.int16).clone())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    assert loss.item() == ref[0] and torch.equal(dW.view(torch.int16), ref[1]), "graph replay differs"
    res = {"eager": [], "graph": []}
    for rnd in range(8):
        for mode in (("eager", "graph") if rnd % 2 == 0 else ("graph", "eager")):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
            with torch.cuda.stream(s):
                for a, b in ev:
                    flush.zero_()
                    a.record(s)
                    if mode == "eager":
                        step()
                    else:
                        g.replay()
                    b.record(s)
            torch.cuda.synchronize()
            res[mode] += [a.elapsed_time(b) for a, b in ev]
    out = {"config": cfg, "eager_ms_median": statistics.median(res["eager"]),
           "graph_ms_median": statistics.median(res["graph"]), "steps_each": len(res["eager"]),
           "bit_identical": True}
    print(json.dumps(out))
    h.close()


if __name__ == "__main__":
    main()
