#!/usr/bin/env python
"""Experiment: does the workspace's allocation type (torch caching allocator vs cuMemCreate
with compression NONE / GENERIC) change the backward's time under the power cap?  The
dlogits ring lives in the workspace; ncu shows its writes going through the L2's inline
compression (lrc__ilc_input_sectors_compressible) with 0% success.  Prints one JSON line."""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def vmm_alloc(nbytes, comp):
    from cuda.bindings import driver as cu
    cu.cuInit(0)
    prop = cu.CUmemAllocationProp()
    prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = 0
    prop.allocFlags.compressionType = comp
    err, gran = cu.cuMemGetAllocationGranularity(prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED)
    assert err == 0, err
    size = (nbytes + gran - 1) // gran * gran
    err, handle = cu.cuMemCreate(size, prop, 0)
    assert err == 0, err
    err, ptr = cu.cuMemAddressReserve(size, 0, 0, 0)
    assert err == 0, err
    assert cu.cuMemMap(ptr, size, 0, handle, 0)[0] == 0
    desc = cu.CUmemAccessDesc()
    desc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    desc.location.id = 0
    desc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    assert cu.cuMemSetAccess(ptr, size, [desc], 1)[0] == 0

    class Buf:
        __cuda_array_interface__ = {"shape": (size,), "typestr": "|u1", "data": (int(ptr), False), "version": 3}
    return Buf()


def main():
    import numpy as np
    import torch
    from cuda.bindings import driver as cu

    import __graft_entry__
    import paper_2601_02609_b200 as cce
    import workload

    __graft_entry__.build()
    dev = torch.device("cuda:0")
    c = workload.CONFIGS["qwen05b"]
    p = workload.make_config("qwen05b", seed=42)
    t = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).to(dev)  # noqa: E731
    H, W = t(p["H"]), t(p["W"])
    y = torch.from_numpy(p["labels"]).to(dev)
    one = torch.ones((), dtype=torch.float32, device=dev)
    dH, dW = torch.empty_like(H), torch.empty_like(W)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {}
    kinds = {"torch": None, "vmm_none": cu.CUmemAllocationCompType.CU_MEM_ALLOCATION_COMP_NONE,
             "vmm_generic": cu.CUmemAllocationCompType.CU_MEM_ALLOCATION_COMP_GENERIC}
    order = sys.argv[1:] or ["torch", "vmm_none", "vmm_generic", "torch", "vmm_none"]
    for name in order:
        h = cce.CCEHandle(vocab_total=c.V)
        need = cce.cce_workspace_bytes(h.h, c.N, c.D, c.V)
        if kinds[name] is None:
            ws = torch.empty(need, dtype=torch.uint8, device=dev)
        else:
            ws = torch.as_tensor(vmm_alloc(need, kinds[name]), device=dev)[:need]
        h._ws = ws
        loss = torch.empty((), dtype=torch.float32, device=dev)
        for _ in range(5):
            cce.cce_forward(h.h, H, W, y, loss, None, None, ws)
            cce.cce_backward(h.h, one, dH, dW)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        for a, b in ev:
            flush.zero_()
            a.record()
            cce.cce_forward(h.h, H, W, y, loss, None, None, ws)
            cce.cce_backward(h.h, one, dH, dW)
            b.record()
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in ev)
        out.setdefault(name, []).append(round(ms[len(ms) // 2], 4))
        h.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
