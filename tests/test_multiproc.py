"""World-size-2 (gloo, CPU) test of the vocabulary-sharded combine that the CUDA
path performs with NCCL: each rank holds the vocabulary
shard `shard_range(V, rank, 2)`, computes per-row partial (max, sum-exp, target
logit) with the oracle, all-gathers them and merges in rank order; the result must
equal the unsharded oracle on every rank.  The partial dH of each shard
(sum over the shard's vocabulary of G W, with the GLOBAL lse) is all-reduced and
must equal the full dH."""
import math
import os
import socket

import numpy as np
import pytest

import oracle
import workload


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, D, V, seed, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_02609_b200 import shard_range
        p = workload.make_problem(N, D, V, seed=seed, ignore="bern40")
        lo, hi = shard_range(V, rank, world)
        m, d, zy = oracle.partial_stats(p["H"], p["W"][lo:hi], p["labels"], lo)
        local = torch.tensor(np.stack([m, d, zy], 1))
        gathered = [torch.zeros_like(local) for _ in range(world)]
        dist.all_gather(gathered, local)
        # rank-order merge (what k_finalize does after the NCCL allgather)
        valid = p["labels"] != -100
        lse = np.zeros(N)
        zsum = np.zeros(N)
        for n in np.nonzero(valid)[0]:
            M = max(float(g[n, 0]) for g in gathered)
            S = sum(float(g[n, 1]) * math.exp(float(g[n, 0]) - M) for g in gathered if float(g[n, 1]) > 0)
            lse[n] = M + math.log(S)
            zsum[n] = sum(float(g[n, 2]) for g in gathered)
        loss = float(np.mean((lse - zsum)[valid]))
        # partial dH over this shard with the global lse, then all-reduce (a10)
        Hf = oracle._bits(p["H"]); Wf = oracle._bits(p["W"])
        s = 1.0 / valid.sum()
        z = Hf @ Wf[lo:hi].T
        G = s * (np.exp(z - lse[:, None]) * valid[:, None])
        yl = p["labels"] - lo
        own = valid & (yl >= 0) & (yl < hi - lo)
        G[np.nonzero(own)[0], yl[own]] -= s
        dH = torch.tensor(G @ Wf[lo:hi])
        dist.all_reduce(dH)
        q.put((rank, loss, lse[valid].tolist(), dH.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("V", [1000, 997])
def test_two_rank_vocab_sharded_combine(V):
    import torch.multiprocessing as mp
    N, D, seed = 40, 16, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, N, D, V, seed, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = workload.make_problem(N, D, V, seed=seed, ignore="bern40")
    ref = oracle.cce(p["H"], p["W"], p["labels"])
    valid = p["labels"] != -100
    for rank, loss, lse, dH in res:
        assert abs(loss - ref["loss"]) <= 1e-12
        np.testing.assert_allclose(lse, ref["lse"][valid], rtol=1e-13)
        np.testing.assert_allclose(dH, ref["dH"], rtol=1e-10, atol=1e-14)
    assert res[0][1] == res[1][1]                       # identical on every rank


def test_shard_range_partition():
    from paper_2601_02609_b200 import shard_range
    for V in (151936, 1000, 7):
        for world in (1, 2, 3, 8, 16):
            spans = [shard_range(V, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == V
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
