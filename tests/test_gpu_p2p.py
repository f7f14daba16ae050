"""The vocabulary-sharded exchange over peer memory (CCE_FLAG_P2P_COMBINE, SURVEY 8(f)
NEXT #4): 2 or 3 PROCESSES, one rank per GPU, their workspaces mapped into each other with
CUDA IPC.  The stats are pushed by the merge kernel and the dH tiles are reduced and broadcast
by the backward kernel's RED items across the processes; every rank must match the unsharded
oracle and the others bit for bit, over two consecutive steps (the per-step flag epochs).
Skipped with fewer GPUs than ranks (see _need_gpus); on one GPU the same kernels run as
co-resident rank groups of ONE launch (tests/test_gpu_p2p_emulated.py)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle
import workload
from cce_testutil import TOL_GRAD, TOL_LOSS, TOL_LSE, rel_fro

pytestmark = pytest.mark.gpu


def _need_gpus(world):
    """Ranks whose kernels wait on one another must run on their own GPUs: several such
    processes time-sliced on ONE GPU can raise Xid 109 (context-switch timeout) on this
    driver (B200_PROFILING.md), so with fewer GPUs than ranks these tests are skipped; the
    exchange's arithmetic is covered on one GPU by test_gpu_sharded.py (split-phase) and the
    host logic by tests/test_multiproc.py (gloo)."""
    import torch
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (one process per GPU); {torch.cuda.device_count()} visible")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["CCE_ROOT"]); sys.path.insert(0, os.path.join(os.environ["CCE_ROOT"], "tests"))
import numpy as np, torch, torch.distributed as dist
import paper_2601_02609_b200 as cce, workload
from cce_testutil import to_dev
rank, world, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
absent = int(os.environ.get("CCE_ABSENT", "-1"))   # a rank that attaches but never steps
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + os.environ["CCE_PORT"], rank=rank, world_size=world)
dev = torch.device("cuda", rank)
torch.cuda.set_device(dev)
p = workload.make_problem(700, 128, 3000, seed=606, ignore="bern40")
H, W, y = to_dev(p, dev)
N, D = H.shape
V = W.shape[0]
lo, hi = cce.shard_range(V, rank, world)
Wr = W[lo:hi].contiguous()
mode = os.environ.get("CCE_MODE", "plain")   # plain | ls (label smoothing + z-loss) | rms (RMSNorm prologue)
h = cce.CCEHandle(vocab_total=V, vocab_offset=lo, rank=rank, world=world, flags=cce.FLAG_P2P_COMBINE,
                  label_smoothing=0.1 if mode == "ls" else 0.0, z_loss=1e-4 if mode == "ls" else 0.0)
if mode == "rms":
    Xb, gb = workload.make_rmsnorm_inputs(606, N, D)
    Xt = torch.from_numpy(Xb.view(np.int16)).view(torch.bfloat16).to(dev)
    gt = torch.from_numpy(gb.view(np.int16)).view(torch.bfloat16).to(dev)
ws = h.workspace(N, D, hi - lo, dev)
mine = cce.cce_p2p_export(ws)
allh = [None] * world
dist.all_gather_object(allh, mine)
cce.cce_p2p_attach(h.h, ws, N, D, [a[0] for a in allh], [a[1] for a in allh])
dist.barrier()
one = torch.ones((), dtype=torch.float32, device=dev)
if mode == "fwdonly":
    # forward-only loop (evaluation): consecutive forwards with different labels and no
    # backward in between -- the stats exchange must not let step e+1 overwrite what a peer
    # still reads for step e (double-buffered by step parity)
    losses = []
    for step in range(4):
        loss, lse, nv = h.forward(H, Wr, torch.roll(y, step))
        losses.append(loss)
    torch.cuda.synchronize()
    np.savez(out, losses=np.array([l.item() for l in losses]), err=cce.cce_get_error(h.h))
    dist.barrier()
    h.close()
    dist.destroy_process_group()
    sys.exit(0)
for step in range(0 if rank == absent else 2):
    dH = torch.empty_like(H)
    dW = torch.empty_like(Wr)
    if mode == "rms":
        loss, lse, nv = h.forward_rmsnorm(Xt, gt, 1e-6, Wr, y)
        dg = torch.empty_like(gt)
        h.backward_rmsnorm(one, dH, dg, dW)
    else:
        loss, lse, nv = h.forward(H, Wr, y)
        h.backward(one, dH, dW)
    torch.cuda.synchronize()
err = cce.cce_get_error(h.h)
if rank == absent:
    np.savez(out, err=0)
    dist.barrier()
    sys.exit(0)
np.savez(out, loss=loss.item(), lse=lse.cpu().numpy(), dH=dH.view(torch.int16).cpu().numpy(),
         dW=dW.view(torch.int16).cpu().numpy(), err=err, lo=lo, hi=hi, nv=int(nv.item()))
dist.barrier()   # peers read this workspace until here
h.close()
dist.destroy_process_group()
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(tmp_path, world, absent=-1, mode="plain"):
    _need_gpus(world)
    import __graft_entry__
    __graft_entry__.build()
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, CCE_ROOT=ROOT, CCE_PORT=str(_free_port()), CCE_ABSENT=str(absent), CCE_MODE=mode)
    procs = [subprocess.Popen([sys.executable, str(script), str(r), str(world), str(tmp_path / f"r{r}.npz")], env=env,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT) for r in range(world)]
    logs = []
    for pr in procs:
        try:
            logs.append(pr.communicate(timeout=240)[0].decode(errors="replace"))
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("P2P worker timed out")
    assert all(pr.returncode == 0 for pr in procs), "\n".join(logs)[-3000:]
    return [np.load(tmp_path / f"r{r}.npz") for r in range(world)]


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_exchange_between_processes(tmp_path, world):
    res = _run(tmp_path, world)
    p = workload.make_problem(700, 128, 3000, seed=606, ignore="bern40")
    ref = oracle.cce(p["H"], p["W"], p["labels"])
    valid = p["labels"] != -100
    for r in res:
        assert int(r["err"]) == 0
        assert float(r["loss"]) == float(res[0]["loss"])
        assert np.array_equal(r["lse"].view(np.int32), res[0]["lse"].view(np.int32))
        assert np.array_equal(r["dH"], res[0]["dH"])
    o = res[0]
    assert abs(float(o["loss"]) - ref["loss"]) <= TOL_LOSS
    rel = np.abs(o["lse"][valid] - ref["lse"][valid]) / np.maximum(np.abs(ref["lse"][valid]), 1.0)
    assert rel.max() <= TOL_LSE
    f = lambda b: (b.astype(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)  # noqa: E731
    assert np.all(o["dH"][~valid] == 0)
    assert rel_fro(f(o["dH"]), ref["dH"]) <= TOL_GRAD
    dW = np.concatenate([f(r["dW"]) for r in res])
    assert rel_fro(dW, ref["dW"]) <= TOL_GRAD


def test_p2p_missing_peer_times_out_instead_of_hanging(tmp_path):
    """A rank that attaches but never steps: the other rank's bounded waits expire, the step
    completes with loss = NaN and cce_get_error reports CCE_ERR_NCCL (7); the GPU is not hung."""
    res = _run(tmp_path, 2, absent=1)
    assert int(res[0]["err"]) == 7
    assert np.isnan(float(res[0]["loss"]))


@pytest.mark.parametrize("mode", ["ls", "rms"])
def test_p2p_exchange_with_regularised_loss_and_rmsnorm(tmp_path, mode):
    """The peer-memory exchange carries the label-smoothing logit sums (4th stat) and feeds
    the RMSNorm prologue's backward (dH reduced across ranks before dX / dgamma)."""
    res = _run(tmp_path, 2, mode=mode)
    p = workload.make_problem(700, 128, 3000, seed=606, ignore="bern40")
    if mode == "ls":
        ref = oracle.cce(p["H"], p["W"], p["labels"], label_smoothing=0.1, z_loss=1e-4)
        dref = ref["dH"]
    else:
        X, g = workload.make_rmsnorm_inputs(606, 700, 128)
        ref = oracle.cce_rmsnorm(X, g, p["W"], p["labels"], eps=1e-6)
        dref = ref["dX"]
    f = lambda b: (b.astype(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)  # noqa: E731
    for r in res:
        assert int(r["err"]) == 0
        assert np.array_equal(r["dH"], res[0]["dH"])
    assert abs(float(res[0]["loss"]) - ref["loss"]) <= TOL_LOSS
    assert rel_fro(f(res[0]["dH"]), dref) <= TOL_GRAD
    assert rel_fro(np.concatenate([f(r["dW"]) for r in res]), ref["dW"]) <= TOL_GRAD


def test_p2p_forward_only_loop(tmp_path):
    """back-to-back forwards without a backward (evaluation loops) over peer memory."""
    p = workload.make_problem(700, 128, 3000, seed=606, ignore="bern40")
    res = _run(tmp_path, 2, mode="fwdonly")
    for step in range(4):
        ref = oracle.cce(p["H"], p["W"], np.roll(p["labels"], step))
        for r in res:
            assert int(r["err"]) == 0
            assert abs(float(r["losses"][step]) - ref["loss"]) <= TOL_LOSS, (step, float(r["losses"][step]), ref["loss"])
