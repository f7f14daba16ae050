"""bench.py's JSON-line contract, checked on CPU through the reference arm (the oracle on the
host cores, the one leg that runs without a GPU): one line, the required keys, the reference
arm's extra fields.  The GPU arm's line is produced on the B200 (profiles/r01_bench.json)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "tiny",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 1 and d["warmup"] == 3
    assert d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1


def test_committed_gpu_bench_line_has_the_contract_keys():
    """The committed B200 line (profiles/r01_bench.json): roofline, cpu_baseline, e2e, clocks,
    launch count and memory report present and consistent."""
    path = os.path.join(ROOT, "profiles", "r01_bench.json")
    d = json.loads(open(path).read().strip().splitlines()[-1])
    for k in ("roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches", "memory"):
        assert k in d, k
    r = d["roofline"]
    assert r["bound"] == "tensor" and 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["gpu_launches"] > 0 and d["memory"]["no_NxV_buffer"] is True
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0


def test_self_launch_builds_a_torchrun_command(monkeypatch):
    """`bench.py --gpus N` without WORLD_SIZE re-launches itself through torch.distributed.run,
    one process per GPU, rendezvous on 127.0.0.1, passing its own arguments through."""
    sys.path.insert(0, ROOT)
    import bench
    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "7"])
    assert bench._self_launch(4) == 0 or "cmd" in seen
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "7"]


def test_committed_r02_lines_carry_in_bench_parity():
    """Round-2 bench lines carry the in-bench oracle-golden check."""
    for f in ("r02_bench_default_same_box.json", "r02_bench_designb.json", "r02_bench_long_200steps.json"):
        d = json.loads(open(os.path.join(ROOT, "profiles", f)).read().strip().splitlines()[-1])
        assert d["parity"]["ok"] is True and d["parity"]["rows_checked"] == 4915, f
        assert d["parity"]["lse_max_rel_err"] <= 1e-3 and d["parity"]["loss_abs_err"] <= 2e-3


def test_clock_sampler_keeps_the_timed_region_samples():
    """The clock record covers the timed region: samples are stamped as they arrive and the
    statistics use the ones inside (t0, t1 + one period); throttle reasons are collected."""
    sys.path.insert(0, ROOT)
    import bench
    s = bench.ClockSampler(0, period_ms=10)
    s.proc = object()  # (no nvidia-smi on the CPU box: feed rows directly)
    s.t = type("T", (), {"join": lambda self, timeout=None: None})()
    s.proc = type("P", (), {"terminate": lambda self: None, "wait": lambda self, timeout=None: 0})()
    row = lambda mhz, w, cap: ["0", str(mhz), "1965", str(w), "0x0", "Not Active", "Not Active", "Not Active", cap]  # noqa: E731
    s.stamped = [(0.5, row(1965, 100.0, "Not Active")),      # idle lead-in, outside the window
                 (1.00, row(1400, 900.0, "Active")), (1.01, row(1380, 950.0, "Active")),
                 (1.02, row(1390, 920.0, "Not Active")),
                 (3.0, row(1965, 80.0, "Not Active"))]       # after the window
    c = s.stop(window=(0.99, 1.02))
    assert c["samples_in_timed_region"] == 3 and c["samples"] == 3
    assert c["sm_mhz"] == 1390 and c["reasons"] == ["sw_power_cap"] and c["power_w_max"] == 950.0
    s.stamped = [(0.5, row(1965, 100.0, "Not Active"))]       # nothing inside: fall back to every sample
    c = s.stop(window=(0.99, 1.02))
    assert c["samples"] == 1 and c["samples_in_timed_region"] == 0
