"""Host-side logic of bench.py (no GPU): the multi-GPU launch contract and the volume check."""
import json
import os
import subprocess
import sys
import types

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _args(**kw):
    base = dict(gpus=None, impl="ours")
    base.update(kw)
    return types.SimpleNamespace(**base)


def test_world_size_from_torchrun_env(monkeypatch):
    import bench
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert bench.world_size(_args()) == 4
    assert bench.world_size(_args(gpus=4)) == 4


def test_world_size_mismatch_exits_nonzero(monkeypatch):
    import bench
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit) as ei:
        bench.world_size(_args(gpus=8))
    assert ei.value.code == 2


def test_world_size_single_and_reference(monkeypatch):
    import bench
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    assert bench.world_size(_args()) == 1
    assert bench.world_size(_args(gpus=1)) == 1
    # the reference arm never spawns: rank 0 alone runs the oracle
    assert bench.world_size(_args(gpus=8, impl="reference")) == 8


def test_gpus_n_without_torchrun_spawns_n_ranks(monkeypatch):
    """`--gpus N` without torchrun re-launches bench.py through torch.distributed.run with N
    ranks on 127.0.0.1 and exits with their status (the command is captured, not run)."""
    import bench
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    seen = {}

    def fake_call(cmd):
        seen["cmd"] = cmd
        return 0
    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "8", "--steps", "3"])
    with pytest.raises(SystemExit) as ei:
        bench.world_size(_args(gpus=8))
    assert ei.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == [os.path.join(ROOT, "bench.py"), "--gpus", "8", "--steps", "3"][-4:]


def test_nccl_info_summary(tmp_path):
    import bench
    (tmp_path / "x.a.1.log").write_text("host:1:1 [0] NCCL INFO comm 0x1 rank 0 nRanks 8 nNodes 1 localRanks 8\n"
                                        "host:1:1 [0] NCCL INFO NVLS multicast support is available\n")
    s = bench.nccl_info_summary(str(tmp_path / "x.*.log"), 8)
    assert s["nranks_seen"] == [8] and s["comm_nranks_ok"] and s["nvls_mentioned"]
    assert not bench.nccl_info_summary(str(tmp_path / "x.*.log"), 4)["comm_nranks_ok"]


def test_reference_arm_line_fields():
    """The reference arm prints one JSON line with the measured per-sample step time."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "mlp1m",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["n_gpus"] == 1 and line["unit"] == "Gparams/s"
    assert line["ms_per_step"] > 0 and line["ms_per_step_kind"].startswith("measured")
    assert line["cpu_baseline"]["kind"] == "oracle" and line["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_arm_under_torchrun_prints_once():
    """Under torchrun with N ranks the reference arm runs on rank 0 alone: exactly one JSON
    line, n_gpus = N, and every rank exits 0."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--impl", "reference", "--config", "mlp1m", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
