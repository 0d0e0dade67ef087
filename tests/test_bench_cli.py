"""bench.py's launcher logic (CPU): --gpus N > 1 outside torchrun re-launches the
script under torch.distributed.run with N ranks on 127.0.0.1; inside torchrun a
--gpus that disagrees with WORLD_SIZE fails loudly instead of reporting
single-GPU numbers as multi-GPU."""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_relaunch_under_torchrun(monkeypatch):
    b = _bench()
    calls = []
    monkeypatch.setattr(b.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "5", "--warmup", "3"])
    assert b.main() == 0
    (cmd,) = calls
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[cmd.index(os.path.abspath(os.path.join(ROOT, "bench.py"))) + 1:] == [
        "--gpus", "4", "--steps", "5", "--warmup", "3"]


def test_world_size_mismatch_fails(monkeypatch, capsys):
    b = _bench()
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4"])
    assert b.main() == 2
    assert "WORLD_SIZE=2" in capsys.readouterr().err


def test_single_gpu_does_not_relaunch(monkeypatch):
    b = _bench()
    monkeypatch.setattr(b.subprocess, "call", lambda cmd: (_ for _ in ()).throw(AssertionError("relaunched")))
    monkeypatch.setenv("WORLD_SIZE", "1")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2"])
    assert b.main() == 2           # mismatch detected, no relaunch inside a torchrun environment


def test_reference_arm_nonzero_rank_exits_clean(monkeypatch):
    b = _bench()
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--gpus", "2"])
    assert b.main() == 0
