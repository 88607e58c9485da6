"""bench.py's host-side contract on CPU: `--gpus N` without a launcher re-runs
itself under torch.distributed.run with N ranks on 127.0.0.1 (the driver's SCALE
run uses the same command form as the N=1 BENCH run)."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT


def test_self_launch_builds_torchrun_command(monkeypatch, capsys):
    sys.path.insert(0, ROOT)
    import bench
    seen = {}

    def fake_run(cmd, env=None, **kw):
        seen["cmd"], seen["env"] = cmd, env
        out = "NCCL INFO comm 0x1 rank 0 nranks 4\n{\"metric\": \"m\"}\nNCCL INFO Destroy COMPLETE\n"
        return subprocess.CompletedProcess(cmd, 0, stdout=out, stderr="")

    monkeypatch.setattr(subprocess, "run", fake_run)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "5"])
    args = bench.main.__globals__["argparse"].Namespace(gpus=4, impl="b200")
    with pytest.raises(SystemExit) as e:
        bench.self_launch(args)
    assert e.value.code == 0
    # the JSON line is relayed last, after NCCL's init / teardown lines
    out = capsys.readouterr().out.splitlines()
    assert out[-1] == '{"metric": "m"}' and out[0].startswith("NCCL INFO")
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "5"]
    assert seen["env"]["NCCL_DEBUG"] in ("INFO", os.environ.get("NCCL_DEBUG", "INFO"))


def test_no_self_launch_for_one_gpu_or_under_torchrun(monkeypatch):
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    assert bench.self_launch(argparse.Namespace(gpus=1, impl="b200")) is False
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert bench.self_launch(argparse.Namespace(gpus=4, impl="b200")) is False
    monkeypatch.delenv("WORLD_SIZE")
    assert bench.self_launch(argparse.Namespace(gpus=4, impl="reference")) is False
