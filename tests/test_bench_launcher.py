"""bench.py --gpus N without torchrun re-launches itself under torch.distributed.run with
one process per GPU (the driver's N=1,2,4,8 runs work either way)."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_n_spawns_one_rank_per_gpu(monkeypatch):
    sys.path.insert(0, ROOT)
    import bench
    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3", "--warmup", "3"])
    try:
        bench.main()
    except SystemExit as e:
        assert e.code == 0
    assert len(calls) == 1
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-6:] == ["--gpus", "4", "--steps", "3", "--warmup", "3"]


def test_reference_arm_does_not_spawn(monkeypatch):
    sys.path.insert(0, ROOT)
    import bench
    ran = []
    monkeypatch.setattr(bench, "run_reference", lambda args: ran.append(args.gpus))
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: (_ for _ in ()).throw(AssertionError("spawned")))
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--gpus", "8"])
    bench.main()
    assert ran == [8]
