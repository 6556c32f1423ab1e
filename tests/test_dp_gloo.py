"""Data-parallel path on CPU: two processes over gloo (world size 2).

Pins the semantics of ``paper_1807_01702_b200.dp``: batch sharding,
per-replica BN statistics (the reference's single-device semantics applied per
shard), one SUM all-reduce of the flat gradient buffer, and SGD with the averaging
folded into the learning rate.  Each rank computes its shard's gradients with the
CPU oracle; the all-reduced result must equal the sum of both shards' oracle
gradients computed independently, and the post-step weights must match
w - lr * mean_over_ranks(grad).
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _graph():
    from paper_1807_01702_b200 import fusion, graph as G
    spec = G.densenet_micro(batch=4)
    g, _ = fusion.plan(G.build_model(spec, seed=0), fusion.FusionLevel.BNFF)
    return g


def _shard_grads(g, x_shard, dy_shard):
    """Oracle gradients of one shard, flattened in engine parameter order."""
    from oracle import executor as OX
    sub = {g.inputs[0]: x_shard}
    res = OX.forward(g, sub)
    ref = OX.backward(g, res, {g.outputs[0]: dy_shard})
    return np.concatenate([np.asarray(ref.params[k], np.float64).reshape(-1) for k in g.params])


class FakeEngine:
    """Stands in for ``Engine`` on CPU: backward() writes this rank's oracle grads into
    the flat gradient buffer; optimizer_step() applies w -= lr * g (K12 semantics)."""

    def __init__(self, w0, grads, lr):
        self.wflat = torch.tensor(w0, dtype=torch.float64)
        self.gflat = torch.zeros_like(self.wflat)
        self._g = torch.tensor(grads, dtype=torch.float64)
        self.lr = lr
        self.calls = []

    def forward(self):
        self.calls.append("fwd")

    def backward(self):
        self.calls.append("bwd")
        self.gflat.copy_(self._g)

    def optimizer_step(self):
        self.calls.append("opt")
        self.wflat -= self.lr * self.gflat


def _worker(rank, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(WORLD), LOCAL_RANK=str(rank))
    from paper_1807_01702_b200 import dp
    from paper_1807_01702_b200.tensor import Rng
    r, _, w = dp.init("gloo")
    assert (r, w) == (rank, WORLD) and dist.is_initialized()
    g = _graph()
    n, c, h, ww = g.slots[g.inputs[0]].shape
    rng = Rng(1)
    xg = rng.uniform((n * WORLD, c, h, ww), -1.0, 1.0).astype(np.float64)
    dyg = rng.normal((n * WORLD,) + tuple(g.slots[g.outputs[0]].shape[1:])).astype(np.float64)
    lo, hi = dp.shard_batch(n * WORLD, WORLD, rank)
    mine = _shard_grads(g, xg[lo:hi], dyg[lo:hi])
    # reference: both shards' oracle gradients, computed independently on this rank
    expect = sum(_shard_grads(g, xg[k * n:(k + 1) * n], dyg[k * n:(k + 1) * n]) for k in range(WORLD))
    w0 = np.concatenate([np.asarray(g.params[k], np.float64).reshape(-1) for k in g.params])
    lr = 0.1
    eng = FakeEngine(w0, mine, lr / WORLD)  # averaging folded into the learning rate
    tr = dp.DPTrainer(eng)
    assert tr.world == WORLD
    tr.step()
    assert eng.calls == ["fwd", "bwd", "opt"]
    got = eng.gflat.numpy()
    err = np.max(np.abs(got - expect)) / max(np.max(np.abs(expect)), 1e-30)
    assert err < 1e-12, f"rank {rank}: all-reduced grads differ from the shard sum ({err:.2e})"
    w1 = eng.wflat.numpy()
    np.testing.assert_allclose(w1, w0 - lr * expect / WORLD, rtol=0, atol=1e-12)
    # per-replica BN statistics: a rank's own gradient differs from the global-batch one
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.stack([mine, got, w1]))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_batch():
    from paper_1807_01702_b200 import dp
    assert dp.shard_batch(8, 2, 0) == (0, 4) and dp.shard_batch(8, 2, 1) == (4, 8)
    with pytest.raises(ValueError):
        dp.shard_batch(7, 2, 0)


def test_dp_two_ranks_gloo(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(port, str(tmp_path)), nprocs=WORLD, join=True)
    a = np.load(tmp_path / "rank0.npy")
    b = np.load(tmp_path / "rank1.npy")
    # identical all-reduced gradients and post-step weights on both replicas
    np.testing.assert_array_equal(a[1], b[1])
    np.testing.assert_array_equal(a[2], b[2])
    # the shards' own gradients differ (different data, per-replica BN statistics)
    assert np.max(np.abs(a[0] - b[0])) > 0
