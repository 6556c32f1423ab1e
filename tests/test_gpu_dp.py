"""Data-parallel plumbing on the device: the bucketed gradient all-reduce
issued from inside backward on a communication stream and captured in the step's CUDA
graph.  One GPU here, so the NCCL group has one rank: the SUM all-reduce is the
identity and the bucketed engine must match a plain engine bitwise, step after step."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1807_01702_b200 import fusion  # noqa: E402
from paper_1807_01702_b200 import graph as G  # noqa: E402
from paper_1807_01702_b200.tensor import Rng  # noqa: E402


@pytest.fixture(scope="module")
def nccl_world1():
    import torch.distributed as dist
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_bucketed_allreduce_in_graph_matches_plain(nccl_world1, dtype):
    from paper_1807_01702_b200 import dp
    from paper_1807_01702_b200.engine import Engine
    g0 = G.build_model(G.densenet_micro(2, (3, 3), 8), seed=0)
    g, _ = fusion.plan(g0, fusion.parse_level("bnff+icf"))
    rng = Rng(1)
    x = rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0)
    dy = rng.normal(g.slots[g.outputs[0]].shape)
    out = []
    for buckets in (False, True):
        eng = Engine(g, dtype=dtype, lr=0.05, dp_buckets=buckets, bucket_bytes=16 << 10)
        if buckets:
            # reverse-layer buckets: disjoint, contiguous, covering the whole flat gradient
            assert len(eng.buckets) >= 3
            assert eng.buckets[0][1] == eng.gflat.numel() and eng.buckets[-1][0] == 0
            assert all(a[0] == b[1] for a, b in zip(eng.buckets, eng.buckets[1:]))
        tr = dp.DPTrainer(eng)
        eng.set_input(x)
        eng.set_loss_grad(dy)
        tr.capture()
        for _ in range(2):
            tr.step()
        torch.cuda.synchronize()
        out.append((eng.gflat.cpu().numpy(), eng.wflat.cpu().numpy()))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
