"""Data-parallel training across the GPUs of one node (batch sharding).

One process per GPU (torchrun), NCCL over NVLink/NVSwitch for the single
exchange step of the path: the sum all-reduce of the flat fp32 parameter
gradient buffer, issued in reverse-layer buckets from inside
backward on a communication stream as each bucket's gradients become final,
and captured with the rest of the step in one CUDA graph.  BN
statistics stay per-GPU as in the paper/reference unless ``sync_bn`` is set
(engine option): then the 2*C float64 (sum, sum^2) of every BN and the 2*C
(dbeta, dgamma) sums are all-reduced before they are finalised.

Gradient averaging is folded into the learning rate (lr / world) so the
all-reduce is a plain SUM on the engine's own buffer with no extra kernel.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def init(backend: str = "nccl"):
    """Initialise the default process group from torchrun's env (no-op for world 1)."""
    rank, local, world = env_rank()
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, local, world


def shard_batch(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) rows of a global batch owned by ``rank`` (equal shards; weak scaling
    keeps the per-GPU batch fixed and grows the global batch with the world)."""
    if global_batch % world:
        raise ValueError(f"global batch {global_batch} not divisible by world {world}")
    per = global_batch // world
    return rank * per, (rank + 1) * per


def allreduce_grads(flat: torch.Tensor, group=None):
    """SUM all-reduce of the flat gradient buffer (in place)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat


class DPTrainer:
    """Drive an ``Engine`` data-parallel.  With bucketed all-reduces (the default for
    world > 1, ``Engine(dp_buckets=True)``) the whole step -- forward, backward with the
    gradient SUM all-reduces issued bucket by bucket on the communication stream, SGD --
    is ONE captured CUDA graph; otherwise (dp_buckets=False) a fwd+bwd graph, one flat
    all-reduce, and the SGD graph.  With world == 1 this is exactly ``Engine.step``."""

    def __init__(self, engine, group=None):
        self.eng = engine
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.parts = None
        self.fused = self.world == 1 or getattr(engine, "dp_buckets", False)

    def capture(self):
        if self.fused:
            self.eng.capture()
        else:
            self.parts = self.eng.capture(split=True)

    def step(self):
        if self.fused:
            self.eng.step()
            return
        if self.parts is None:
            self.eng.forward()
            self.eng.backward()
            allreduce_grads(self.eng.gflat, self.group)
            self.eng.optimizer_step()
            return
        g1, g2 = self.parts
        g1.replay()
        allreduce_grads(self.eng.gflat, self.group)
        g2.replay()
