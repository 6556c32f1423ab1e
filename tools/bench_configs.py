"""Device-timed training step of every BASELINE.json config other than the headline
(C3 DenseNet-121 is bench.py): C1 the CONV3x3-BN-ReLU-CONV1x1 block (N=8, C=64, 32x32),
C2 DenseNet-BC-100 k=12 CIFAR 32x32 b64, C4 ResNet-50 224x224 b128 -- each at its fused
level and at the unfused baseline, plus the numpy oracle's rate on a bounded sample.
One JSON line per config.  (C5, the BN-layer sweep, is tools/c5_sweep.py.)

    python tools/bench_configs.py [--steps 10] [--warmup 3] [--only c1,c2,c4] [--dtype bf16]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def spec_of(name):
    from paper_1807_01702_b200 import graph as G
    if name == "c1":
        return None, 8
    if name == "c2":
        return G.densenet_bc100(64), 64
    if name == "c4":
        return G.resnet50(128), 128
    raise ValueError(name)


def build(name, level, dtype):
    from paper_1807_01702_b200 import fusion, graph as G
    spec, batch = spec_of(name)
    g0 = G.build_block(8, 64, 32, seed=0) if spec is None else G.build_model(spec, seed=0)
    if name == "c2":  # k = 12 pieces: widened to 16-byte channel multiples (graph.pad_channels)
        g0, _ = G.pad_channels(g0, 8)
    g, _ = fusion.plan(g0, fusion.parse_level(level))
    return g, batch


def device_ms(g, dtype, steps, warmup):
    import torch
    from paper_1807_01702_b200.engine import Engine
    from paper_1807_01702_b200.tensor import Rng
    eng = Engine(g, dtype=dtype, input_grad=False, lr=1e-3)
    rng = Rng(1)
    eng.set_input(rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0))
    eng.set_loss_grad(rng.normal(g.slots[g.outputs[0]].shape))
    eng.capture()
    for _ in range(warmup):
        eng.step()
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for _ in range(steps):
        eng.step()
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    nbytes = sum(t.nbytes for t in eng.all_thunks())
    flops = sum(t.flops for t in eng.all_thunks())
    launches = sum(getattr(t, "launches", 1) for t in eng.all_thunks())
    del eng
    torch.cuda.empty_cache()
    return ms, nbytes, flops, launches


def cpu_rate(name, level, sample_batch):
    """numpy oracle (restating bnfuse) on a bounded sample of the same model: images/s."""
    import numpy as np
    from oracle import executor as OX
    from paper_1807_01702_b200 import fusion, graph as G
    from paper_1807_01702_b200.tensor import Rng
    spec, _ = spec_of(name)
    g0 = G.build_block(sample_batch, 64, 32, seed=0) if spec is None else \
        G.build_model(spec.with_batch(sample_batch), seed=0)
    g, _ = fusion.plan(g0, fusion.parse_level(level))
    rng = Rng(1)
    x = rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0)
    dy = rng.normal(g.slots[g.outputs[0]].shape)
    t = []
    for _ in range(2):
        t0 = time.perf_counter()
        res = OX.forward(g, {g.inputs[0]: x})
        OX.backward(g, res, {g.outputs[0]: dy})
        t.append(time.perf_counter() - t0)
    return sample_batch / float(np.min(t))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default="c1,c2,c4")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    hbm = 6554.6
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        pass
    for name in a.only.split(","):
        fused_level = {"c1": "bnff", "c2": "bnff+icf", "c4": "bnff"}[name]
        from paper_1807_01702_b200.errors import UnsupportedError
        dtype, note = a.dtype, ""
        g, batch = build(name, fused_level, dtype)
        try:
            ms, nb, fl, nl = device_ms(g, dtype, a.steps, a.warmup)
        except UnsupportedError as e:  # e.g. k=12 pieces at 16-byte-unaligned channel offsets
            dtype, note = "f32", f"bf16 unsupported ({e}); fp32 (3xTF32) path"
            ms, nb, fl, nl = device_ms(g, dtype, a.steps, a.warmup)
        gu, _ = build(name, "baseline", dtype)
        ums, unb, _, _ = device_ms(gu, dtype, a.steps, a.warmup)
        if name == "c2":
            note = "growth-rate-12 pieces padded to 16 channels (graph.pad_channels; exact zeros)"
        line = {"config": name, "level": fused_level, "dtype": dtype, "note": note, "batch": batch,
                "ms_per_step": round(ms, 4), "images_per_s": round(batch / (ms * 1e-3), 1),
                "unfused_ms_per_step": round(ums, 4), "speedup_vs_unfused": round(ums / ms, 3),
                "algorithmic_bytes_per_step": nb, "unfused_algorithmic_bytes_per_step": unb,
                "bn_bytes_reduction": round(1 - nb / unb, 4), "flops_per_step": fl,
                "achieved_gbs_step_avg": round(nb / (ms * 1e-3) / 1e9, 1), "hbm_peak_gbs": hbm,
                "gpu_launches_per_step": nl}
        if not a.no_cpu:
            sb = {"c1": 8, "c2": 4, "c4": 1}[name]
            line["cpu_oracle_images_per_s"] = round(cpu_rate(name, fused_level, sb), 3)
            line["cpu_sample"] = f"batch {sb} fwd+bwd, best of 2 (numpy oracle, {len(os.sched_getaffinity(0))} threads)"
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
