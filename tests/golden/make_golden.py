"""Generate parity fixtures from the REAL reference (run in the build container).

    python tests/golden/make_golden.py            # needs /root/reference (read-only)

Imports ``bnfuse`` from /root/reference/pkg/src and writes, under tests/golden/:

* ``graphs.json``   -- node/slot tables, rewrite counts and parameter digests of
                       every preset (plus the BASELINE configs) at every fusion
                       level: pins our builders + rewriter to the reference's.
* ``model_<case>_<level>_<dtype>.npz`` -- one forward+backward of small models
                       through ``bnfuse.execute`` (x ~ U(-1,1), dy ~ N(0,1) from
                       Rng(seed+1), as verify.py:50-52): outputs, parameter
                       gradients, input gradients.
* ``block_c1_<level>.npz`` -- BASELINE config C1 (8x64x32x32 conv3x3-BN-ReLU-conv1x1)
                       digests: per-channel sums of output and input gradient, a
                       fixed sample of elements, and full parameter gradients.

Nothing at GPU-test time reads /root/reference; only these fixtures travel.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from bnfuse import execute, fusion  # noqa: E402
from bnfuse import graph as RG  # noqa: E402
from bnfuse.tensor import Rng  # noqa: E402

LEVELS = ["baseline", "rcf", "rcf+mvf", "bnff", "bnff+icf"]


def extra_specs():
    return {
        # BASELINE config C2 through the reference builder
        "densenet-bc-100": RG.ModelSpec(family="densenet", blocks=(16, 16, 16), growth_rate=12,
                                        bottleneck_mult=4, input_dims=(64, 24, 32, 32),
                                        scale="micro", stem="conv3", name="densenet-bc-100"),
        # tiny full-scale DenseNet: 7x7/s2 stem, stem BN+ReLU+pool, transition, head
        "densenet-tiny-full": RG.ModelSpec(family="densenet", blocks=(2, 2), growth_rate=8,
                                           bottleneck_mult=4, input_dims=(2, 3, 32, 32),
                                           scale="full", stem="conv7-pool", base_channels=16,
                                           name="densenet-tiny-full"),
        # tiny ResNet with a stride-2 stage: pooled + zero-padded shortcut
        "resnet-tiny-strided": RG.ModelSpec(family="resnet", blocks=(1, 1),
                                            input_dims=(2, 8, 8, 8), scale="micro", stem="conv3",
                                            base_channels=16,
                                            resnet_stages=((1, 4, 16, 1), (1, 8, 32, 2)),
                                            name="resnet-tiny-strided"),
    }


def attrs_summary(node):
    a = node.attrs
    out = {}
    for key in ("clip_input", "onepass", "emit_stats", "defer_backward", "physical", "k",
                "pad_channels", "fanout"):
        if a is not None and hasattr(a, key):
            out[key] = getattr(a, key)
    if a is not None and hasattr(a, "conv"):
        c = a.conv
        out["conv"] = [c.name, c.in_c, c.out_c, c.kh, c.stride, c.pad]
    if a is not None and hasattr(a, "bn"):
        out["bn"] = a.bn.name
    return out


def graph_record(g, fp=None):
    rec = {
        "nodes": [[n.id, n.kind, n.name, list(n.inputs), list(n.outputs),
                   list(n.saved_for_backward), attrs_summary(n)] for n in g.nodes],
        "slots": [[s.id, list(s.shape), s.kind, s.name, list(s.buffer) if s.buffer else None]
                  for s in sorted(g.slots.values(), key=lambda s: s.id)],
        "inputs": list(g.inputs), "outputs": list(g.outputs),
        "buffer_groups": {k: list(v) for k, v in g.buffer_groups.items()},
    }
    if fp is not None:
        kinds = sorted({r.kind for r in fp.rewrites})
        rec["rewrite_counts"] = {k: fp.count(k) for k in kinds}
        rec["unfused_bn_ids"] = list(fp.unfused_bn_ids)
        rec["bn_map"] = {str(k): list(v) for k, v in fp.bn_map.items()}
    return rec


def param_digests(g):
    return {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()[:16]
            for k, v in g.params.items()}


def make_graphs():
    specs = {name: fn() for name, fn in RG.PRESETS.items()}
    specs["densenet-121"] = RG.densenet121(2)
    specs["resnet-50"] = RG.resnet50(2)
    specs.update(extra_specs())
    out = {}
    for name, spec in specs.items():
        g = RG.build_model(spec, seed=0)
        entry = {"spec": {"family": spec.family, "blocks": list(spec.blocks),
                          "growth_rate": spec.growth_rate,
                          "bottleneck_mult": spec.bottleneck_mult,
                          "input_dims": list(spec.input_dims), "scale": spec.scale,
                          "stem": spec.stem, "base_channels": spec.base_channels,
                          "resnet_stages": [list(s) for s in spec.resnet_stages],
                          "name": spec.name},
                 "params": param_digests(g), "levels": {}}
        for lv in LEVELS:
            g2, fp = fusion.plan(g, fusion.parse_level(lv))
            entry["levels"][lv] = graph_record(g2, fp)
        out[name] = entry
    with open(os.path.join(HERE, "graphs.json"), "w") as f:
        json.dump(out, f, sort_keys=True)
    print("graphs.json:", len(out), "models")


def run_model(g, seed):
    rng = Rng(seed + 1)
    dtype = next(iter(g.params.values())).dtype
    x = rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0, dtype=dtype)
    dy = {s: rng.normal(g.slots[s].shape, dtype=dtype) for s in g.outputs}
    acts = execute.forward(g, {g.inputs[0]: x}, ctx=execute.ExecCtx(budget=64 << 20))
    grads = execute.backward(g, acts, dy, ctx=execute.ExecCtx(budget=64 << 20))
    return x, dy, acts, grads


def save_model_case(name, spec, levels, dtypes, seed=0):
    for dt in dtypes:
        g0 = RG.build_model(spec, seed=seed, dtype=dt)
        for lv in levels:
            g, _ = fusion.plan(g0, fusion.parse_level(lv))
            x, dy, acts, grads = run_model(g, seed)
            payload = {"x": x}
            for s in g.outputs:
                payload[f"out_{s}"] = np.asarray(acts.vals[s])
                payload[f"dy_{s}"] = dy[s]
            for k, v in grads.params.items():
                payload[f"grad::{k}"] = np.asarray(v)
            for s, v in grads.inputs.items():
                payload[f"dx_{s}"] = np.asarray(v)
            tag = "f32" if dt == np.float32 else "f64"
            fn = os.path.join(HERE, f"model_{name}_{lv.replace('+', '_')}_{tag}.npz")
            np.savez_compressed(fn, **payload)
    print("model", name, "done")


def make_block_c1():
    # C1: conv3x3(64->64) -> BN -> ReLU -> conv1x1(64->64), N=8, 32x32, seed 0
    from bnfuse.graph import _bn_relu_conv, _ParamFactory, ConvAttrs, Graph, CONV
    g = Graph(meta={"family": "block"})
    pf = _ParamFactory(g, Rng(0), np.float32)
    x = g.new_slot((8, 64, 32, 32), name="input")
    g.inputs = [x]
    cp = pf.conv("conv1", 64, 64, 3, stride=1, pad=1)
    t0 = g.new_slot((8, 64, 32, 32), name="conv1.out")
    g.add_node(CONV, ConvAttrs(conv=cp), [x], [t0], saved=[x], name="conv1")
    g.outputs = [_bn_relu_conv(g, pf, t0, 64, 1, 1, 0, "mid")]
    g.validate()
    sample = np.random.default_rng(7).integers(0, 8 * 64 * 32 * 32, size=4096)
    for lv in ("baseline", "bnff"):
        g2, _ = fusion.plan(g, fusion.parse_level(lv))
        xin, dy, acts, grads = run_model(g2, 0)
        out = np.asarray(acts.vals[g2.outputs[0]])
        dx = np.asarray(grads.inputs[g2.inputs[0]])
        payload = {"sample_idx": sample,
                   "out_chsum": out.astype(np.float64).sum(axis=(0, 2, 3)),
                   "out_sample": out.reshape(-1)[sample],
                   "dx_chsum": dx.astype(np.float64).sum(axis=(0, 2, 3)),
                   "dx_sample": dx.reshape(-1)[sample],
                   "x_sum": np.float64(xin.astype(np.float64).sum())}
        for k, v in grads.params.items():
            payload[f"grad::{k}"] = np.asarray(v)
        np.savez_compressed(os.path.join(HERE, f"block_c1_{lv}.npz"), **payload)
    print("block c1 done")


def main():
    make_graphs()
    ex = extra_specs()
    small = {
        "single-bn-toy": RG.single_bn_toy(4),
        "densenet-micro": RG.densenet_micro(2),
        "resnet-micro": RG.resnet_micro(2),
        "gradcheck-micro": RG.gradcheck_micro(2),
        "densenet-tiny-full": ex["densenet-tiny-full"],
        "resnet-tiny-strided": ex["resnet-tiny-strided"],
    }
    for name, spec in small.items():
        save_model_case(name, spec, LEVELS, (np.float32,))
        save_model_case(name, spec, ["baseline", "bnff"], (np.float64,))
    make_block_c1()


if __name__ == "__main__":
    main()
