"""Builders + rewriter vs fixtures generated from the reference (tests/golden/graphs.json).

Pins: node/slot numbering and names, buffer annotations, attrs, per-level
rewrite counts, unfused-BN ids, bn_map and the bit-exact parameter draws
(sha256 of every parameter array) for every preset and BASELINE config.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_1807_01702_b200 import fusion
from paper_1807_01702_b200 import graph as G

from conftest import GOLDEN

with open(os.path.join(GOLDEN, "graphs.json")) as f:
    GRAPHS = json.load(f)


def spec_from(d):
    return G.ModelSpec(family=d["family"], blocks=tuple(d["blocks"]), growth_rate=d["growth_rate"],
                       bottleneck_mult=d["bottleneck_mult"], input_dims=tuple(d["input_dims"]),
                       scale=d["scale"], stem=d["stem"], base_channels=d["base_channels"],
                       resnet_stages=tuple(tuple(s) for s in d["resnet_stages"]), name=d["name"])


def attrs_summary(node):
    a, out = node.attrs, {}
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


def record(g, fp):
    kinds = sorted({r.kind for r in fp.rewrites})
    return {
        "nodes": [[n.id, n.kind, n.name, list(n.inputs), list(n.outputs),
                   list(n.saved_for_backward), attrs_summary(n)] for n in g.nodes],
        "slots": [[s.id, list(s.shape), s.kind, s.name, list(s.buffer) if s.buffer else None]
                  for s in sorted(g.slots.values(), key=lambda s: s.id)],
        "inputs": list(g.inputs), "outputs": list(g.outputs),
        "buffer_groups": {k: list(v) for k, v in g.buffer_groups.items()},
        "rewrite_counts": {k: fp.count(k) for k in kinds},
        "unfused_bn_ids": list(fp.unfused_bn_ids),
        "bn_map": {str(k): list(v) for k, v in fp.bn_map.items()},
    }


@pytest.mark.parametrize("name", sorted(GRAPHS))
def test_params_bit_identical(name):
    g = G.build_model(spec_from(GRAPHS[name]["spec"]), seed=0)
    got = {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()[:16]
           for k, v in g.params.items()}
    assert sorted(got) == sorted(GRAPHS[name]["params"])
    assert got == GRAPHS[name]["params"]


@pytest.mark.parametrize("name", sorted(GRAPHS))
@pytest.mark.parametrize("level", ["baseline", "rcf", "rcf+mvf", "bnff", "bnff+icf"])
def test_rewrite_matches_reference(name, level):
    g = G.build_model(spec_from(GRAPHS[name]["spec"]), seed=0)
    g2, fp = fusion.plan(g, fusion.parse_level(level))
    want = GRAPHS[name]["levels"][level]
    got = json.loads(json.dumps(record(g2, fp)))
    for key in want:
        assert got[key] == want[key], f"{name}@{level}: {key} differs"


def test_densenet121_counts():
    g = G.build_model(G.densenet121(2))
    assert g.meta["conv_count"] == 120
    g2, fp = fusion.plan(g, fusion.FusionLevel.BNFF)
    kinds = [n.kind for n in g2.nodes]
    assert kinds.count(G.FUSED_NRC) == 119 and kinds.count(G.FUSED_CONV_STATS) == 1
    assert kinds.count(G.SUBBN1) == 62
    g3, _ = fusion.plan(g, fusion.FusionLevel.BNFF_ICF)
    assert [n.kind for n in g3.nodes].count(G.SUBBN1) == 0


def test_params_shared_by_reference():
    g = G.build_model(G.densenet_micro(2))
    g2, _ = fusion.plan(g, fusion.FusionLevel.BNFF_ICF)
    for k, v in g.params.items():
        assert g2.params[k] is v


def test_parse_level_errors():
    from paper_1807_01702_b200.errors import InvalidSpecError
    assert fusion.parse_level("BNFF") is fusion.FusionLevel.BNFF
    with pytest.raises(InvalidSpecError):
        fusion.parse_level("nope")


def test_pad_channels_is_exact_on_the_oracle():
    """graph.pad_channels (k = 12 pieces widened to 16, transitions to multiples of 8):
    the padded graph run by the oracle reproduces the logical graph's outputs bitwise and
    its parameter gradients to fp32 summation-order noise, at every fusion level."""
    import numpy as np
    from oracle import executor as OX
    from paper_1807_01702_b200 import fusion
    from paper_1807_01702_b200.tensor import Rng
    g0 = G.build_model(G.densenet_micro(2, (3, 3), 12), seed=0)
    g2, pm = G.pad_channels(g0, 8)
    assert all(c % 8 == 0 for c, _, _ in g2.buffer_groups.values())
    for lvl in ("baseline", "bnff", "bnff+icf"):
        ga, _ = fusion.plan(g0, fusion.parse_level(lvl))
        gb, _ = fusion.plan(g2, fusion.parse_level(lvl))
        rng = Rng(1)
        x = rng.uniform(ga.slots[ga.inputs[0]].shape, -1.0, 1.0)
        dy = rng.normal(ga.slots[ga.outputs[0]].shape)
        ra = OX.forward(ga, {ga.inputs[0]: x})
        ba = OX.backward(ga, ra, {ga.outputs[0]: dy})
        dyp = pm.pad(g2.outputs[0], dy, gb.slots[gb.outputs[0]].shape[1])
        rb = OX.forward(gb, {gb.inputs[0]: x})
        bb = OX.backward(gb, rb, {gb.outputs[0]: dyp})
        assert np.array_equal(ra.vals[ga.outputs[0]], pm.unpad(g2.outputs[0], rb.vals[gb.outputs[0]]))
        pb = pm.params_from(bb.params)
        for k, v in ba.params.items():
            assert np.max(np.abs(pb[k] - v)) <= 1e-5 * max(float(np.max(np.abs(v))), 1.0), (lvl, k)


def test_cli_bench_schema_matches_reference():
    """The device bench writes the reference's frozen CSV schema (cli.py:109-110) and
    accepts its flags (cli.py:294-317)."""
    import importlib.util
    import os
    from paper_1807_01702_b200 import cli
    ref = "/root/reference/pkg/src/bnfuse/cli.py"
    if os.path.exists(ref):
        src = open(ref).read()
        start = src.index("BENCH_HEADER = [")
        header = eval(src[start + len("BENCH_HEADER = "):src.index("]", start) + 1])  # noqa: S307
        assert cli.BENCH_HEADER == header
    a = cli.make_parser().parse_args(["bench", "--model", "densenet-micro", "--batch", "4", "--fusion",
                                      "all", "--iters", "3", "--warmup", "1", "--seed", "2", "--out",
                                      "x.csv", "--dtype", "f32", "--gpus", "1"])
    assert (a.model, a.batch, a.iterations, a.warmup, a.seed, a.out_path) == ("densenet-micro", 4, 3, 1, 2, "x.csv")
    assert importlib.util.find_spec("paper_1807_01702_b200.cli") is not None
