"""GPU parity on the BENCHED topologies: DenseNet-121 (C3), DenseNet-BC-100 k=12 (C2) and
ResNet-50 (C4) at batch 2, through the device Engine, against the fp64 oracle
(the reference's own whole-model check runs entire graphs the same way,
``verify.py:46-73``; builders ``graph.py:392-523``).

Bars (stated here, per the north star, and why):
  These graphs at batch 2 are badly conditioned in their GRADIENTS: the reference's own
  fp32 run (numpy, this oracle in fp32) sits at a median scaled-max error of 1.2e-3
  (DenseNet-121), 2.8e-4 (BC-100) and 1.2e-2 (ResNet-50) from fp64, up to 3e-2 / 1e-1
  on single tensors -- ReLU masks flip where a pre-activation is within rounding of zero
  and BN over 98 pixels per channel amplifies it (batch 8 is worse, not better).  A flat
  1e-4 bar on every end-to-end gradient is unattainable by the reference's own fp32
  arithmetic, so the check is split at the discontinuity:
  * fp32 mode (fp32 storage, 3xTF32 tcgen05, f64 statistics):
      - FORWARD: output and every BN statistics vector within scaled max 2e-4 of fp64;
      - BACKWARD at fixed forward state: the oracle's fp64 backward run over the
        device's own forward activations/statistics (no ReLU decision can differ), every
        parameter gradient and the input gradient within relative L2 2e-4;
      - post-step weights: exactly the SGD of the device gradients (1e-6);
      - end-to-end gradients vs fp64: recorded beside the reference-fp32 floor
        (BNFF_PARITY_LOG), not barred.
    The 2e-4 (vs 1e-4 at block/micro scale, test_gpu_parity.py) is the stated 3xTF32
    tolerance at depth: tcgen05 accumulates fp32 with truncation, so one conv with
    K ~ 1100 lands at 7.9e-6 relative RMS vs 2.1e-7 for a CPU sgemm regardless of the
    split's term set (tools/tf32_probe.py, profiles/r2_tf32_probe.txt), and 50-120
    layers compound it.
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import executor as OX  # noqa: E402
from paper_1807_01702_b200 import fusion  # noqa: E402
from paper_1807_01702_b200 import graph as G  # noqa: E402
from paper_1807_01702_b200.tensor import Rng  # noqa: E402

F32_FWD = 2e-4
F32_BWD = 2e-4
BF16_OUT = 1e-1
LR = 0.1

MODELS = {
    "densenet-121": lambda: G.densenet121(2),
    "densenet-bc-100": lambda: G.densenet_bc100(2),
    "resnet-50": lambda: G.resnet50(2),
}

_ORACLE: dict = {}


def scaled(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(float(np.linalg.norm(b)), 1e-30))


def oracle(model, level):
    """fp64 oracle forward + backward of the planned graph (cached per model/level)."""
    key = (model, level)
    if key not in _ORACLE:
        g0 = G.build_model(MODELS[model](), seed=0)
        g, _ = fusion.plan(g0, fusion.parse_level(level))
        rng = Rng(1)
        x = rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0)
        dy = rng.normal(g.slots[g.outputs[0]].shape)
        res = OX.forward(g, {g.inputs[0]: x.astype(np.float64)})
        ref = OX.backward(g, res, {g.outputs[0]: dy.astype(np.float64)})
        # the reference's own fp32 arithmetic on the same inputs: its distance from fp64 is
        # the conditioning floor of this graph at this batch
        r32 = OX.forward(g, {g.inputs[0]: x.astype(np.float32)})
        b32 = OX.backward(g, r32, {g.outputs[0]: dy.astype(np.float32)})
        _ORACLE[key] = (g0, g, x, dy, res, ref, r32, b32)
    return _ORACLE[key]


def _report(tag, errs, floor=None):
    path = os.environ.get("BNFF_PARITY_LOG")
    if path:
        import json
        with open(path, "a") as f:
            f.write(json.dumps({"case": tag, "errors": errs, "cpu_fp32_floor": floor}) + "\n")


def _floors(g, res, ref, r32, b32, metric):
    """Distance of the reference's own fp32 run from fp64, tensor by tensor (same metric)."""
    fl = {"__out__": metric(r32.vals[g.outputs[0]], res.vals[g.outputs[0]])}
    for k, v in ref.params.items():
        if k.endswith(".bias"):
            scale = max(float(np.max(np.abs(ref.params[_conv_of_bias(k)]))), 1e-30)
            fl[k] = float(np.max(np.abs(b32.params[k] - v))) / scale
        else:
            fl[k] = metric(b32.params[k], v)
    if b32.inputs.get(g.inputs[0]) is not None:
        fl["__dx__"] = metric(b32.inputs[g.inputs[0]], ref.inputs[g.inputs[0]])
    return fl


def device_forward_state(g, eng, res):
    """The oracle's forward Result with every activation and statistic replaced by the
    device's own (fp64 copies): the oracle backward over it differs from the device
    backward only by backward arithmetic -- no ReLU decision can flip between them,
    because both read the same pre-activations."""
    from oracle import ops as O
    from oracle.executor import Result
    from paper_1807_01702_b200.params import ChannelStats
    vals = {}
    for sid, v in res.vals.items():
        if isinstance(v, np.ndarray):
            vals[sid] = eng.act(sid).astype(np.float64) if (sid in eng.acts and sid not in g.inputs) else v
        elif sid in eng.stats:
            st = eng.stats_of(sid)
            vals[sid] = ChannelStats(st["sum"], st["sumsq"], v.count, st["mean"], st["var"])
        else:
            vals[sid] = v
    for node in g.nodes:  # the saved post-ReLU input is recomputed from x on the device too
        if node.kind == G.FUSED_NRC and node.outputs[1] not in eng.acts:
            x, st = vals[node.inputs[0]], vals[node.inputs[1]]
            vals[node.outputs[1]] = O.relu_fwd(O.bn_apply(x, st, node.attrs.bn))
    node_stats = {}
    for nid, v in res.node_stats.items():
        d = eng.node_stats.get(nid)
        node_stats[nid] = v if d is None else ChannelStats(
            d.sum.cpu().numpy(), d.sumsq.cpu().numpy(), v.count, d.mean.cpu().numpy(), d.var.cpu().numpy())
    return Result(vals, node_stats)


def _conv_of_bias(name):
    return name[: -len(".bias")] + ".weight"


@pytest.mark.parametrize("level", ["baseline", "bnff+icf"])
@pytest.mark.parametrize("model", list(MODELS))
def test_benched_model_f32(model, level):
    from paper_1807_01702_b200.engine import Engine
    g0, g, x, dy, res, ref, r32, b32 = oracle(model, level)
    if any(sl.kind == "feature" and sl.shape[1] % 4 for sid, sl in g0.slots.items() if sid not in g0.inputs):
        pytest.skip("fp32 16-byte rows need pad_channels (BC-100's 150-channel transition): "
                    "covered by test_padded_growth12_densenet")
    eng = Engine(g, dtype="f32", input_grad=True, lr=LR)
    eng.set_input(x)
    eng.set_loss_grad(dy)
    eng.forward()
    eng.backward()
    torch.cuda.synchronize()
    flat = {"__out__": scaled(eng.output(), res.vals[g.outputs[0]])}
    grads = eng.param_grads()
    errs = {}
    for k, v in ref.params.items():
        if k.endswith(".bias"):
            scale = max(float(np.max(np.abs(ref.params[_conv_of_bias(k)]))), 1e-30)
            errs[k] = float(np.max(np.abs(grads[k] - v))) / scale
        else:
            errs[k] = rel_l2(grads[k], v)
    errs["__dx__"] = rel_l2(eng.input_grad_nchw(), ref.inputs[g.inputs[0]])
    for sid in eng.stats:  # every BN statistics slot the device produced
        want = res.vals.get(sid)
        if want is None:
            continue
        got = eng.stats_of(sid)
        flat[f"__stats{sid}.mean__"] = scaled(got["mean"], want.mean)
        flat[f"__stats{sid}.var__"] = scaled(got["var"], want.var)
    # post-step weights: the device SGD applied to the device gradients, exactly
    # (w' = w - lr * g in fp32; the gradients themselves are held to the bars below)
    eng.optimizer_step()
    torch.cuda.synchronize()
    now = eng.params_now()
    for k, w0 in g.params.items():
        want = np.asarray(w0, np.float32) - np.float32(LR) * grads[k].astype(np.float32)
        flat[f"post::{k}"] = float(np.max(np.abs(now[k] - want))) / max(float(np.max(np.abs(want))), 1e-30)
    # backward parity at fixed forward state: oracle backward over the device's activations
    bgf = OX.backward(g, device_forward_state(g, eng, res), {g.outputs[0]: dy.astype(np.float64)})
    bw = {}
    for k, v in bgf.params.items():
        if k.endswith(".bias"):
            scale = max(float(np.max(np.abs(bgf.params[_conv_of_bias(k)]))), 1e-30)
            bw[f"bwd::{k}"] = float(np.max(np.abs(grads[k] - v))) / scale
        else:
            bw[f"bwd::{k}"] = rel_l2(grads[k], v)
    bw["bwd::__dx__"] = rel_l2(eng.input_grad_nchw(), bgf.inputs[g.inputs[0]])
    floor = _floors(g, res, ref, r32, b32, rel_l2)
    _report(f"{model}/{level}/f32", {**flat, **errs, **bw}, floor)
    post = {k: e for k, e in flat.items() if k.startswith("post::")}
    fwd = {k: e for k, e in flat.items() if not k.startswith("post::")}
    bad = {k: e for k, e in fwd.items() if e > F32_FWD}
    assert not bad, f"forward above {F32_FWD}: " + ", ".join(
        f"{k}={e:.2e}" for k, e in sorted(bad.items(), key=lambda kv: -kv[1])[:8])
    bad = {k: e for k, e in post.items() if e > 1e-6}
    assert not bad, "post-step weights != SGD of the device gradients: " + ", ".join(
        f"{k}={e:.2e}" for k, e in sorted(bad.items(), key=lambda kv: -kv[1])[:8])
    bad = {k: e for k, e in bw.items() if e > F32_BWD}
    assert not bad, f"backward at fixed forward state above {F32_BWD}: " + ", ".join(
        f"{k}={e:.2e}" for k, e in sorted(bad.items(), key=lambda kv: -kv[1])[:8])
    assert all(np.isfinite(e) for e in errs.values())


@pytest.mark.parametrize("level", ["baseline", "bnff+icf"])
@pytest.mark.parametrize("model", list(MODELS))
def test_benched_model_bf16(model, level):
    from paper_1807_01702_b200.engine import Engine
    g0, g, x, dy, res, ref, r32, b32 = oracle(model, level)
    pad = any(sl.kind == "feature" and sl.shape[1] % 8
              for sid, sl in g0.slots.items() if sid not in g0.inputs)
    if pad:  # growth rate 12: the exact-zero padded graph (graph.pad_channels) on the device
        g2, pm = G.pad_channels(g0, 8)
        gd, _ = fusion.plan(g2, fusion.parse_level(level))
        eng = Engine(gd, dtype="bf16", input_grad=False)
        eng.set_input(x)
        eng.set_loss_grad(pm.pad(g2.outputs[0], dy, gd.slots[gd.outputs[0]].shape[1]))
        eng.forward()
        eng.backward()
        torch.cuda.synchronize()
        out = pm.unpad(g2.outputs[0], eng.output())
        grads = pm.params_from(eng.param_grads())
    else:
        eng = Engine(g, dtype="bf16", input_grad=False)
        eng.set_input(x)
        eng.set_loss_grad(dy)
        eng.forward()
        eng.backward()
        torch.cuda.synchronize()
        out = eng.output()
        grads = eng.param_grads()
    errs = {"__out__": rel_l2(out, res.vals[g.outputs[0]])}
    for k, v in ref.params.items():
        if not k.endswith(".bias"):
            errs[k] = rel_l2(grads[k], v)
    _report(f"{model}/{level}/bf16", errs, _floors(g, res, ref, r32, b32, rel_l2))
    assert errs["__out__"] <= BF16_OUT, errs["__out__"]
    assert all(np.isfinite(e) for e in errs.values())
