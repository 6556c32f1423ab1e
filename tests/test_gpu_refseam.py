"""The drop-in at the reference's own seam (refseam.py), against the UNMODIFIED
reference package installed in baseline/_ref (pip install --no-deps of
/root/reference/pkg; it travels to the GPU box with the repo snapshot).

  * install(): the reference executor's own handler tables (_FWD_HANDLERS /
    _BWD_HANDLERS, execute.py:294-307, 477-490) rebound to device kernels; the
    reference's forward/backward (execute.py:513-558) then runs its graphs -- built by
    its own builders -- on the GPU and must match its CPU run (fp32, rel 1e-4 on
    activations and gradients: the reference's own level-equivalence bars are 1e-4 /
    1e-3, verify.py:34-37);
  * refseam.forward/backward: the same signatures on the compiled Engine, fed the
    reference's Graph object directly.
"""

import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def bnfuse():
    if not os.path.isdir(os.path.join(REF, "bnfuse")):
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, REF)
    import bnfuse  # noqa: F401
    from bnfuse import execute, fusion, graph, tensor
    return execute, fusion, graph, tensor


def scaled(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


def _case(bnfuse, preset, level):
    execute, fusion, graph, tensor = bnfuse
    if preset == "densenet-micro-k8":  # 16-byte channel rows throughout (the Engine's layout)
        spec = graph.densenet_micro(2, (3, 3), 8)
    else:
        spec = graph.PRESETS[preset](2)
    g0 = graph.build_model(spec, seed=0)
    g, _ = fusion.plan(g0, fusion.parse_level(level))
    rng = tensor.Rng(1)
    x = rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0)
    loss = {s: rng.normal(g.slots[s].shape) for s in g.outputs}
    return g, x, loss


def _compare(g, acts_a, grads_a, acts_b, grads_b, tol=1e-4):
    for sid in g.outputs:
        assert scaled(acts_b.get(sid), acts_a.get(sid)) < tol, f"output {sid}"
    for k, v in grads_a.params.items():
        if k.endswith(".bias"):  # conv biases feeding a BN: analytically zero gradient
            w = grads_a.params[k[:-5] + ".weight"]
            assert np.max(np.abs(grads_b.params[k] - v)) <= tol * max(np.max(np.abs(w)), 1e-30), k
            continue
        assert scaled(grads_b.params[k], v) < tol, k


@pytest.mark.parametrize("level", ["baseline", "bnff", "bnff+icf"])
@pytest.mark.parametrize("preset", ["densenet-micro", "resnet-micro", "single-bn-toy"])
def test_installed_handlers_run_reference_executor(bnfuse, preset, level):
    from paper_1807_01702_b200 import refseam
    execute = bnfuse[0]
    g, x, loss = _case(bnfuse, preset, level)
    ctx = execute.ExecCtx(budget=64 << 20)
    acts_cpu = execute.forward(g, x, ctx=ctx)
    grads_cpu = execute.backward(g, acts_cpu, loss, ctx=ctx)
    ref_fwd = dict(execute._FWD_HANDLERS)
    refseam.install(execute)
    try:
        assert all(execute._FWD_HANDLERS[k] is not ref_fwd[k] for k in ref_fwd), "not installed"
        calls = []
        orig = refseam.K._call

        def counting(fn, *a, **kw):
            calls.append(kw.get("what", ""))
            return orig(fn, *a, **kw)
        refseam.K._call = counting
        try:
            acts_gpu = execute.forward(g, x, ctx=execute.ExecCtx(budget=64 << 20))
            grads_gpu = execute.backward(g, acts_gpu, loss, ctx=execute.ExecCtx(budget=64 << 20))
        finally:
            refseam.K._call = orig
        assert calls, "no device kernel launched through the installed handlers"
    finally:
        refseam.uninstall(execute)
    assert execute._FWD_HANDLERS == ref_fwd
    _compare(g, acts_cpu, grads_cpu, acts_gpu, grads_gpu)


@pytest.mark.parametrize("level", ["baseline", "bnff+icf"])
@pytest.mark.parametrize("preset", ["densenet-micro-k8", "resnet-micro"])
def test_engine_entry_points_on_reference_graph(bnfuse, preset, level):
    from paper_1807_01702_b200 import refseam
    execute = bnfuse[0]
    g, x, loss = _case(bnfuse, preset, level)
    acts_cpu = execute.forward(g, x, ctx=execute.ExecCtx(budget=64 << 20))
    grads_cpu = execute.backward(g, acts_cpu, loss)
    acts = refseam.forward(g, x, "train", refseam.ExecCtx(dtype="f32"))
    grads = refseam.backward(g, acts, loss)
    _compare(g, acts_cpu, grads_cpu, acts, grads)
    assert scaled(grads.inputs[g.inputs[0]], grads_cpu.inputs[g.inputs[0]]) < 1e-4
