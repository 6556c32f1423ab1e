"""Per-parameter scaled errors of the fp32 densenet-micro-64 fold run vs the fp64 oracle
(diagnostic for test_icf_block_gradient_fold_f32)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from oracle import executor as OX
from paper_1807_01702_b200 import fusion, graph as G
from paper_1807_01702_b200.tensor import Rng
from paper_1807_01702_b200.engine import Engine

def scaled(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))

spec = G.ModelSpec("densenet", (3, 3), 32, 4, (2, 64, 16, 16), "micro", "conv3", name="densenet-micro-64")
g0 = G.build_model(spec, seed=0)
g, _ = fusion.plan(g0, fusion.parse_level(sys.argv[1] if len(sys.argv) > 1 else "bnff+icf"))
rng = Rng(1)
x = rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0)
dy = rng.normal(g.slots[g.outputs[0]].shape)
res = OX.forward(g, {g.inputs[0]: x.astype(np.float64)})
ref = OX.backward(g, res, {g.outputs[0]: dy.astype(np.float64)})
for fold in (True, False):
    eng = Engine(g, dtype="f32", input_grad=True, fold_icf=fold)
    eng.set_input(x); eng.set_loss_grad(dy); eng.forward(); eng.backward(); torch.cuda.synchronize()
    pg = eng.param_grads()
    print("fold", fold, "out", scaled(eng.output(), res.vals[g.outputs[0]]))
    for k, v in ref.params.items():
        e = scaled(pg[k], v)
        print(f"  {k:28s} {e:.2e}{'  <-- ' if e > 1e-4 else ''}")
