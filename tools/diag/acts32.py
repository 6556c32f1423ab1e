"""Per-slot forward errors (engine fp32 vs fp64 oracle) of densenet-micro-64 at bnff+icf, with
the worst channels -- diagnostic."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from oracle import executor as OX
from paper_1807_01702_b200 import fusion, graph as G
from paper_1807_01702_b200.tensor import Rng
from paper_1807_01702_b200.engine import Engine

spec = G.ModelSpec("densenet", (3, 3), 32, 4, (2, 64, 16, 16), "micro", "conv3", name="densenet-micro-64")
g0 = G.build_model(spec, seed=0)
g, _ = fusion.plan(g0, fusion.parse_level("bnff+icf"))
rng = Rng(1)
x = rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0)
dy = rng.normal(g.slots[g.outputs[0]].shape)
res = OX.forward(g, {g.inputs[0]: x.astype(np.float64)})
eng = Engine(g, dtype="f32", input_grad=True, fold_icf=True)
eng.set_input(x); eng.set_loss_grad(dy); eng.forward(); torch.cuda.synchronize()
for sid in sorted(eng.acts.keys(), key=lambda s: str(s)):
    if sid not in res.vals:
        continue
    try:
        a = eng.act(sid).astype(np.float64)
    except Exception as e:
        print(sid, "skip", e); continue
    b = np.asarray(res.vals[sid], np.float64)
    if a.shape != b.shape:
        print(sid, "shape", a.shape, b.shape); continue
    d = np.abs(a - b)
    sc = d.max() / max(np.abs(b).max(), 1e-30)
    ch = d.max(axis=(0, 2, 3)) / max(np.abs(b).max(), 1e-30)
    worst = np.argsort(-ch)[:4]
    loc = np.unravel_index(np.argmax(d), d.shape)
    print(f"{str(sid):30s} {g.slots[sid].shape} scaled {sc:.2e} worst ch {list(worst)} {[f'{ch[c]:.1e}' for c in worst]} at {loc}")
print("-- stats (scaled mean / var error)")
for sid, st in eng.stats.items():
    if sid not in res.vals:
        continue
    o = res.vals[sid]
    s = eng.stats_of(sid)
    em = np.abs(s["mean"] - o.mean).max() / max(np.abs(o.mean).max(), 1e-30)
    ev = np.abs(s["var"] - o.var).max() / max(np.abs(o.var).max(), 1e-30)
    print(f"  {str(sid):8s} C={len(o.mean)} mean {em:.2e} var {ev:.2e} minvar {o.var.min():.3e}")
print("-- backward launches")
print(" ".join(t.what for t in eng.bwd))
print("-- ReLU mask flips (engine fp32 forward state vs fp64 oracle) per FusedNormReluConv")
for n in g.nodes:
    if n.kind != "FusedNormReluConv":
        continue
    xs, ss = n.inputs[0], n.inputs[1]
    bn = n.attrs.bn
    gam = np.asarray(bn.gamma, np.float64)[None, :, None, None]
    bet = np.asarray(bn.beta, np.float64)[None, :, None, None]
    o = res.vals[ss]
    xo = np.asarray(res.vals[xs], np.float64)
    yo = (xo - o.mean[None, :, None, None]) / np.sqrt(o.var[None, :, None, None] + bn.eps) * gam + bet
    s = eng.stats_of(ss)
    xe = eng.act(xs).astype(np.float64)
    ye = (xe - s["mean"][None, :, None, None]) / np.sqrt(s["var"][None, :, None, None] + bn.eps) * gam + bet
    flip = (yo > 0) != (ye > 0)
    print(f"  {n.name:18s} flips {int(flip.sum())} min|y| {np.abs(yo).min():.2e} at flips {np.abs(yo[flip]).max() if flip.any() else 0:.2e}")
