import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import executor as OX
from paper_1807_01702_b200 import fusion, graph as G
from paper_1807_01702_b200.engine import Engine
from paper_1807_01702_b200.tensor import Rng
spec = G.ModelSpec("densenet", (2, 2), 8, 4, (2, 3, 32, 32), "full", "conv7-pool", 16, name="densenet-tiny-full")
g0 = G.build_model(spec, seed=0)
g, _ = fusion.plan(g0, fusion.parse_level("baseline"))
rng = Rng(1)
x = rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0)
dy = rng.normal(g.slots[g.outputs[0]].shape)
eng = Engine(g, dtype="f32", input_grad=True)
eng.set_input(x); eng.set_loss_grad(dy)
eng.forward(); eng.backward(); torch.cuda.synchronize()
for t in eng.bwd:
    print(t.what)
for k,(c1, colt, dw2, kpad) in eng.cols.items():
    print(k, colt.shape, torch.isnan(colt).sum().item())
dx = eng.input_grads[g.inputs[0]]
print('dx nan', torch.isnan(dx).sum().item(), dx.shape)
nanpos = torch.nonzero(torch.isnan(dx))[:10]
print(nanpos)
# find dcol: the buffer right before dx in _bufs
for b in eng._bufs:
    if b.dim()==4 and b.shape[-1]==160:
        print('buf160', b.shape, torch.isnan(b).sum().item(), b.data_ptr()==colt.data_ptr())
