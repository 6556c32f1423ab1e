import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1807_01702_b200 import fusion, graph as G, kernels as K
from paper_1807_01702_b200.engine import Engine
from paper_1807_01702_b200.tensor import Rng

g0 = G.build_block(8, 64, 32, seed=0)
g, _ = fusion.plan(g0, fusion.parse_level("baseline"))
rng = Rng(1)
x = rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0)
eng = Engine(g, dtype="f32")
eng.set_input(x)
eng.forward(); torch.cuda.synchronize()
conv = next(n for n in g.nodes if n.name == "mid.conv").attrs.conv
xin = eng.acts[3]
y_api = K.conv2d_fwd(xin, conv)
torch.cuda.synchronize()
print("engine vs api:", float((eng.acts[4] - y_api).abs().max()), float(y_api.abs().max()))
wp, wt, cs, _ = eng.packs["mid.conv"]
pc = K.PackedConv(conv, torch.float32, cin_store=64)
print("packs equal:", torch.equal(wp, pc.wp), torch.equal(wt, pc.wt), wp.shape, pc.wp.shape)
print("w master:", float((eng.param("mid.conv.weight").view(64, 64, 1, 1).cpu() - torch.from_numpy(conv.weights)).abs().max()))
# rerun only the fprop thunk for the conv
for i in range(3):
    eng.forward(); torch.cuda.synchronize()
    print("rerun", i, float((eng.acts[4] - y_api).abs().max()))
print("bias", eng.param("mid.conv.bias").abs().max())
print(eng.acts[4].shape, eng.acts[4].stride(), eng.acts[3].stride(), xin.data_ptr() == eng.acts[3].data_ptr())
print("wp[:6]", wp[:6].cpu().numpy(), "api", pc.wp[:6].cpu().numpy(), "w", conv.weights.reshape(-1)[:6])
print("wp argmax diff", int((wp - pc.wp).abs().argmax()), float((wp - pc.wp).abs().max()))
eng._run(eng.repack); torch.cuda.synchronize()
print("after repack equal:", torch.equal(wp, pc.wp), torch.equal(wt, pc.wt))
for name, (a, b, c, cv) in eng.packs.items():
    print(name, a.data_ptr(), a.numel(), b.data_ptr(), b.numel(), cv.out_c, cv.in_c, c)
print("wflat ptr", eng.wflat.data_ptr(), eng.wflat.numel(), {k: v for k, v in eng.poff.items()})
