"""One eager training step of a small model under compute-sanitizer (memcheck of every launch)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1807_01702_b200 import fusion, graph as G
from paper_1807_01702_b200.engine import Engine
from paper_1807_01702_b200.tensor import Rng

which = sys.argv[1] if len(sys.argv) > 1 else "densenet"
if which == "densenet":
    spec = G.ModelSpec("densenet", (3, 3), 16, 4, (2, 3, 64, 64), "full", "conv7-pool", 32, name="dn-small")
    g0 = G.build_model(spec, seed=0)
elif which == "densenet12":
    g0, _ = G.pad_channels(G.build_model(G.densenet_micro(2, (3, 3), 12), seed=0), 8)
else:
    g0 = G.build_model(G.resnet50(2), seed=0)
for level in ("baseline", "bnff", "bnff+icf"):
    g, _ = fusion.plan(g0, fusion.parse_level(level))
    eng = Engine(g, dtype="bf16", input_grad=False, lr=1e-3)
    rng = Rng(1)
    eng.set_input(rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0))
    eng.set_loss_grad(rng.normal(g.slots[g.outputs[0]].shape))
    eng.step()
    torch.cuda.synchronize()
    print(which, level, "ok", len(eng.all_thunks()), "launches")
