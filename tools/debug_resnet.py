"""Find the first failing launch of a model step: eager launches, synchronize after each."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1807_01702_b200 import fusion, graph as G
from paper_1807_01702_b200.engine import Engine
from paper_1807_01702_b200.tensor import Rng

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 4
level = sys.argv[2] if len(sys.argv) > 2 else "bnff"
g, _ = fusion.plan(G.build_model(G.resnet50(batch), seed=0), fusion.parse_level(level))
eng = Engine(g, dtype="bf16", input_grad=False, lr=1e-3, side_wgrad=False)
rng = Rng(1)
eng.set_input(rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0))
eng.set_loss_grad(rng.normal(g.slots[g.outputs[0]].shape))
torch.cuda.synchronize()
s = eng._stream()
for i, t in enumerate(eng.all_thunks()):
    try:
        t(s)
        torch.cuda.synchronize()
    except Exception as e:
        print("FAILED at", i, t.what, repr(e)[:300])
        prev = eng.all_thunks()[max(0, i - 3):i]
        print("previous:", [p.what for p in prev])
        raise SystemExit(1)
print("all", len(eng.all_thunks()), "launches ok")
