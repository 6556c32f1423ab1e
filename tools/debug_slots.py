"""Per-slot GPU-vs-oracle diff for one graph/level/dtype (debug aid, GPU box)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import executor as OX
from paper_1807_01702_b200 import fusion, graph as G
from paper_1807_01702_b200.engine import Engine
from paper_1807_01702_b200.tensor import Rng


def scaled(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


def main(level="baseline", dtype="f32", n=8, c=64, hw=32):
    g0 = G.build_block(n, c, hw, seed=0)
    g, _ = fusion.plan(g0, fusion.parse_level(level))
    rng = Rng(1)
    x = rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0)
    dy = rng.normal(g.slots[g.outputs[0]].shape)
    res = OX.forward(g, {g.inputs[0]: x.astype(np.float64)})
    eng = Engine(g, dtype=dtype)
    eng.set_input(x); eng.set_loss_grad(dy)
    eng.forward(); torch.cuda.synchronize()
    for node in g.nodes:
        for s in node.outputs:
            if s in eng.acts and g.slots[s].kind == "feature":
                print(f"{node.kind:20s} {node.name:12s} slot {s}: err {scaled(eng.act(s), res.vals[s]):.3e}")
            if g.slots[s].kind == "stats" and s in eng.stats:
                st = eng.stats_of(s); want = res.vals[s]
                print(f"{node.kind:20s} {node.name:12s} stats {s}: mean {scaled(st['mean'], want.mean):.3e} var {scaled(st['var'], want.var):.3e}")
        if node.kind == G.BN:
            st = eng.node_stats[node.id]
            print("  BN mean/var gpu", st.mean[:4].cpu().numpy(), st.var[:4].cpu().numpy())
            want = res.node_stats[node.id]
            print("  BN mean/var ref", want.mean[:4], want.var[:4])


if __name__ == "__main__":
    main(*sys.argv[1:3])
