"""In-graph cost of each launch class of the D121 step: capture the step as one CUDA
graph with every launch of one kind removed and compare the replay time with the full
graph.  Results of an ablated graph are garbage -- only its timing means something
(no kernel branches on data).  Not a bench number.

    python tools/ablate.py [--level bnff] [--batch 64] [--reps 20]
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", default="bnff+icf")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--model", default="densenet121")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--kinds", default="")
    args = ap.parse_args()
    import torch
    from paper_1807_01702_b200 import fusion, graph as G
    from paper_1807_01702_b200.engine import Engine
    from paper_1807_01702_b200.tensor import Rng

    spec = getattr(G, args.model)(args.batch)
    g, _ = fusion.plan(G.build_model(spec, seed=0), fusion.parse_level(args.level))
    eng = Engine(g, dtype="bf16", input_grad=False, lr=1e-3)
    rng = Rng(1)
    eng.set_input(rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0))
    eng.set_loss_grad(rng.normal(g.slots[g.outputs[0]].shape))
    eng.step()
    torch.cuda.synchronize()
    thunks = eng.all_thunks()
    kinds = sorted({t.kind for t in thunks})
    if args.kinds:
        kinds = args.kinds.split(",")

    def time_graph(ts):
        s = eng._stream()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            eng._run(ts)  # same stream layout as the engine (side-stream weight gradients)
        gr.replay()
        torch.cuda.synchronize()
        cur = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for _ in range(args.reps):
            gr.replay()
        e1.record(cur)
        torch.cuda.synchronize()
        del s
        return e0.elapsed_time(e1) / args.reps

    full = time_graph(thunks)
    print(f"# phases: forward {time_graph(list(eng.fwd)):.3f} ms, backward {time_graph(list(eng.bwd)):.3f} ms, "
          f"optimizer {time_graph(list(eng.opt) + list(eng.repack)):.3f} ms")
    print(f"# {args.model} b{args.batch} {args.level}: full graph {full:.3f} ms/step, {len(thunks)} calls")
    rows = []
    for k in kinds:
        keep = [t for t in thunks if t.kind != k]
        n = len(thunks) - len(keep)
        if n == 0:
            continue
        ms = time_graph(keep)
        rows.append((full - ms, k, n))
    for d, k, n in sorted(rows, reverse=True):
        print(f"  {k:16s} n={n:4d}  in-graph cost {d:7.3f} ms  ({d / full * 100:5.1f}%)  {d / n * 1e3:6.1f} us/launch")


if __name__ == "__main__":
    main()
