"""Per-launch device-time table of one DenseNet-121 training step (CUDA events
between consecutive launches on the launching stream; not a bench number).

    python tools/profile_step.py [--level bnff] [--dtype bf16] [--batch 64] [--top 40]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", default="bnff+icf")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--model", default="densenet121")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--json", default="")
    args = ap.parse_args()
    import torch
    from paper_1807_01702_b200 import fusion, graph as G
    from paper_1807_01702_b200.engine import Engine
    from paper_1807_01702_b200.tensor import Rng

    spec = getattr(G, args.model)(args.batch)
    g, _ = fusion.plan(G.build_model(spec, seed=0), fusion.parse_level(args.level))
    eng = Engine(g, dtype=args.dtype, input_grad=False, lr=1e-3)
    rng = Rng(1)
    eng.set_input(rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0))
    eng.set_loss_grad(rng.normal(g.slots[g.outputs[0]].shape))
    for _ in range(2):
        eng.step()
    torch.cuda.synchronize()
    prof = eng.profile_launches(reps=3)
    total = sum(ms for _, ms in prof)
    by = {}
    for t, ms in prof:
        d = by.setdefault(t.kind, [0.0, 0])
        d[0] += ms
        d[1] += 1
    print(f"# {args.model} b{args.batch} {args.level} {args.dtype}: {len(prof)} C-ABI calls, "
          f"sum of launches {total:.3f} ms")
    for k, (ms, n) in sorted(by.items(), key=lambda kv: -kv[1][0]):
        print(f"  {k:16s} n={n:4d} total={ms:8.3f} ms share={ms / total:.3f}")
    import re
    grp = {}
    for t, ms in prof:
        key = t.kind + " " + re.sub(r"\.l\d+\.", ".l*.", t.what.split(" ", 1)[1] if " " in t.what else "")
        d = grp.setdefault(key, [0.0, 0, 0, 0])
        d[0] += ms
        d[1] += 1
        d[2] += t.nbytes
        d[3] += t.flops
    print("# by layer group")
    for k, (ms, n, b, f) in sorted(grp.items(), key=lambda kv: -kv[1][0])[:30]:
        print(f"  {k:36s} n={n:3d} {ms:7.3f} ms  {b / (ms * 1e-3) / 1e9 if ms else 0:6.0f} GB/s "
              f"{f / (ms * 1e-3) / 1e12 if ms else 0:6.1f} TF/s")
    print("# top launches")
    rows = sorted(prof, key=lambda r: -r[1])[: args.top]
    for t, ms in rows:
        gbs = t.nbytes / (ms * 1e-3) / 1e9 if ms > 0 else 0
        tfs = t.flops / (ms * 1e-3) / 1e12 if ms > 0 else 0
        print(f"  {ms * 1e3:9.1f} us  {t.what:40s} {gbs:7.0f} GB/s {tfs:7.1f} TF/s "
              f"bytes={t.nbytes} flops={t.flops}")
    if args.json:
        with open(args.json, "w") as f:
            json.dump([{"what": t.what, "us": ms * 1e3, "bytes": t.nbytes, "flops": t.flops}
                       for t, ms in prof], f)


if __name__ == "__main__":
    main()
