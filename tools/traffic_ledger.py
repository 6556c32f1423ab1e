"""Measured-vs-analytic traffic ledger (the reference's count_sweeps /
compare_ledgers, traffic.py:222-231, 355-365): per launch class of one DenseNet-121 b64
step, the algorithmic HBM bytes the engine attaches to every launch (each tensor counted
once per launch) next to the ncu-measured DRAM bytes of the same class
(profiles/step_dram_bytes.json, ncu --cache-control none over one captured step).

    python tools/traffic_ledger.py [--level bnff+icf] [--json out.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# engine launch kind -> ncu kernel class (tools/ncu_step_bytes.kernel_class)
_KIND_TO_CLASS = {"channel_sums": "channel_sums", "bn_bwd_sums": "channel_sums", "split_bwd": "grad_sum",
                  "bn_dx": "grad_sum", "grad_add": "grad_sum", "subbn2": "bn_apply", "relu_fwd": "relu",
                  "relu_bwd": "relu", "avgpool_bwd": "avgpool", "pack_weights": "pack",
                  "cols_to_weight": "other"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", default="bnff+icf")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    from paper_1807_01702_b200 import fusion, graph as G
    from paper_1807_01702_b200.engine import Engine
    g, _ = fusion.plan(G.build_model(G.densenet121(a.batch), seed=0), fusion.parse_level(a.level))
    eng = Engine(g, dtype="bf16", input_grad=False, lr=1e-3)
    algo = {}
    for t in eng.all_thunks():
        cls = _KIND_TO_CLASS.get(t.kind, t.kind)
        d = algo.setdefault(cls, [0, 0])
        d[0] += t.nbytes
        d[1] += 1
    with open(os.path.join(ROOT, "profiles", "step_dram_bytes.json")) as f:
        meas = json.load(f)["runs"][f"bytes_{a.level}.csv"]
    rows = []
    for cls in sorted(set(algo) | set(meas), key=lambda c: -max(algo.get(c, [0])[0], meas.get(c, {}).get("dram_bytes", 0))):
        ab = algo.get(cls, [0, 0])[0]
        mb = meas.get(cls, {}).get("dram_bytes", 0.0)
        rows.append({"class": cls, "algorithmic_bytes": ab, "ncu_dram_bytes": mb,
                     "ratio": (mb / ab) if ab else None})
    print(f"# DenseNet-121 b{a.batch} {a.level}: algorithmic (engine) vs ncu DRAM bytes per step")
    print(f"{'class':16s} {'algorithmic GB':>15s} {'ncu DRAM GB':>12s} {'ncu/alg':>8s}")
    for r in rows:
        ratio = f"{r['ratio']:.2f}" if r["ratio"] is not None else "-"
        print(f"{r['class']:16s} {r['algorithmic_bytes'] / 1e9:15.3f} {r['ncu_dram_bytes'] / 1e9:12.3f} {ratio:>8s}")
    ta = sum(r["algorithmic_bytes"] for r in rows)
    tm = sum(r["ncu_dram_bytes"] for r in rows)
    print(f"{'total':16s} {ta / 1e9:15.3f} {tm / 1e9:12.3f} {tm / ta:8.2f}")
    if a.json:
        with open(a.json, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
