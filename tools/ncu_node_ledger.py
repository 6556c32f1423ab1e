"""Per-node traffic ledger on the device: the reference rulebook (traffic.count_sweeps) vs
the bytes the engine's launches must touch vs the DRAM bytes ncu measured for them,
node by node (the reference's compare_ledgers idea, traffic.py:355-365, with measured
hardware bytes instead of the executor's self-reported sweeps).

    ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum \
        --csv --log-file out.csv python tools/ncu_node_ledger.py run --dtype bf16
    python tools/ncu_node_ledger.py summarize out.csv --dtype bf16 [--json ledger.json]

`run` executes one eager training step (forward, backward, optimizer) with an empty
marker kernel launched before every engine launch; `summarize` cuts the ncu launch list
at the markers, attributes each group to the graph node that emitted the launch, and
prints the per-node and per-kind comparison.
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(dtype, level, batch):
    from paper_1807_01702_b200 import fusion, graph as G
    from paper_1807_01702_b200.engine import Engine
    from paper_1807_01702_b200.tensor import Rng
    g, _ = fusion.plan(G.build_model(G.densenet121(batch), seed=0), fusion.parse_level(level))
    eng = Engine(g, dtype=dtype, input_grad=True, lr=1e-3, side_wgrad=False)
    rng = Rng(1)
    eng.set_input(rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0))
    eng.set_loss_grad(rng.normal(g.slots[g.outputs[0]].shape))
    return g, eng


def run(a):
    import ctypes as C
    import torch
    g, eng = build(a.dtype, a.level, a.batch)
    eng.step()  # warm
    torch.cuda.synchronize()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for i, t in enumerate(eng.all_thunks()):
        eng.L.bnff_debug_mark(i, s)
        t(s)
    torch.cuda.synchronize()


def read_ncu(path):
    rows = {}
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        key = int(r["ID"])
        unit = r.get("Metric Unit", "byte")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        val = float(r["Metric Value"].replace(",", "")) * scale
        name, acc = rows.get(key, (r["Kernel Name"], 0.0))
        rows[key] = (name, acc + val)
    return [rows[k] for k in sorted(rows)]


def summarize(a):
    from paper_1807_01702_b200 import traffic
    g, eng = build(a.dtype, a.level, a.batch)
    bpe = 2 if a.dtype == "bf16" else 4
    rule = traffic.count_sweeps(g, concat_physical=False, bytes_per_elem=bpe)
    dev = traffic.device_ledger(eng)
    meas = traffic.ncu_ledger(read_ncu(a.csv), eng)
    rows = traffic.compare(g, rule, dev, meas)
    kinds: dict = {}
    for r in rows:
        k = kinds.setdefault(r["kind"], [0, 0, 0.0, 0])
        k[0] += r["rulebook_bytes"]
        k[1] += r["device_bytes"]
        k[2] += r["ncu_bytes"] or 0.0
        k[3] += 1
    other = meas.get(-1, 0.0)
    print(f"# DenseNet-121 b{a.batch} {a.level} {a.dtype}: per node kind, bytes per training step")
    print(f"{'kind':20s} {'nodes':>5s} {'rulebook GB':>12s} {'device GB':>10s} {'ncu DRAM GB':>12s} {'ncu/rule':>9s}")
    for kind, (rb, db, nb, n) in sorted(kinds.items(), key=lambda kv: -kv[1][0]):
        ratio = f"{nb / rb:.2f}" if rb else "-"
        print(f"{kind:20s} {n:5d} {rb / 1e9:12.3f} {db / 1e9:10.3f} {nb / 1e9:12.3f} {ratio:>9s}")
    tr = sum(v[0] for v in kinds.values())
    td = sum(v[1] for v in kinds.values())
    tn = sum(v[2] for v in kinds.values())
    print(f"{'total (nodes)':20s} {'':5s} {tr / 1e9:12.3f} {td / 1e9:10.3f} {tn / 1e9:12.3f} {tn / tr:9.2f}")
    print(f"optimizer / repack launches (no node): ncu {other / 1e9:.3f} GB")
    # per launch class (engine thunk kind): the bench's roofline.traffic source
    thunks = eng.all_thunks()
    by_kind: dict = {}
    ti = -1
    for name, nb in read_ncu(a.csv):
        if "mark_kernel" in name:
            ti += 1
            continue
        if 0 <= ti < len(thunks):
            d = by_kind.setdefault(thunks[ti].kind, {"launches": 0, "dram_bytes": 0.0, "kernels": 0})
            d["dram_bytes"] += nb
            d["kernels"] += 1
    for t in thunks:
        if t.kind in by_kind:
            by_kind[t.kind]["launches"] += 1
    if a.step_bytes:
        path = a.step_bytes
        meas = {"how": "", "runs": {}}
        if os.path.exists(path):
            with open(path) as f:
                meas = json.load(f)
        meas["how"] = ("ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum over one "
                       "eager D121 b64 training step (tools/ncu_node_ledger.py); per engine launch class: "
                       "launches = engine launches (thunks) of the class, dram_bytes = their summed DRAM bytes")
        meas["runs"][f"bytes_{a.dtype}_{a.level}.csv"] = by_kind
        with open(path, "w") as f:
            json.dump(meas, f, indent=1, sort_keys=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"model": "densenet-121", "batch": a.batch, "level": a.level, "dtype": a.dtype,
                       "bytes_per_elem": bpe, "per_node": rows,
                       "per_kind": {k: {"nodes": v[3], "rulebook_bytes": v[0], "device_bytes": v[1],
                                        "ncu_bytes": v[2]} for k, v in kinds.items()},
                       "unattributed_ncu_bytes": other}, f, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["run", "summarize"])
    ap.add_argument("csv", nargs="?", default="")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--level", default="bnff+icf")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--json", default="")
    ap.add_argument("--step-bytes", default="", help="merge per-class bytes into this step_dram_bytes.json")
    a = ap.parse_args()
    run(a) if a.mode == "run" else summarize(a)


if __name__ == "__main__":
    main()
