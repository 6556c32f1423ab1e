"""BASELINE config C5: BN-layer sweep over C and HxW, fused (BNFF) vs unfused chain.

Each point is one BN layer between two convs, CONV1x1 -> BN -> ReLU -> CONV1x1 (C -> C,
batch N, bf16), run as one captured training step (fwd + bwd) through the device
engine (the 1x1 convs keep every C on the tcgen05 window kernels, so the comparison
isolates the BN restructuring).  Bytes: ncu with caches flushed before every kernel,
DRAM reads + bytes written into L2 (every written byte reaches HBM eventually).  Modes:

    # device time per step + algorithmic BN-tensor sweeps (no profiler)
    python tools/c5_sweep.py --time --out gpurun_out/c5_time.json
    # ncu HBM bytes per step, one NVTX range per (point, level)
    ncu --profile-from-start off --cache-control all --nvtx \
        --metrics dram__bytes_read.sum,lts__t_sectors_op_write.sum,gpu__time_duration.sum \
        --csv --log-file gpurun_out/c5_ncu.csv python tools/c5_sweep.py --ncu
    python tools/c5_sweep.py --summarize gpurun_out/c5_ncu.csv gpurun_out/c5_time.json
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

POINTS = [(c, hw) for c in (64, 128, 256, 512, 1024) for hw in (7, 14, 28, 56, 112)
          if c * hw * hw <= 512 * 56 * 56]
LEVELS = ("baseline", "bnff")


def _engine(c, hw, level, n):
    from paper_1807_01702_b200 import fusion, graph as G
    from paper_1807_01702_b200.engine import Engine
    from paper_1807_01702_b200.tensor import Rng
    g, _ = fusion.plan(G.build_block(n, c, hw, seed=0, k1=1), fusion.parse_level(level))
    eng = Engine(g, dtype="bf16", input_grad=True, lr=0.0)
    rng = Rng(1)
    eng.set_input(rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0))
    eng.set_loss_grad(rng.normal(g.slots[g.outputs[0]].shape))
    eng.capture()
    return eng


def run_time(n, out):
    import torch
    res = []
    for c, hw in POINTS:
        row = {"C": c, "HW": hw, "N": n}
        for level in LEVELS:
            eng = _engine(c, hw, level, n)
            for _ in range(3):
                eng.step()
            torch.cuda.synchronize()
            st = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 20
            e0.record(st)
            for _ in range(reps):
                eng.step()
            e1.record(st)
            torch.cuda.synchronize()
            row[f"{level}_us"] = e0.elapsed_time(e1) / reps * 1e3
            del eng
        T = n * c * hw * hw * 2  # bytes of one BN-sized bf16 tensor
        row["T_bytes"] = T
        row["speedup"] = row["baseline_us"] / row["bnff_us"]
        print(json.dumps(row), flush=True)
        res.append(row)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


def run_ncu(n):
    import torch
    for c, hw in POINTS:
        for level in LEVELS:
            eng = _engine(c, hw, level, n)
            for _ in range(2):
                eng.step()
            torch.cuda.synchronize()
            torch.cuda.nvtx.range_push(f"C{c}_HW{hw}_{level}")
            torch.cuda.cudart().cudaProfilerStart()
            eng.step()
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStop()
            torch.cuda.nvtx.range_pop()
            del eng


def summarize(ncu_csv, time_json):
    with open(ncu_csv) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.reader(lines)
    hdr = next(rd)
    im, iv, iid = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    nv = [i for i, h in enumerate(hdr) if "Push/Pop_Range" in h or h.startswith("thread Domain")]
    acc = {}
    for r in rd:
        raw = next((r[i] for i in nv if r[i]), "")
        # '<pid>  "<default domain>:<range>:none:..."'
        tag = raw.split("<default domain>:", 1)[1].split(":", 1)[0] if "<default domain>:" in raw else "?"
        d = acc.setdefault(tag, {})
        d[r[im]] = d.get(r[im], 0.0) + float(r[iv].replace(",", ""))
    times = {}
    if time_json and os.path.exists(time_json):
        for row in json.load(open(time_json)):
            times[(row["C"], row["HW"])] = row
    out = []
    print(f"{'C':>5} {'HW':>4} {'T MB':>8} {'unfused GB':>11} {'fused GB':>9} {'cut':>6} "
          f"{'unf us':>8} {'fus us':>8} {'speedup':>7} {'fused GB/s':>10}")
    for c, hw in POINTS:
        u = acc.get(f"C{c}_HW{hw}_baseline", {})
        fz = acc.get(f"C{c}_HW{hw}_bnff", {})
        ub = u.get("dram__bytes_read.sum", 0) + 32 * u.get("lts__t_sectors_op_write.sum", 0)
        fb = fz.get("dram__bytes_read.sum", 0) + 32 * fz.get("lts__t_sectors_op_write.sum", 0)
        t = times.get((c, hw), {})
        row = {"C": c, "HW": hw, "unfused_bytes": ub, "fused_bytes": fb,
               "reduction": (1 - fb / ub) if ub else None, **t}
        if t:
            row["fused_GBps"] = fb / (t["bnff_us"] * 1e-6) / 1e9
        out.append(row)
        T = 64 * c * hw * hw * 2 / 1e6
        print(f"{c:5d} {hw:4d} {T:8.1f} {ub / 1e9:11.3f} {fb / 1e9:9.3f} "
              f"{(1 - fb / ub) if ub else 0:6.3f} {t.get('baseline_us', 0):8.1f} {t.get('bnff_us', 0):8.1f} "
              f"{t.get('speedup', 0):7.3f} {row.get('fused_GBps', 0):10.0f}")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--ncu", action="store_true")
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--out", default="gpurun_out/c5_time.json")
    ap.add_argument("--summarize", nargs="*")
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    if a.summarize:
        res = summarize(a.summarize[0], a.summarize[1] if len(a.summarize) > 1 else None)
        if a.json:
            with open(a.json, "w") as f:
                json.dump(res, f, indent=1)
    elif a.ncu:
        run_ncu(a.n)
    else:
        run_time(a.n, a.out)


if __name__ == "__main__":
    main()
