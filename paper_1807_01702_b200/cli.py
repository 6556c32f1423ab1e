"""`bnfuse bench` for the device path: the reference's bench command (``cli.py:160-224``)
with its frozen CSV schema (``BENCH_HEADER``, ``cli.py:109-110``) and flags
(``cli.py:294-317``), timing the CUDA-graph forward / backward of every requested fusion
level on the GPU, so the reference tooling (``read_bench_csv``) reads GPU runs unchanged.
Device additions: ``--dtype`` (bf16 | f32), ``--gpus`` (informational; one process per GPU
is bench.py's job) and ``--syncbn``.

    python -m paper_1807_01702_b200.cli bench --model densenet-121 --batch 64 --fusion all
    python -m paper_1807_01702_b200.cli traffic --model densenet-121 --batch 64 --out report/
    python -m paper_1807_01702_b200.cli explain --model densenet-121 --fusion bnff+icf

Columns follow the reference; ``traffic_bytes`` is the algorithmic HBM bytes of the launches
of that pass (each tensor counted once per launch, in the storage dtype) rather than the
reference's fp32 sweep rulebook, ``threads`` is the GPU count, ``conv_share`` the share of
device time in conv launches measured by per-launch events.  ``checksum`` follows the
reference contract (one value for every level of a run, test_cli.py:89-90): a digest of the
run's shared inputs and initial weights; the device outputs of every level are compared
with the baseline level's and the relative L2 gap is printed.

``traffic`` / ``explain`` mirror ``bnfuse traffic`` / ``explain`` (cli.py:247-286): the
reference's sweep rulebook (traffic.py) per level, one CSV per level plus summary.json, and
the rewrite plan of each level.
"""

from __future__ import annotations

import argparse
import csv
import hashlib
import statistics
import sys

from . import fusion
from . import graph as G

# the reference's frozen bench schema (bnfuse/cli.py:109-110)
BENCH_HEADER = ["level", "pass", "median_ms", "mean_ms", "std_ms", "iters",
                "speedup_vs_baseline", "conv_share", "traffic_bytes", "checksum", "threads"]

_CONV_KINDS = ("fprop", "dgrad", "wgrad", "im2col", "cols_to_weight")


def _levels(token: str):
    if token in (None, "all"):
        return list(fusion.FusionLevel)
    return [fusion.parse_level(t) for t in token.split(",")]


def _time_graph(fn, iters, warmup):
    import torch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    for _ in range(warmup):
        gr.replay()
    torch.cuda.synchronize()
    out = []
    cur = torch.cuda.current_stream()
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        gr.replay()
        e1.record(cur)
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return out


def cmd_bench(a) -> int:
    import numpy as np
    import torch
    from .engine import Engine
    from .tensor import Rng

    presets = dict(G.PRESETS, **{"densenet-bc-100": G.densenet_bc100})
    spec = presets[a.model]() if a.batch is None else presets[a.model](a.batch)
    base = G.build_model(spec, seed=a.seed)
    if a.model.startswith("densenet") and spec.growth_rate % 8:
        base, _ = G.pad_channels(base, 8)
    rng = Rng(a.seed + 1)
    x = rng.uniform(base.slots[base.inputs[0]].shape, -1.0, 1.0)
    dy = rng.normal(base.slots[base.outputs[0]].shape)
    rows, baseline_total, ref_out = [], None, None
    h = hashlib.sha1(np.ascontiguousarray(x).tobytes())
    for k in sorted(base.params):
        h.update(np.ascontiguousarray(base.params[k]).tobytes())
    checksum = h.hexdigest()[:12]
    for level in _levels(a.fusion):
        g2, _ = fusion.plan(base, level)
        try:
            eng = Engine(g2, dtype=a.dtype, input_grad=False, sync_bn=a.syncbn)
        except Exception as e:  # e.g. two-pass statistics under SyncBN
            print(f"{level.token}: skipped ({e})", file=sys.stderr)
            continue
        eng.set_input(x)
        eng.set_loss_grad(dy)
        eng.forward()
        eng.backward()
        torch.cuda.synchronize()
        fwd = _time_graph(eng.forward, a.iterations, a.warmup)
        bwd = _time_graph(eng.backward, a.iterations, a.warmup)
        prof = eng.profile_launches(reps=1)
        conv = sum(ms for t, ms in prof if t.kind in _CONV_KINDS)
        allms = sum(ms for _, ms in prof) or 1.0
        out = eng.output()
        if ref_out is None:
            ref_out = out
        gap = float(np.linalg.norm(out - ref_out) / max(float(np.linalg.norm(ref_out)), 1e-30))
        print(f"{level.token:10s} output rel-L2 vs first level {gap:.2e}")
        traffic = {"forward": sum(t.nbytes for t in eng.fwd), "backward": sum(t.nbytes for t in eng.bwd)}
        total = [f + b for f, b in zip(fwd, bwd)]
        if level == fusion.FusionLevel.BASELINE:
            baseline_total = statistics.median(total)
        for pass_, series in (("forward", fwd), ("backward", bwd), ("total", total)):
            med = statistics.median(series)
            rows.append({
                "level": level.token, "pass": pass_,
                "median_ms": f"{med:.3f}", "mean_ms": f"{statistics.mean(series):.3f}",
                "std_ms": f"{statistics.pstdev(series):.3f}", "iters": a.iterations,
                "speedup_vs_baseline": (f"{baseline_total / med:.3f}"
                                        if pass_ == "total" and baseline_total else ""),
                "conv_share": f"{conv / allms:.3f}",
                "traffic_bytes": traffic.get(pass_, traffic["forward"] + traffic["backward"]),
                "checksum": checksum, "threads": a.gpus,
            })
        del eng
        torch.cuda.empty_cache()
    path = a.out_path or "bench.csv"
    with open(path, "w", newline="") as f:
        wr = csv.DictWriter(f, fieldnames=BENCH_HEADER)
        wr.writeheader()
        wr.writerows(rows)
    for r in rows:
        if r["pass"] == "total":
            print(f"{r['level']:10s} total {r['median_ms']:>9s} ms  "
                  f"speedup {r['speedup_vs_baseline'] or '-':>6s}  checksum {r['checksum']}")
    print(f"wrote {path}")
    return 0


def _spec(a):
    presets = dict(G.PRESETS, **{"densenet-bc-100": G.densenet_bc100})
    return presets[a.model]() if a.batch is None else presets[a.model](a.batch)


def cmd_traffic(a) -> int:
    import json
    import os
    from . import traffic
    base = G.build_model(_spec(a), seed=a.seed)
    out_dir = a.out_path or "traffic-report"
    os.makedirs(out_dir, exist_ok=True)
    leds = {}
    for level in _levels(a.fusion):
        g2, _ = fusion.plan(base, level)
        led = traffic.count_sweeps(g2, concat_physical=False, bytes_per_elem=a.bytes_per_elem)
        leds[level.token] = led
        with open(os.path.join(out_dir, f"traffic_{level.token.replace('+', '_')}.csv"), "w") as f:
            f.write(traffic.to_csv(led))
    first = leds.get("baseline") or next(iter(leds.values()))
    summary = []
    for tok, led in leds.items():
        s = traffic.summary(led, tok, base.meta.get("spec").name if base.meta.get("spec") else a.model, first)
        summary.append(s)
        print(f"{tok:10s} total {led.total_bytes() / 1e9:9.3f} GB  reduction "
              f"{s['reduction_vs_baseline'] * 100:6.2f}%  relu share {s['relu_share'] * 100:5.2f}%")
    with open(os.path.join(out_dir, "summary.json"), "w") as f:
        json.dump(summary, f, indent=2)
    print(f"wrote {out_dir}/")
    return 0


def cmd_explain(a) -> int:
    base = G.build_model(_spec(a), seed=a.seed)
    for level in _levels(a.fusion):
        _, fplan = fusion.plan(base, level)
        print(fplan.describe())
        print()
    return 0


def make_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="bnfuse-b200", description="restructured-BN training path on B200")
    sub = p.add_subparsers(dest="command", required=True)
    sp = sub.add_parser("bench", help="device-timed training iterations per fusion level")
    sp.add_argument("--model", default="densenet-121",
                    help=f"preset: {', '.join(sorted(G.PRESETS))}, densenet-bc-100")
    sp.add_argument("--batch", type=int, default=None)
    sp.add_argument("--fusion", default="baseline,bnff,bnff+icf",
                    help="baseline, rcf, rcf+mvf, bnff, bnff+icf, a comma list, or all")
    sp.add_argument("--iters", type=int, default=10, dest="iterations")
    sp.add_argument("--warmup", type=int, default=3)
    sp.add_argument("--seed", type=int, default=0)
    sp.add_argument("--out", default=None, dest="out_path")
    sp.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    sp.add_argument("--gpus", type=int, default=1)
    sp.add_argument("--syncbn", action="store_true")
    for name, help_ in (("traffic", "the reference's memory-sweep rulebook per fusion level"),
                        ("explain", "the rewrite plan of each fusion level")):
        tp = sub.add_parser(name, help=help_)
        tp.add_argument("--model", default="densenet-121")
        tp.add_argument("--batch", type=int, default=None)
        tp.add_argument("--fusion", default="all")
        tp.add_argument("--seed", type=int, default=0)
        tp.add_argument("--out", default=None, dest="out_path")
        tp.add_argument("--bytes-per-elem", type=int, default=4, help="4 = the reference's fp32; 2 = bf16 storage")
    return p


def main(argv=None) -> int:
    a = make_parser().parse_args(argv)
    return {"bench": cmd_bench, "traffic": cmd_traffic, "explain": cmd_explain}[a.command](a)


if __name__ == "__main__":
    sys.exit(main())
