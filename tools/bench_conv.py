"""Kernel-level check + timing of the window-shift conv kernels against the generic
implicit-GEMM kernels (same bf16 math), on DenseNet-121 shapes.

    python tools/bench_conv.py [--quick]

Prints, per case: rel-L2 difference window vs generic (outputs, stats), and the
device time of each (CUDA events, median of reps).  Not a bench number.
"""

from __future__ import annotations

import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1807_01702_b200 import _lib  # noqa: E402
from paper_1807_01702_b200 import kernels as K  # noqa: E402
from paper_1807_01702_b200.params import ConvParams  # noqa: E402


def rel(a, b):
    a = a.float()
    b = b.float()
    return float((a - b).norm() / max(float(b.norm()), 1e-30))


def timeit(fn, reps=10):
    """Device time per call: fn captured once into a CUDA graph, replayed `reps` times
    between two events (host launch overhead excluded)."""
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    gr.replay()
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for _ in range(reps):
        gr.replay()
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def tables(c, dev, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    mean = (torch.rand(c, generator=g) * 0.4 - 0.2).to(dev)
    scale = (torch.rand(c, generator=g) * 0.5 + 0.75).to(dev)
    beta = (torch.rand(c, generator=g) * 0.4 - 0.2).to(dev)
    inv = (torch.rand(c, generator=g) * 0.5 + 0.75).to(dev)
    k1 = (torch.rand(c, generator=g) * 0.02 - 0.01).to(dev)
    k2 = (torch.rand(c, generator=g) * 0.02 - 0.01).to(dev)
    return mean, scale, beta, inv, k1, k2


def case(n, hw, cin, cout, k, mode, pro, epi, reps):
    dev = "cuda"
    torch.manual_seed(0)
    p = ConvParams(in_c=cin, out_c=cout, kh=k, kw=k, weights=(np.random.RandomState(1).uniform(-1, 1, (cout, cin, k, k)) /
                            np.sqrt(cin * k * k)).astype(np.float32),
                   bias=np.random.RandomState(2).uniform(-0.1, 0.1, cout).astype(np.float32),
                   stride=1, pad=k // 2, name=f"c{k}")
    pw = K.PackedConv(p, torch.bfloat16, dev, window=True)
    pg = K.PackedConv(p, torch.bfloat16, dev, window=False)
    L = _lib.lib()
    res = {}
    if mode == "wgrad":
        x = torch.randn(n, hw, hw, cin, device=dev).to(torch.bfloat16)
        dy = torch.randn(n, hw, hw, cout, device=dev).to(torch.bfloat16)
        dyx = torch.randn(n, hw, hw, cout, device=dev).to(torch.bfloat16)
        xm, xs, xb, _, _, _ = tables(cin, dev, 6)
        m, s_, b, inv, k1, k2 = tables(cout, dev, 7)
        xc = K.coef(xm, xs, xb) if pro in (_lib.PRO_BN_RELU,) else K.coef()
        dpro = _lib.PRO_BN_DX if epi else _lib.PRO_NONE
        dc = K.coef(m, inv, k1, k2, s_) if dpro == _lib.PRO_BN_DX else K.coef()
        ws_n = L.bnff_wgrad_workspace(n, hw, hw, k, k, cin, cout, 0)
        outs = {}
        for nm, sp in (("win", 0), ("gen", -1)):
            ws = torch.empty(ws_n, dtype=torch.float32, device=dev)
            dw = torch.zeros((cout, cin, k, k), dtype=torch.float32, device=dev)
            db = torch.zeros(cout, dtype=torch.float32, device=dev)
            a = _lib.WgradArgs(_lib.BF16, k, k, 1, k // 2, K.view(x), pro, xc, K.view(dy), K.view(dyx),
                               dpro, dc, sp, K._ptr(ws), K._ptr(dw), cin, K._ptr(db))

            def run(a=a):
                _lib.check(L.bnff_conv_wgrad(ctypes.byref(a), K._stream()), "wgrad")
            t = timeit(run, reps)
            outs[nm] = (dw.clone(), db.clone(), t)
        res["out"] = rel(outs["win"][0], outs["gen"][0])
        res["stats"] = rel(outs["win"][1], outs["gen"][1])
        res["t_win"], res["t_gen"] = outs["win"][2], outs["gen"][2]
        res["nbytes"] = (x.numel() + dy.numel() * (2 if dpro else 1)) * 2
    elif mode == "fprop":
        x = torch.randn(n, hw, hw, cin, device=dev).to(torch.bfloat16)
        m, s, b, inv, _, _ = tables(cin, dev, 3)
        tb = (m, s, b) if pro == _lib.PRO_BN_RELU else None
        outs = {}
        for nm, pc in (("win", pw), ("gen", pg)):
            y = torch.empty(n, hw, hw, cout, device=dev, dtype=torch.bfloat16)
            part = torch.zeros((L.bnff_stat_rows(), 2, cout), dtype=torch.float64, device=dev)

            def run(pc=pc, y=y, part=part):
                K._fprop(x, pc, y, pro, tb, part)
            t = timeit(run, reps)
            outs[nm] = (y.clone(), part.sum(0).clone(), t)
        res["out"] = rel(outs["win"][0], outs["gen"][0])
        res["stats"] = rel(outs["win"][1], outs["gen"][1])
        res["t_win"], res["t_gen"] = outs["win"][2], outs["gen"][2]
        nbytes = (x.numel() + n * hw * hw * cout) * 2
    else:
        dy = torch.randn(n, hw, hw, cout, device=dev).to(torch.bfloat16)
        dyx = torch.randn(n, hw, hw, cout, device=dev).to(torch.bfloat16)
        x = torch.randn(n, hw, hw, cin, device=dev).to(torch.bfloat16)
        m, s, b, inv, k1, k2 = tables(cout, dev, 4)
        em, es, eb, einv, _, _ = tables(cin, dev, 5)
        g = s
        pkg = (dy, dyx, (m, inv, k1, k2, g)) if pro == _lib.PRO_BN_DX else None
        outs = {}
        for nm, pc in (("win", pw), ("gen", pg)):
            part = torch.zeros((L.bnff_stat_rows(), 2, cin), dtype=torch.float64, device=dev)
            holder = {}

            def run(pc=pc, part=part, holder=holder):
                holder["dx"] = K._dgrad(dy, pc, x, epi, x, (em, es, eb, einv), part, pkg)
            t = timeit(run, reps)
            outs[nm] = (holder["dx"].clone(), part.sum(0).clone(), t)
        res["out"] = rel(outs["win"][0], outs["gen"][0])
        res["stats"] = rel(outs["win"][1], outs["gen"][1]) if epi == _lib.DG_NRC else 0.0
        res["t_win"], res["t_gen"] = outs["win"][2], outs["gen"][2]
        nbytes = (dy.numel() * (2 if pkg else 1) + x.numel() * (2 if epi else 1)) * 2
    flops = 2 * n * hw * hw * cin * cout * k * k
    if mode == "wgrad":
        nbytes = res.pop("nbytes")
    print(f"{mode:5s} n{n} {hw:3d}^2 {cin:4d}->{cout:4d} k{k} pro{pro} epi{epi}: "
          f"out {res['out']:.2e} stats {res['stats']:.2e} | win {res['t_win']:8.1f} us "
          f"({nbytes / res['t_win'] / 1e3:6.0f} GB/s, {flops / res['t_win'] / 1e6:6.1f} TF/s) "
          f"gen {res['t_gen']:8.1f} us", flush=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--only", default="", help="comma-separated case indices")
    a = ap.parse_args()
    P = _lib
    cases = [
        # small correctness cases (odd sizes, partial tiles)
        (2, 9, 64, 32, 3, "fprop", P.PRO_BN_RELU, 0),
        (2, 9, 96, 128, 1, "fprop", P.PRO_BN_RELU, 0),
        (2, 9, 32, 128, 3, "dgrad", P.PRO_BN_DX, P.DG_NRC),
        (2, 9, 128, 32, 3, "dgrad", P.PRO_BN_DX, P.DG_NRC),
        (3, 5, 128, 32, 3, "dgrad", P.PRO_NONE, P.DG_CLIP),
        (3, 5, 64, 64, 3, "fprop", P.PRO_RELU, 0),
        (2, 9, 96, 128, 1, "dgrad", P.PRO_BN_DX, P.DG_NRC),
        (2, 7, 128, 32, 3, "fprop", P.PRO_NONE, 0),
        (2, 7, 160, 128, 1, "dgrad", P.PRO_NONE, P.DG_PLAIN),
        (2, 7, 256, 128, 1, "fprop", P.PRO_RELU, 0),
        (2, 8, 512, 256, 1, "fprop", P.PRO_BN_RELU, 0),
        (2, 8, 320, 128, 1, "dgrad", P.PRO_BN_DX, P.DG_NRC),
    ]
    cases += [
        # TMA window tiling: kt rows per tile with a partial last tile (14: kt=8),
        # a BN_DX x operand on a 3x3 with row tiles, uneven slabs, ragged pixel counts
        (2, 14, 64, 32, 3, "fprop", P.PRO_BN_RELU, 0),
        (2, 12, 32, 64, 3, "dgrad", P.PRO_BN_DX, P.DG_NRC),
        (3, 11, 96, 128, 1, "dgrad", P.PRO_BN_DX, P.DG_NRC),
        (1, 30, 64, 32, 3, "fprop", P.PRO_RELU, 0),
        # 3x3 with streamed weights (ResNet widths: 9 taps of each slab ride with the stage)
        (2, 14, 256, 256, 3, "fprop", P.PRO_BN_RELU, 0),
        (2, 12, 128, 128, 3, "dgrad", P.PRO_BN_DX, P.DG_NRC),
        (3, 7, 512, 512, 3, "dgrad", P.PRO_NONE, P.DG_CLIP),
        (2, 14, 256, 256, 3, "wgrad", P.PRO_BN_RELU, 1),
    ]
    cases += [
        (2, 9, 128, 32, 3, "wgrad", P.PRO_BN_RELU, 0),
        (2, 16, 160, 16, 1, "wgrad", P.PRO_NONE, 1),
        (2, 9, 96, 128, 1, "wgrad", P.PRO_BN_RELU, 1),
        (3, 6, 320, 128, 1, "wgrad", P.PRO_NONE, 1),
        (2, 5, 64, 64, 3, "wgrad", P.PRO_RELU, 0),
        (2, 4, 512, 256, 1, "wgrad", P.PRO_BN_RELU, 0),
    ]
    if not a.quick:
        cases += [
            (64, 56, 128, 32, 3, "fprop", P.PRO_BN_RELU, 0),
            (64, 56, 128, 32, 3, "dgrad", P.PRO_NONE, P.DG_NRC),
            (64, 56, 128, 128, 1, "fprop", P.PRO_BN_RELU, 0),
            (64, 56, 224, 128, 1, "dgrad", P.PRO_BN_DX, P.DG_NRC),
            (64, 28, 128, 32, 3, "fprop", P.PRO_BN_RELU, 0),
            (64, 28, 480, 128, 1, "fprop", P.PRO_BN_RELU, 0),
            (64, 14, 128, 32, 3, "fprop", P.PRO_BN_RELU, 0),
            (64, 14, 992, 128, 1, "dgrad", P.PRO_BN_DX, P.DG_NRC),
            (64, 7, 128, 32, 3, "dgrad", P.PRO_NONE, P.DG_NRC),
            (64, 56, 256, 128, 1, "fprop", P.PRO_BN_RELU, 0),
            (64, 56, 128, 32, 3, "wgrad", P.PRO_BN_RELU, 0),
            (64, 56, 224, 128, 1, "wgrad", P.PRO_BN_RELU, 1),
            (64, 28, 128, 32, 3, "wgrad", P.PRO_BN_RELU, 0),
            (64, 14, 992, 128, 1, "wgrad", P.PRO_BN_RELU, 1),
            (64, 7, 128, 32, 3, "wgrad", P.PRO_BN_RELU, 0),
        ]
    worst = 0.0
    if a.only:
        cases = [cases[int(i)] for i in a.only.split(",")]
    for c in cases:
        r = case(*c, reps=a.reps)
        worst = max(worst, r["out"], r["stats"])
    print(f"worst rel-L2 window vs generic: {worst:.3e}")


if __name__ == "__main__":
    main()
