"""Standalone HBM throughput of the memory-bound kernels (K5 channel sums, K6
bn_apply, K7/K8 grad_sum / deferred BN dx, ReLU) on DenseNet-121 block-1-sized tensors
(N=64, 56x56, C in {64, 128, 256}) in bf16 and fp32: algorithmic bytes (each tensor once)
/ CUDA-event time, median of 20 after 5 warm-ups, against MEASURED_PEAKS.json's HBM figure.

    python tools/kernel_bw.py [--json out.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, reps=20, warm=5):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    import numpy as np
    import torch
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6650.0
    import ctypes as C
    from paper_1807_01702_b200 import _lib
    from paper_1807_01702_b200.kernels import coef, view
    L = _lib.lib()
    stream = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
    rows = []
    for dt in (torch.bfloat16, torch.float32):
        code = _lib.BF16 if dt == torch.bfloat16 else _lib.F32
        for c in (64, 128, 256):
            n, hw = 64, 56
            x = torch.randn((n, hw, hw, c), device="cuda").to(dt)
            dy = torch.randn((n, hw, hw, c), device="cuda").to(dt)
            out = torch.empty_like(x)
            f32 = lambda: torch.rand(c, device="cuda") + 0.5  # noqa: E731
            m, s_, b_, inv, k1, k2, g = (f32() for _ in range(7))
            tiles = L.bnff_sum_tiles(n * hw * hw)
            part = torch.zeros((tiles, 2, c), dtype=torch.float64, device="cuda")
            nb = x.numel() * x.element_size()
            t_dx = (_lib.GradTerm * 1)(_lib.GradTerm(view(dy), view(x), 1, coef(m, inv, k1, k2, g)))
            t_sp = (_lib.GradTerm * 2)(_lib.GradTerm(view(x), view(x), 0, coef()),
                                       _lib.GradTerm(view(dy), view(dy), 0, coef()))
            cases = {  # raw C-ABI launches on preallocated buffers (one kernel each)
                "K5 channel_sums (x, x^2)": (lambda: L.bnff_channel_sums(code, 0, view(x), view(x), coef(), part.data_ptr(), stream()), nb),
                "K5b bn bwd sums (dy, dy*xhat)": (lambda: L.bnff_channel_sums(code, 1, view(x), view(dy), coef(m, inv), part.data_ptr(), stream()), 2 * nb),
                "K6 bn_apply (+ReLU)": (lambda: L.bnff_bn_apply(code, view(x), view(out), coef(m, s_, b_), 1, stream()), 2 * nb),
                "K7 deferred BN dx": (lambda: L.bnff_grad_sum(code, view(out), 0, t_dx, 1, stream()), 3 * nb),
                "K8 split sum (2 branches)": (lambda: L.bnff_grad_sum(code, view(out), 0, t_sp, 2, stream()), 3 * nb),
                "relu_bwd": (lambda: L.bnff_relu_bwd(code, view(x), view(dy), view(out), stream()), 3 * nb),
            }
            for name, (fn, b) in cases.items():
                ms = timeit(fn)
                gbs = b / (ms * 1e-3) / 1e9
                rows.append({"kernel": name, "dtype": str(dt).split(".")[-1], "C": c, "bytes": b, "ms": ms,
                             "GB/s": round(gbs, 1), "frac": round(gbs / peak, 3)})
                print(f"{name:30s} {rows[-1]['dtype']:9s} C={c:4d} {b / 1e6:8.1f} MB {ms * 1e3:8.1f} us "
                      f"{gbs:7.0f} GB/s  {gbs / peak:.2f} of {peak:.0f}", flush=True)
    if a.json:
        json.dump({"peak_gbs": peak, "rows": rows}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
