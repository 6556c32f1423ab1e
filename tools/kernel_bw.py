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
    from paper_1807_01702_b200 import kernels as K
    from paper_1807_01702_b200.params import BNParams
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6650.0
    rows = []
    for dt in (torch.bfloat16, torch.float32):
        for c in (64, 128, 256):
            n, hw = 64, 56
            x = torch.randn((n, hw, hw, c), device="cuda").to(dt)
            dy = torch.randn((n, hw, hw, c), device="cuda").to(dt)
            bn = BNParams(np.ones(c, np.float32), np.zeros(c, np.float32))
            st = K.bn_stats_onepass(x)
            nb = x.numel() * x.element_size()
            cases = {
                "K5 channel_sums (x, x^2)": (lambda: K.bn_stats_onepass(x), nb),
                "K6 bn_apply (+ReLU)": (lambda: K.bn_fwd(x, st, bn, relu=True), 2 * nb),
                "K7 deferred BN dx": (lambda: K.bn_dx_from_sums(x, dy, st, bn, np.ones(c), np.ones(c)), 3 * nb),
                "K8 split sum (2 branches)": (lambda: K.fused_split_bwd_bn_dx([x, dy]), 3 * nb),
                "relu_bwd": (lambda: K.relu_bwd(x, dy), 3 * nb),
            }
            for name, (fn, b) in cases.items():
                ms = timeit(fn)
                gbs = b / (ms * 1e-3) / 1e9
                rows.append({"kernel": name, "dtype": str(dt).split(".")[-1], "C": c, "bytes": b, "ms": ms,
                             "GB/s": round(gbs, 1), "frac": round(gbs / peak, 3)})
                print(f"{name:28s} {rows[-1]['dtype']:9s} C={c:4d} {b / 1e6:8.1f} MB {ms * 1e3:8.1f} us "
                      f"{gbs:7.0f} GB/s  {gbs / peak:.2f} of {peak:.0f}", flush=True)
    if a.json:
        json.dump({"peak_gbs": peak, "rows": rows}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
