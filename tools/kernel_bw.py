"""Standalone HBM throughput of the memory-bound kernels (K5 channel sums, K6
bn_apply, K7/K8 grad_sum / deferred BN dx, ReLU) on DenseNet-121 block-1-sized tensors
(N=64, 56x56, C in {64, 128, 256}) in bf16 and fp32: algorithmic bytes (each tensor once)
/ device time, against MEASURED_PEAKS.json's HBM figure.  Timing: the C-ABI arguments are
built once, and 24 back-to-back launches rotate over enough distinct buffer sets (>= 512 MB
in total) that no launch finds its inputs in the 126 MB L2; one CUDA-event pair brackets the
24 launches (GPU-bound queue: no host gap between kernels), median of 5 such runs.

    python tools/kernel_bw.py [--json out.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fns, reps=5, per=24):
    """fns: launch closures over distinct buffer sets; median over reps of (time of `per`
    back-to-back launches cycling through fns) / per"""
    import torch
    for f in fns:
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(per):
            fns[i % len(fns)]()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / per)
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
    rows = []
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for dt in (torch.bfloat16, torch.float32):
        code = _lib.BF16 if dt == torch.bfloat16 else _lib.F32
        for c in (64, 128, 256):
            n, hw = 64, 56
            nb = n * hw * hw * c * torch.empty((), dtype=dt).element_size()
            nsets = max(2, -(-512 * 2**20 // (3 * nb)))
            f32 = lambda: torch.rand(c, device="cuda") + 0.5  # noqa: E731
            m, s_, b_, inv, k1, k2, g = (f32() for _ in range(7))
            tiles = L.bnff_sum_tiles(n * hw * hw)
            keep, cases = [], {}
            for _ in range(nsets):
                x = torch.randn((n, hw, hw, c), device="cuda").to(dt)
                dy = torch.randn((n, hw, hw, c), device="cuda").to(dt)
                out = torch.empty_like(x)
                part = torch.zeros((tiles, 2, c), dtype=torch.float64, device="cuda")
                t_dx = (_lib.GradTerm * 1)(_lib.GradTerm(view(dy), view(x), 1, coef(m, inv, k1, k2, g)))
                t_sp = (_lib.GradTerm * 2)(_lib.GradTerm(view(x), view(x), 0, coef()),
                                           _lib.GradTerm(view(dy), view(dy), 0, coef()))
                vx, vdy, vo = view(x), view(dy), view(out)
                c0, cmi, cms = coef(), coef(m, inv), coef(m, s_, b_)
                keep += [x, dy, out, part, t_dx, t_sp]
                pp = part.data_ptr()
                for name, fn, b in (  # raw C-ABI launches, arguments prebuilt (one kernel each)
                        ("K5 channel_sums (x, x^2)",
                         lambda vx=vx, pp=pp: L.bnff_channel_sums(code, 0, vx, vx, c0, pp, st), nb),
                        ("K5b bn bwd sums (dy, dy*xhat)",
                         lambda vx=vx, vdy=vdy, pp=pp: L.bnff_channel_sums(code, 1, vx, vdy, cmi, pp, st), 2 * nb),
                        ("K6 bn_apply (+ReLU)", lambda vx=vx, vo=vo: L.bnff_bn_apply(code, vx, vo, cms, 1, st), 2 * nb),
                        ("K7 deferred BN dx", lambda vo=vo, t=t_dx: L.bnff_grad_sum(code, vo, 0, t, 1, st), 3 * nb),
                        ("K8 split sum (2 branches)", lambda vo=vo, t=t_sp: L.bnff_grad_sum(code, vo, 0, t, 2, st),
                         3 * nb),
                        ("relu_bwd", lambda vx=vx, vdy=vdy, vo=vo: L.bnff_relu_bwd(code, vx, vdy, vo, st), 3 * nb)):
                    cases.setdefault(name, ([], b))[0].append(fn)
            for name, (fns, b) in cases.items():
                ms = timeit(fns)
                gbs = b / (ms * 1e-3) / 1e9
                rows.append({"kernel": name, "dtype": str(dt).split(".")[-1], "C": c, "bytes": b, "ms": ms,
                             "GB/s": round(gbs, 1), "frac": round(gbs / peak, 3)})
                print(f"{name:30s} {rows[-1]['dtype']:9s} C={c:4d} {b / 1e6:8.1f} MB {ms * 1e3:8.1f} us "
                      f"{gbs:7.0f} GB/s  {gbs / peak:.2f} of {peak:.0f}", flush=True)
            del keep, cases
            torch.cuda.empty_cache()
    if a.json:
        json.dump({"peak_gbs": peak, "rows": rows}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
