"""One DenseNet-121 training step bracketed by cudaProfilerStart/Stop, for ncu byte counts.

    ncu --profile-from-start off --cache-control none \
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,gpu__time_duration.sum \
        --csv --log-file out.csv python tools/ncu_step_bytes.py --level bnff
    python tools/ncu_step_bytes.py --summarize out.csv [out2.csv ...]

With --cache-control none the sum of dram__bytes over every kernel of the step is the
step's real HBM traffic (write-backs land on whichever later kernel evicts them; the
step total is exact up to the <= 126 MB left dirty in L2).  lts__t_sectors_op_write
counts bytes written into L2 by each kernel (its algorithmic output traffic).
"""

from __future__ import annotations

import argparse
import csv
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONV_KERNELS = ("wconv_kernel", "wgrad_kernel", "igemm_kernel", "wg_reduce_kernel",
                "wgrad_reduce_kernel")


def run(level, dtype, batch):
    import torch
    from paper_1807_01702_b200 import fusion, graph as G
    from paper_1807_01702_b200.engine import Engine
    from paper_1807_01702_b200.tensor import Rng
    g, _ = fusion.plan(G.build_model(G.densenet121(batch), seed=0), fusion.parse_level(level))
    eng = Engine(g, dtype=dtype, input_grad=True, lr=1e-3)
    rng = Rng(1)
    eng.set_input(rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0))
    eng.set_loss_grad(rng.normal(g.slots[g.outputs[0]].shape))
    eng.capture()
    for _ in range(3):
        eng.step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    eng.step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()


def kernel_class(name: str) -> str:
    """ncu kernel name -> engine launch class (engine thunk `kind`)."""
    if "wgrad_kernel" in name or "wg_reduce_kernel" in name or "wgrad_reduce_kernel" in name \
            or "wgrad_f32_kernel" in name \
            or "igemm_kernel<2" in name or "igemm_kernel<(int)2" in name:
        return "wgrad"
    if "wconv_kernel" in name:  # template <BN, RB, TAPS, MODE[, SW]>: MODE 1 = dgrad
        args = name.split("<", 1)[1].split(">", 1)[0].split(",")
        return "dgrad" if args[3].strip().endswith("1") else "fprop"
    if "igemm_kernel<1" in name or "igemm_kernel<(int)1" in name:
        return "dgrad"
    if "igemm_kernel" in name:
        return "fprop"
    if "norm_relu_pool" in name:
        return "norm_relu_pool"
    if "pool_relu_bn_bwd" in name:
        return "pool_relu_bn_bwd"
    if "finalize_coeffs" in name:
        return "bn_coeffs"
    for k in ("stats_finalize", "dx_coeffs", "bn_coeffs", "im2col", "col2im", "avgpool", "grad_sum",
              "channel_sums", "sgd", "pack", "relu", "bn_apply"):
        if k in name:
            return k
    return "other"


def summarize(paths, json_out=""):
    out = {}
    classes = {}
    for path in paths:
        with open(path) as f:
            lines = [ln for ln in f if ln.startswith('"')]
        rd = csv.reader(lines)
        hdr = next(rd)
        ik, im, iv, iid = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                           hdr.index("Metric Value"), hdr.index("ID"))
        per = {}
        for r in rd:
            d = per.setdefault(r[iid], {"name": r[ik]})
            d[r[im]] = float(r[iv].replace(",", ""))
        tot = {"launches": len(per)}
        for cat in ("all", "conv", "other"):
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_op_write.sum",
                      "gpu__time_duration.sum"):
                tot[f"{cat}:{m}"] = 0.0
        cls = classes.setdefault(path, {})
        for d in per.values():
            c = cls.setdefault(kernel_class(d["name"]), {"launches": 0, "dram_bytes": 0.0, "ns": 0.0})
            c["launches"] += 1
            c["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
            c["ns"] += d.get("gpu__time_duration.sum", 0.0)
            cat = "conv" if any(k in d["name"] for k in CONV_KERNELS) else "other"
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_op_write.sum",
                      "gpu__time_duration.sum"):
                v = d.get(m, 0.0)
                tot[f"all:{m}"] += v
                tot[f"{cat}:{m}"] += v
        out[path] = tot
        gb = 1e-9
        print(f"== {path}: {tot['launches']} launches")
        for cat in ("all", "conv", "other"):
            rd_ = tot[f"{cat}:dram__bytes_read.sum"]
            wr_ = tot[f"{cat}:dram__bytes_write.sum"]
            l2w = tot[f"{cat}:lts__t_sectors_op_write.sum"] * 32
            t = tot[f"{cat}:gpu__time_duration.sum"] * 1e-6
            print(f"  {cat:5s} dram read {rd_ * gb:8.3f} GB  dram write {wr_ * gb:8.3f} GB  "
                  f"dram total {(rd_ + wr_) * gb:8.3f} GB  L2 writes {l2w * gb:8.3f} GB  "
                  f"kernel time {t:8.3f} ms")
    if json_out:
        import json
        with open(json_out, "w") as f:
            json.dump({"how": "ncu --profile-from-start off --cache-control none --clock-control none "
                              "--metrics dram__bytes_read.sum,dram__bytes_write.sum,... over one captured "
                              "D121 b64 step (tools/ncu_step_bytes.py)",
                       "runs": {os.path.basename(k): v for k, v in classes.items()},
                       "totals": {os.path.basename(k): v for k, v in out.items()}}, f, indent=1)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", default="bnff")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--summarize", nargs="*")
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    if a.summarize:
        summarize(a.summarize, a.json)
    else:
        run(a.level, a.dtype, a.batch)


if __name__ == "__main__":
    main()
