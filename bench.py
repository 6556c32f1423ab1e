"""DenseNet-121 (224x224, batch 64/GPU) training throughput with the restructured
(BN fission-n-fusion) path on B200 -- the BASELINE.json headline metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU)

A step = forward + backward + SGD over one synthetic batch (x ~ U(-1,1), output
gradient ~ N(0,1), He-uniform weights, seed 0 -- the reference's generators),
replayed as one CUDA graph of libbnff kernels.  `value` is device-timed (CUDA
events on the launching stream, barrier + synchronize on both sides, max over
ranks) with inputs resident in HBM; `e2e` times the same step through the
public API with the batch copied host->device from pinned memory and the result
copied back every step.  Rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

_NCPU = len(os.sched_getaffinity(0))
os.environ.setdefault("OPENBLAS_NUM_THREADS", str(_NCPU))
os.environ.setdefault("OMP_NUM_THREADS", str(_NCPU))

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DenseNet-121 train images/sec at 1/2/4/8 B200; BN HBM bytes/iter vs unfused"
WORKLOAD = "densenet-121 224x224 fwd+bwd+SGD, batch 64 per GPU (BASELINE config C3)"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), float(pk["bf16_tflops"]), float(pk.get("bf16_tflops_sustained", pk["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3:]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[3][1:5])
                          if v.lower() == "active"})
        loaded = [r for r in rows if r[2] > 200.0] or rows
        return {"sm_mhz": float(np.median([r[0] for r in loaded])), "sm_max_mhz": rows[0][1],
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(r[2] for r in rows)}


# ---------------------------------------------------------------------------
# CPU oracle (reference algorithm restated in numpy) -- baseline / reference arm
# ---------------------------------------------------------------------------
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _reference_modules():
    """The unmodified reference package (installed into baseline/_ref, which travels to
    the GPU box), or None when it is absent -- then the numpy oracle port stands in."""
    if not os.path.isdir(os.path.join(REF_DIR, "bnfuse")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        from bnfuse import execute, fusion, graph, tensor  # noqa: F401
        return execute, fusion, graph, tensor
    except Exception:
        return None


def cpu_rate(batch: int, iters: int, warmup: int, level: str):
    """DenseNet-121 fwd+bwd on the host cores: the reference itself (`bnfuse` from
    baseline/_ref, ExecCtx with a 64 MiB tile budget -- SURVEY 8d) when installed, else
    the oracle port.  Returns (img/s, per-iteration seconds, kind)."""
    mods = _reference_modules()
    times = []
    if mods is not None:
        execute, fusion, graph, tensor = mods
        g, _ = fusion.plan(graph.build_model(graph.densenet121(batch), seed=0), fusion.parse_level(level))
        rng = tensor.Rng(1)
        x = rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0)
        loss = {s: rng.normal(g.slots[s].shape) for s in g.outputs}
        for i in range(warmup + iters):
            ctx = execute.ExecCtx(budget=64 << 20, workers=1)
            t0 = time.perf_counter()
            acts = execute.forward(g, x, ctx=ctx)
            execute.backward(g, acts, loss, ctx=ctx)
            if i >= warmup:
                times.append(time.perf_counter() - t0)
        kind = "reference"
    else:
        from oracle import executor as OX
        from paper_1807_01702_b200 import fusion, graph as G
        from paper_1807_01702_b200.tensor import Rng
        g, _ = fusion.plan(G.build_model(G.densenet121(batch), seed=0), fusion.parse_level(level))
        rng = Rng(1)
        x = rng.uniform(g.slots[g.inputs[0]].shape, -1.0, 1.0)
        dy = rng.normal(g.slots[g.outputs[0]].shape)
        for i in range(warmup + iters):
            t0 = time.perf_counter()
            OX.train_step(g, x, dy)
            if i >= warmup:
                times.append(time.perf_counter() - t0)
        kind = "port"
    return batch / float(np.median(times)), times, kind


def cpu_baseline(batch: int, iters: int, warmup: int, levels=("baseline", "bnff")):
    """b4, median of >= 3 iterations after a warmup, at baseline and bnff."""
    per = {}
    kind = None
    for lv in levels:
        rate, times, kind = cpu_rate(batch, iters, warmup, lv)
        per[lv] = {"value": rate, "ms_per_iter_median": 1e3 * float(np.median(times))}
    best = max(per, key=lambda k: per[k]["value"])
    src = "bnfuse (the reference, baseline/_ref) execute.forward/backward, ExecCtx(budget=64 MiB)" \
        if kind == "reference" else "numpy oracle port of bnfuse execute/fused/ops"
    return {"value": per[best]["value"], "unit": "images/s", "cores": _NCPU, "kind": kind,
            "level": best, "per_level": per,
            "sample": f"densenet-121 batch {batch} fwd+bwd, median of {iters} iterations after "
                      f"{warmup} warmup, levels {list(levels)} (value = the faster level); {src}; "
                      f"OpenBLAS threads = {os.environ.get('OPENBLAS_NUM_THREADS')}"}


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    batch = args.ref_batch
    rate, times, kind = cpu_rate(batch, args.steps, args.warmup, args.level)
    line = {
        "metric": METRIC, "value": rate, "unit": "images/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.median(times)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (x~U(-1,1), dy~N(0,1), He-uniform weights, seed 0)",
        "config": {"workload": WORKLOAD + f"; CPU sample batch {batch}", "level": args.level},
        "impl": "reference",
        "cpu_baseline": {"value": rate, "unit": "images/s", "cores": _NCPU, "kind": kind,
                         "sample": f"densenet-121 batch {batch} fwd+bwd at {args.level}, "
                                   f"{args.steps} timed iterations after {args.warmup} warmup "
                                   + ("(bnfuse from baseline/_ref, ExecCtx budget 64 MiB)"
                                      if kind == "reference" else
                                      "(numpy oracle restating bnfuse execute/fused/ops)")},
        "e2e": {"value": rate, "unit": "images/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def build_engine(level, dtype, batch, lr, world, sync_bn=False):
    from paper_1807_01702_b200 import fusion, graph as G
    from paper_1807_01702_b200.engine import Engine
    g, _ = fusion.plan(G.build_model(G.densenet121(batch), seed=0), fusion.parse_level(level))
    # input_grad: the stem's input gradient too, so both arms do the reference's full backward
    eng = Engine(g, dtype=dtype, input_grad=True, lr=lr / world, sync_bn=sync_bn)
    eng.level_name = level
    return g, eng


def timed_steps(trainer, steps, warmup, dist_on):
    import torch
    import torch.distributed as dist
    for _ in range(warmup):
        trainer.step()
    torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
    stream = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        trainer.step()
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    if dist_on:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    return ms


def tensor_peak(dtype, tf_sust):
    """Tensor-pipe ceiling for ALGORITHMIC conv FLOPs (2*M*N*K) timed inside the step:
    bf16 -> the measured sustained bf16 rate; fp32 -> 3xTF32 issues three TF32 MMAs per
    product at half the bf16 rate, so the ceiling is sustained bf16 / 6."""
    if dtype == "bf16":
        return tf_sust, "measured bf16_tflops_sustained"
    return tf_sust / 6.0, "measured bf16_tflops_sustained / 6 (3xTF32: 3 TF32 MMAs per product, TF32 = bf16/2)"


def roofline(eng, dtype, hbm, tflops, tf_src, peak_kind):
    """Per-launch event timing pass -> dominant kernel class and its roofline position.
    `achieved` = the class's algorithmic bytes (or FLOPs) per step / its summed launch
    time; `traffic` = ncu DRAM bytes of the same class per engine launch (thunk)."""
    prof = eng.profile_launches(reps=3)
    by = {}
    for t, ms in prof:
        k = t.kind
        d = by.setdefault(k, {"ms": 0.0, "bytes": 0, "flops": 0, "n": 0})
        d["ms"] += ms
        d["bytes"] += t.nbytes
        d["flops"] += t.flops
        d["n"] += 1
    total = sum(d["ms"] for d in by.values())
    kind, d = max(by.items(), key=lambda kv: kv[1]["ms"])
    gbs = d["bytes"] / (d["ms"] * 1e-3) / 1e9
    tfs = d["flops"] / (d["ms"] * 1e-3) / 1e12
    ridge = tflops * 1e12 / (hbm * 1e9)
    ai = d["flops"] / max(d["bytes"], 1)
    if ai >= ridge:
        ach, peak, unit, bound, psrc = tfs, tflops, "TFLOP/s", "tensor", tf_src
    else:
        ach, peak, unit, bound, psrc = gbs, hbm, "GB/s", "hbm", peak_kind + " hbm_gbs"
    shares = {k: round(v["ms"] / total, 4) for k, v in sorted(by.items(), key=lambda kv: -kv[1]["ms"])}
    traffic, tsrc = None, None
    try:  # ncu-measured DRAM bytes of the same launch class (committed capture, same workload)
        with open(os.path.join(ROOT, "profiles", "step_dram_bytes.json")) as f:
            meas = json.load(f)
        run = meas["runs"].get(f"bytes_{dtype}_{level_of(eng)}.csv", {}).get(kind)
        if run and d["n"]:
            traffic = round(run["dram_bytes"] / d["n"])  # per engine launch, like `achieved`
            tsrc = (f"profiles/step_dram_bytes.json bytes_{dtype}_{level_of(eng)}.csv: ncu "
                    f"dram__bytes_read+write of the class / {d['n']} launches per step")
    except (OSError, KeyError, ValueError):
        pass
    # whole-step roofline bound: sum over launches of max(bytes/BW, flops/peak)
    bound_ms = sum(max(t.nbytes / (hbm * 1e9), t.flops / (tflops * 1e12)) for t, _ in prof) * 1e3
    return {
        "kernel": kind, "bound": bound, "achieved": round(ach, 2), "peak": round(peak, 1), "unit": unit,
        "frac": round(ach / peak, 4), "traffic": traffic, "traffic_source": tsrc,
        "algorithmic_bytes_per_launch": round(d["bytes"] / max(d["n"], 1)), "peak_source": psrc,
        "launches_per_step": d["n"], "kernel_ms_per_step": round(d["ms"], 4),
        "algorithmic_bytes_per_step": d["bytes"], "algorithmic_flops_per_step": d["flops"],
        "also_gbs": round(gbs, 1), "also_tflops": round(tfs, 2),
    }, {"step_ms_sum_of_launches": round(total, 3), "kernel_shares": shares,
        "step_roofline_bound_ms": round(bound_ms, 3),
        "step_bytes": sum(t.nbytes for t, _ in prof), "step_flops": sum(t.flops for t, _ in prof)}


def level_of(eng):
    return getattr(eng, "level_name", "bnff+icf")


def kernel_launches_per_step(eng):
    return sum(getattr(t, "launches", 1) for t in eng.all_thunks())


def measure(args, dtype, x, dy, rank, local, world):
    """One precision mode: device-timed step, e2e step, roofline, unfused comparison."""
    import torch
    import torch.distributed as dist
    from paper_1807_01702_b200 import dp
    dist_on = world > 1
    hbm, tf_burst, tf_sust, peak_kind = load_peaks()
    tflops, tf_src = tensor_peak(dtype, tf_sust)
    batch = args.batch
    g, eng = build_engine(args.level, dtype, batch, args.lr, world, args.syncbn)
    trainer = dp.DPTrainer(eng)
    eng.set_input(x)
    eng.set_loss_grad(dy)
    trainer.capture()

    with ClockSampler(local) as clk:
        ms = timed_steps(trainer, args.steps, args.warmup, dist_on)
    clocks = clk.summary()
    value = world * batch * args.steps / (ms * 1e-3)

    # ---- end to end: host batch -> device each step, result -> host each step
    x_pin = torch.from_numpy(x).pin_memory()
    out_sid = g.outputs[0]
    out_dev = eng.acts[out_sid]
    out_pin = torch.empty(tuple(out_dev.shape), dtype=out_dev.dtype).pin_memory()
    # the loader pattern: each step's batch is copied host->device on a copy stream into
    # one of two device buffers, one step ahead of the compute that consumes it
    xd = [torch.empty(tuple(x_pin.shape), dtype=torch.float32, device="cuda") for _ in range(2)]
    copy_st = torch.cuda.Stream()
    main_st = torch.cuda.current_stream()
    landed = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]

    def prefetch(i):
        b = i % 2
        copy_st.wait_event(consumed[b])  # the conversion of step i-2 has read this buffer
        with torch.cuda.stream(copy_st):
            xd[b].copy_(x_pin, non_blocking=True)
        landed[b].record(copy_st)

    def e2e_step(i):
        b = i % 2
        main_st.wait_event(landed[b])
        eng.set_input(xd[b])
        consumed[b].record(main_st)
        if i + 1 not in (args.warmup, args.warmup + args.steps):  # no copy across the region edges
            prefetch(i + 1)
        trainer.step()
        out_pin.copy_(out_dev, non_blocking=True)

    for ev in consumed:
        ev.record(main_st)
    prefetch(0)
    for i in range(args.warmup):
        e2e_step(i)
    torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    prefetch(args.warmup)  # the first timed step's copy is inside the timed region
    for i in range(args.steps):
        e2e_step(args.warmup + i)
    e1.record(st)
    torch.cuda.synchronize()
    ems = e0.elapsed_time(e1)
    if dist_on:
        tt = torch.tensor([ems], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ems = float(tt.item())
    e2e = {"value": world * batch * args.steps / (ems * 1e-3), "unit": "images/s",
           "h2d_bytes_per_step": int(x_pin.numel() * 4),
           "d2h_bytes_per_step": int(out_pin.numel() * out_pin.element_size())}

    res = {"dtype": dtype, "value": value, "ms_per_step": ms / args.steps, "e2e": e2e,
           "clocks": clocks, "gpu_launches": kernel_launches_per_step(eng) * args.steps}
    if rank == 0:
        res["roofline"], res["step_profile"] = roofline(eng, dtype, hbm, tflops, tf_src, peak_kind)
    del trainer, eng
    if world == 1 and not args.no_unfused:
        _, ueng = build_engine("baseline", dtype, batch, args.lr, 1)
        ueng.set_input(x)
        ueng.set_loss_grad(dy)
        ueng.capture()
        ums = timed_steps(ueng, args.steps, args.warmup, False)
        _, ustep = roofline(ueng, dtype, hbm, tflops, tf_src, peak_kind)
        res["unfused"] = {"level": "baseline", "value": batch * args.steps / (ums * 1e-3),
                          "unit": "images/s", "ms_per_step": ums / args.steps,
                          "algorithmic_step_bytes": ustep["step_bytes"],
                          "kernel_shares": ustep["kernel_shares"]}
        res["speedup_vs_unfused"] = round(value / res["unfused"]["value"], 4)
        fb = res["step_profile"]["step_bytes"]
        res["bn_bytes"] = {
            "fused_step_bytes": fb, "unfused_step_bytes": ustep["step_bytes"],
            "reduction": round(1 - fb / ustep["step_bytes"], 4),
            "definition": "algorithmic HBM bytes per step summed over launches (each tensor "
                          "counted once per launch); ncu dram bytes in profiles/"}
        del ueng
    torch.cuda.empty_cache()
    return res


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` without torchrun: re-launch this script under
    torch.distributed.run with one process per GPU (rank 0 prints the line)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def run_ours(args):
    import torch
    from paper_1807_01702_b200 import dp
    from paper_1807_01702_b200.tensor import Rng

    rank, local, world = dp.init("nccl")
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    batch = args.batch
    from paper_1807_01702_b200 import fusion, graph as G
    g, _ = fusion.plan(G.build_model(G.densenet121(batch), seed=0), fusion.parse_level(args.level))
    # synthetic batch: rows [rank*b, (rank+1)*b) of one global batch drawn with seed 1
    rng = Rng(1)
    n, c, h, w = g.slots[g.inputs[0]].shape
    xg = rng.uniform((n * world, c, h, w), -1.0, 1.0)
    lo, hi = dp.shard_batch(n * world, world, rank)
    x = np.ascontiguousarray(xg[lo:hi])
    dy = rng.normal(g.slots[g.outputs[0]].shape)

    modes = [args.dtype] + [m for m in args.also.split(",") if m and m != args.dtype]
    results = {m: measure(args, m, x, dy, rank, local, world) for m in modes}
    head = results[args.dtype]
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.cpu_batch, args.cpu_iters, 1)
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": head["value"], "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (x~U(-1,1), dy~N(0,1), He-uniform weights, seed 0)",
        "config": {"workload": WORKLOAD, "model": "densenet-121", "global_batch": batch * world,
                   "per_gpu_batch": batch, "image": 224, "level": args.level,
                   "parallelism": f"dp{world}", "sync_bn": bool(args.syncbn),
                   "precision": ("fp32 storage, 3xTF32 tcgen05 with fp32 accumulation, f64 "
                                 "per-channel sums (the reference's fp32 arithmetic)")
                   if args.dtype == "f32" else "bf16 storage, bf16 tcgen05, fp32 accumulation",
                   "l2": "inputs larger than L2 (activations ~GBs/step stream through HBM)",
                   "cuda_graph": True, "input_grad": True},
        "e2e": head["e2e"], "roofline": head.get("roofline"), "cpu_baseline": cpu,
        "clocks": head["clocks"], "gpu_launches": head["gpu_launches"],
    }
    for k in ("unfused", "speedup_vs_unfused", "step_profile", "bn_bytes"):
        if k in head:
            line[k] = head[k]
    for m in modes[1:]:
        line[f"{m}_mode"] = results[m]
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--level", default="bnff+icf")
    ap.add_argument("--dtype", default="f32", choices=["bf16", "f32"],
                    help="headline precision (f32 = the reference's fp32 arithmetic)")
    ap.add_argument("--also", default="bf16",
                    help="further precision modes measured into <mode>_mode objects")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--ref-batch", type=int, default=4)
    ap.add_argument("--cpu-batch", type=int, default=4)
    ap.add_argument("--cpu-iters", type=int, default=3)
    ap.add_argument("--no-unfused", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--syncbn", action="store_true",
                    help="global-batch BN statistics across replicas (2*C all-reduces per BN)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
