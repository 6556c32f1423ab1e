"""Summarise one kernel of an ncu --set full report: headline metrics, tensor-pipe
activity, stall reasons, and the hottest SASS basic blocks (by executed instructions and
by stall samples) -- the evidence used to decide what bounds a conv kernel.

    python tools/ncu_stalls.py report.ncu-rep [--top 20]
"""

from __future__ import annotations

import argparse
import csv
import io
import subprocess


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=20)
    a = ap.parse_args()
    rows = ncu_csv(a.rep, "--page", "raw")
    h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
    raw = dict(zip(h, v))
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_tc_wavefronts_mem_shared.sum",
            "launch__grid_size", "launch__registers_per_thread"]
    for k in keys:
        if k in raw:
            print(f"{k:70s} {raw[k]}")
    # shared-memory pressure (the 3xTF32 kernels transform operands in place)
    for k in sorted(raw):
        if (k.startswith("l1tex__throughput") or "mem_shared" in k or k.startswith("l1tex__data_bank_conflicts")) \
                and (k.endswith(".pct_of_peak_sustained_active") or k.endswith(".sum")):
            print(f"{k:70s} {raw[k]}")
    print("-- stalls (per issue active)")
    st = []
    for k, val in raw.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio"):
            try:
                st.append((float(val), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    for val, k in sorted(st, reverse=True)[:10]:
        print(f"  {k:30s} {val:.3f}")
    src = ncu_csv(a.rep, "--page", "source", "--print-source", "sass")
    hdr = src[1]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iss, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    lines = []
    for r in src[2:]:
        try:
            lines.append((r[ia][-5:], int(r[iex]), int(r[iss]), r[isrc].strip()))
        except (ValueError, IndexError):
            pass
    tot_i = sum(x[1] for x in lines) or 1
    tot_s = sum(x[2] for x in lines) or 1
    blocks, cur = [], None
    for ad, n, s, t in lines:
        if cur and cur[1] == n:
            cur[2] += n
            cur[3] += s
            cur[4] += 1
            cur[5].append(t)
        else:
            cur = [ad, n, n, s, 1, [t]]
            blocks.append(cur)
    print("-- hottest basic blocks (instructions executed | stall samples)")
    for b in sorted(blocks, key=lambda b: -(b[2] / tot_i + b[3] / tot_s))[: a.top]:
        ops = ",".join(sorted({t.split()[0] if not t.startswith("@") else t.split()[1] for t in b[5]})[:8])
        print(f"  {b[0]} x{b[1]:8d} n={b[4]:4d} inst {b[2] / tot_i * 100:5.1f}% stall {b[3] / tot_s * 100:5.1f}%  {ops}")


if __name__ == "__main__":
    main()
