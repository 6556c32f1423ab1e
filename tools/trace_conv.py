"""Timeline of CTA 0 of one window-conv launch (bnff_debug_trace): per stage the producer
issue, the TMA landing, the end of the in-place transform, the MMA issue/commit; per tile
the epilogue's accumulator-full and release.  Prints the average phase latencies -- the
evidence for what a window kernel waits on.

    python tools/trace_conv.py --only 25
"""

from __future__ import annotations

import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench_conv  # noqa: E402
from paper_1807_01702_b200 import _lib  # noqa: E402

EV = ["issue", "issued", "landed", "transformed", "mma_start", "mma_commit", "accf", "acce", "start", "setup"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", type=int, required=True)
    a = ap.parse_args()
    L = _lib.lib()
    buf = torch.zeros(16 * 1024, dtype=torch.int64, device="cuda")
    L.bnff_debug_trace(ctypes.c_void_p(buf.data_ptr()))
    sys.argv = ["bench_conv", "--only", str(a.only), "--reps", "1"]
    bench_conv.main()
    torch.cuda.synchronize()
    L.bnff_debug_trace(None)
    t = buf.cpu().numpy().reshape(16, 1024).astype(np.float64)
    t0 = t[8, 0]
    t = np.where(t > 0, (t - t0) / 1e3, np.nan)  # us since kernel start
    ns = int(np.sum(~np.isnan(t[0])))
    nt = int(np.sum(~np.isnan(t[6])))
    print(f"setup done at {t[9, 0]:.2f} us; {ns} stages, {nt} tiles; last commit {np.nanmax(t[5]):.2f} us, "
          f"last acce {np.nanmax(t[7]):.2f} us")
    d = lambda x, y: np.nanmean(t[y, :ns] - t[x, :ns])  # noqa: E731
    print(f"  producer waits for a free stage  {d(0, 1):7.2f} us")
    print(f"  TMA issue -> landed              {d(1, 2):7.2f} us")
    print(f"  landed -> transformed            {d(2, 3):7.2f} us")
    print(f"  transformed -> MMA start         {d(3, 4):7.2f} us")
    print(f"  MMA start -> commit issued       {d(4, 5):7.2f} us")
    gaps = np.diff(t[4, :ns])
    print(f"  MMA start interval (per stage)   {np.nanmean(gaps):7.2f} us")
    print(f"  epilogue: accf interval per tile {np.nanmean(np.diff(t[6, :nt])):7.2f} us, "
          f"accf -> acce {np.nanmean(t[7, :nt] - t[6, :nt]):7.2f} us")
    nc = int(np.sum(~np.isnan(t[10])))
    e = lambda x, y: np.nanmean(t[y, :nc] - t[x, :nc])  # noqa: E731
    print(f"  epilogue chunk (group 0): wait x + row pass {e(10, 11):6.2f} us, column pass {e(11, 12):6.2f} us, "
          f"store pass {e(12, 13):6.2f} us, chunk start interval {np.nanmean(np.diff(t[10, :nc])):6.2f} us")
    for i in range(min(ns, 12)):
        print("   stage %2d: " % i + " ".join(f"{EV[e]}={t[e, i]:7.2f}" for e in range(6)))


if __name__ == "__main__":
    main()
