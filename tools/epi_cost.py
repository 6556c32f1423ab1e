"""Cost of each 1x1 dgrad epilogue component (D121 block-1 shape, n64 56^2 224<-128):
the same window dgrad timed with the epilogue variants PLAIN (store only), CLIP (+x mask
tile), NRC without / with statistics, NRC_ACC (the ICF fold).  Not a bench number.

    python tools/epi_cost.py
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench_conv  # noqa: E402
from paper_1807_01702_b200 import _lib  # noqa: E402
from paper_1807_01702_b200 import kernels as K  # noqa: E402
from paper_1807_01702_b200.params import ConvParams  # noqa: E402


def main():
    n, hw, cin, cout = 64, 56, int(os.environ.get("CIN", 224)), 128
    dev = "cuda"
    p = ConvParams(in_c=cin, out_c=cout, kh=1, kw=1,
                   weights=(np.random.RandomState(1).uniform(-1, 1, (cout, cin, 1, 1)) / np.sqrt(cin)).astype(np.float32),
                   bias=np.zeros(cout, np.float32), stride=1, pad=0, name="c1")
    pw = K.PackedConv(p, torch.bfloat16, dev, window=True)
    L = _lib.lib()
    dy = torch.randn(n, hw, hw, cout, device=dev).to(torch.bfloat16)
    dyx = torch.randn(n, hw, hw, cout, device=dev).to(torch.bfloat16)
    x = torch.randn(n, hw, hw, cin, device=dev).to(torch.bfloat16)
    m, s, b, inv, k1, k2 = bench_conv.tables(cout, dev, 4)
    em, es, eb, einv, _, _ = bench_conv.tables(cin, dev, 5)
    pkg = (dy, dyx, (m, inv, k1, k2, s))
    part = torch.zeros((L.bnff_stat_rows(), 2, cin), dtype=torch.float64, device=dev)
    G = torch.zeros(n, hw, hw, cin, device=dev, dtype=torch.bfloat16)
    rows = []
    for name, epi, use_pkg, st in (("plain, dy only", _lib.DG_PLAIN, False, False),
                                   ("plain, BN_DX prologue", _lib.DG_PLAIN, True, False),
                                   ("clip (x mask)", _lib.DG_CLIP, True, False),
                                   ("nrc, no stats", _lib.DG_NRC, True, False),
                                   ("nrc + stats", _lib.DG_NRC, True, True),
                                   ("nrc_acc (fold) + stats", getattr(_lib, "DG_NRC_ACC", 3), True, True)):
        def run(epi=epi, use_pkg=use_pkg, st=st):
            K._dgrad(dy, pw, x, epi, x, (em, es, eb, einv), part if st else None, pkg if use_pkg else None)
        t = bench_conv.timeit(run, 20)
        rows.append((name, t))
    tiles = (n * hw * hw // 128) * ((cin + 127) // 128)
    print(f"1x1 dgrad n{n} {hw}^2 {cin}<-{cout}: {tiles} tiles on 148 SMs")
    for name, t in rows:
        print(f"  {name:28s} {t:8.1f} us   {t * 148 / tiles:6.2f} us per tile per SM")


if __name__ == "__main__":
    main()
