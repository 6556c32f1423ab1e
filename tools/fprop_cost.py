"""Cost of the window fprop prologue/epilogue components on one shape (default: the
D121 block-1 1x1, n64 56^2 256->128): operand prologue NONE / RELU / BN_RELU, with and
without the statistics epilogue.  Not a bench number.

    python tools/fprop_cost.py [K] [CIN] [COUT] [HW]
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
    a = [int(v) for v in sys.argv[1:]]
    k, cin, cout, hw = (a + [1, 256, 128, 56][len(a):])[:4]
    n, dev = 64, "cuda"
    p = ConvParams(in_c=cin, out_c=cout, kh=k, kw=k,
                   weights=(np.random.RandomState(1).uniform(-1, 1, (cout, cin, k, k)) / np.sqrt(cin * k * k)).astype(np.float32),
                   bias=np.zeros(cout, np.float32), stride=1, pad=k // 2, name="c")
    pw = K.PackedConv(p, torch.bfloat16, dev, window=True)
    L = _lib.lib()
    x = torch.randn(n, hw, hw, cin, device=dev).to(torch.bfloat16)
    m, s, b, _, _, _ = bench_conv.tables(cin, dev, 3)
    y = torch.empty(n, hw, hw, cout, device=dev, dtype=torch.bfloat16)
    part = torch.zeros((L.bnff_stat_rows(), 2, cout), device=dev)
    print(f"k{k} n{n} {hw}^2 {cin}->{cout}")
    for name, pro, st in (("none", _lib.PRO_NONE, False), ("relu", _lib.PRO_RELU, False),
                          ("bn_relu", _lib.PRO_BN_RELU, False), ("bn_relu + stats", _lib.PRO_BN_RELU, True)):
        tb = (m, s, b) if pro == _lib.PRO_BN_RELU else None

        def run(pro=pro, tb=tb, st=st):
            K._fprop(x, pw, y, pro, tb, part if st else None)
        t = bench_conv.timeit(run, 20)
        gb = (x.numel() + y.numel()) * 2 / t / 1e3
        print(f"  {name:18s} {t:8.1f} us  {gb:7.0f} GB/s")


if __name__ == "__main__":
    main()
