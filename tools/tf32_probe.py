"""Accuracy of the fp32 (3xTF32) conv path against fp64, beside the CPU's own fp32 (sgemm)
on the same inputs: relative RMS and scaled-max errors of y = conv(x, w) for a DenseNet-like
1x1 (K = 1024) and 3x3 (K = 1152).  BNFF_TF32_MODE selects the MMA term set."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1807_01702_b200 import kernels as K
    from paper_1807_01702_b200.params import ConvParams
    rng = np.random.default_rng(0)
    for (n, c, hw, oc, k) in [(8, 1024, 14, 128, 1), (8, 128, 28, 32, 3)]:
        x = rng.normal(size=(n, c, hw, hw)).astype(np.float32)
        w = (rng.uniform(-1, 1, (oc, c, k, k)) / np.sqrt(c * k * k)).astype(np.float32)
        p = ConvParams(c, oc, k, k, pad=k // 2, weights=w, name="p")
        xd = torch.from_numpy(np.ascontiguousarray(x.transpose(0, 2, 3, 1))).cuda()
        y = K.conv2d_fwd(xd, p).permute(0, 3, 1, 2).contiguous().cpu().numpy().astype(np.float64)
        # fp64 and fp32 references via im2col
        def conv(xx, ww):
            xp = np.pad(xx, ((0, 0), (0, 0), (k // 2, k // 2), (k // 2, k // 2)))
            acc = np.zeros((n, oc, hw, hw), xx.dtype)
            for i in range(k):
                for j in range(k):
                    acc += np.einsum("nchw,oc->nohw", xp[:, :, i:i + hw, j:j + hw], ww[:, :, i, j], optimize=True)
            return acc
        y64 = conv(x.astype(np.float64), w.astype(np.float64))
        y32 = conv(x, w).astype(np.float64)
        def errs(a):
            d = a - y64
            return float(np.sqrt(np.mean(d * d)) / np.sqrt(np.mean(y64 * y64))), float(np.max(np.abs(d)) / np.max(np.abs(y64)))
        print(f"mode={os.environ.get('BNFF_TF32_MODE', '0')} k={k} K={c * k * k}: gpu rms {errs(y)[0]:.3e} max {errs(y)[1]:.3e} | "
              f"cpu-fp32 rms {errs(y32)[0]:.3e} max {errs(y32)[1]:.3e}", flush=True)


if __name__ == "__main__":
    main()
