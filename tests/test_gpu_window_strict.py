"""Strict bf16 parity of the TMA window kernels (wconv_kernel / wgrad_kernel), the kernels
the bf16 step actually runs, with bf16-EXACT inputs and weights: every product is exact
in the fp32 accumulator, so the only differences from the fp64 oracle are fp32
accumulation order and the final bf16 rounding of stored tensors.

Bars (stated):
  * stored bf16 outputs (fprop y, dgrad dx / dt1): every element within 1 bf16 ulp of the
    fp64 result rounded to bf16, plus 1e-5 of the tensor's scale (fp32 accumulation of
    K products cannot be closer than that on elements near zero);
  * fp32 outputs -- dw, dbias -- and the epilogue statistics (sum, sum of squares of the
    STORED values; sum dt1, sum dt1*xhat): scaled max error <= 1e-5;
  * BN-prologue paths: the device normalises in fp32 with its own (mean, gamma*inv,
    beta - mean*gamma*inv) tables and rounds the operand to bf16; the host oracle is fed
    exactly that operand (the tables read back from the device, the same single-rounding
    FMA), so the same bars apply.
Shapes cover 1x1 and 3x3 windows, 7^2 .. 56^2 maps, N tiles of 32..256 (register-store and
TMA-store epilogues) and channel counts up to 1024.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ops as O  # noqa: E402
from paper_1807_01702_b200 import kernels as K  # noqa: E402
from paper_1807_01702_b200.params import BNParams, ConvParams  # noqa: E402


def bf(a):
    """round to bf16 (RNE) and back, on the host"""
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).float().numpy()


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a.transpose(0, 2, 3, 1))).to("cuda", torch.bfloat16)


def to_host(t):
    return t.float().permute(0, 3, 1, 2).contiguous().cpu().numpy()


def ulp_err(gpu, ref64, rel=1e-5):
    """max over elements of |gpu - bf16(ref)| / (1 bf16 ulp at ref + rel * max|ref|):
    <= 1 passes the stored-output bar"""
    r = bf(ref64.astype(np.float32)).astype(np.float64)
    mag = np.maximum(np.abs(r), 1e-30)
    ulp = 2.0 ** (np.floor(np.log2(mag)) - 7)
    return float(np.max(np.abs(gpu.astype(np.float64) - r) / (ulp + rel * float(np.max(np.abs(ref64))))))


def f32fma(a, b, c):
    """fmaf(a, b, c) of float32 arrays: exact product and sum in float64, one rounding"""
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(np.float32)


def scaled(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


# (n, c_in, hw, c_out, k): window-eligible stride-1 convs of the benched graphs
SHAPES = [
    (8, 64, 56, 128, 1),     # block-1 CPL 1x1, TMA epilogue (N tile 128)
    (4, 256, 28, 128, 1),    # trans / CPL in 1x1
    (8, 512, 14, 128, 1),
    (16, 1024, 7, 128, 1),   # block-4 width
    (2, 128, 14, 512, 1),    # wide N (256-wide tiles)
    (4, 32, 28, 64, 1),      # narrow: register-store epilogue
    (4, 128, 56, 32, 3),     # CPL 3x3 at 56^2
    (8, 128, 28, 32, 3),
    (16, 128, 14, 32, 3),
    (32, 128, 7, 32, 3),     # whole-image tiles
]


def _data(shape, seed):
    n, c, hw, oc, k = shape
    rng = np.random.default_rng(seed)
    x = bf(rng.uniform(-1, 1, (n, c, hw, hw)))
    w = bf(rng.uniform(-1, 1, (oc, c, k, k)) / np.sqrt(c * k * k))
    dy = bf(rng.normal(size=(n, oc, hw, hw)))
    return x, w, dy


@pytest.mark.parametrize("clip", [False, True], ids=["plain", "relu"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_window_conv_bf16_exact(shape, clip):
    n, c, hw, oc, k = shape
    x, w, dy = _data(shape, sum(shape) + int(clip))
    p = ConvParams(c, oc, k, k, pad=k // 2, weights=w, name="w")
    p64 = ConvParams(c, oc, k, k, pad=k // 2, weights=w.astype(np.float64), name="w")
    pc = K.PackedConv(p, torch.bfloat16)
    assert pc.wf is not None, "window kernel not eligible"
    xd, dyd = to_dev(x), to_dev(dy)
    xe = np.maximum(x, 0).astype(np.float64) if clip else x.astype(np.float64)
    y_ref = O.conv_fwd(xe, p64)
    y = K.conv2d_fwd(xd, pc, clip_input=clip)
    dx, dw, db = K.conv2d_bwd(xd, dyd, pc, clip_input=clip)
    torch.cuda.synchronize()
    dx_ref, dw_ref, db_ref = O.conv_bwd(xe, dy.astype(np.float64), p64)
    if clip:
        dx_ref = np.where(x > 0, dx_ref, 0.0)
    assert ulp_err(to_host(y), y_ref) <= 1.0, "fprop output"
    assert ulp_err(to_host(dx), dx_ref) <= 1.0, "dgrad output"
    assert scaled(dw.cpu().numpy(), dw_ref) <= 1e-5, "wgrad"
    assert scaled(db.cpu().numpy(), db_ref) <= 1e-5, "dbias"


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_window_fprop_stats_epilogue(shape):
    """sub-BN1 statistics fused into the fprop epilogue = moments of the STORED bf16 y."""
    n, c, hw, oc, k = shape
    x, w, _ = _data(shape, 7 + sum(shape))
    p = ConvParams(c, oc, k, k, pad=k // 2, weights=w, name="w")
    out = torch.empty((n, hw, hw, oc), dtype=torch.bfloat16, device="cuda")
    st = K.fused_conv_stats_fwd(to_dev(x), K.PackedConv(p, torch.bfloat16), out)
    y = to_host(out).astype(np.float64)
    want = O.stats_onepass(y)
    assert ulp_err(to_host(out), O.conv_fwd(x.astype(np.float64),
                                             ConvParams(c, oc, k, k, pad=k // 2, weights=w.astype(np.float64)))) <= 1.0
    assert scaled(st.sum_x.cpu().numpy(), want.sum_x) <= 1e-5
    assert scaled(st.sum_x2.cpu().numpy(), want.sum_x2) <= 1e-5


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_window_nrc_forward_backward(shape):
    """BN_RELU operand prologue (fprop + recompute in wgrad) and the NRC dgrad epilogue
    (mask relu(bn(x)) > 0, sum dt1, sum dt1*xhat)."""
    n, c, hw, oc, k = shape
    x, w, dy = _data(shape, 11 + sum(shape))
    rng = np.random.default_rng(3)
    bn = BNParams(rng.uniform(0.5, 1.5, c).astype(np.float32), rng.uniform(-0.5, 0.5, c).astype(np.float32))
    p = ConvParams(c, oc, k, k, pad=k // 2, weights=w, name="w")
    p64 = ConvParams(c, oc, k, k, pad=k // 2, weights=w.astype(np.float64), name="w")
    pc = K.PackedConv(p, torch.bfloat16)
    xd = to_dev(x)
    st = K.bn_stats_onepass(xd)
    m32, s32, b32, i32 = (t.cpu().numpy().reshape(1, c, 1, 1) for t in K._tables(st, bn, xd.device))
    # the device's operand: bf16(relu(fmaf(x, s, fmaf(-m, s, b)))) and its mask
    pre = f32fma(x, s32, f32fma(-m32, s32, b32))
    t = bf(np.maximum(pre, 0)).astype(np.float64)
    y = torch.empty((n, hw, hw, oc), dtype=torch.bfloat16, device="cuda")
    K.fused_norm_relu_conv_fwd(xd, st, bn, pc, y)
    assert ulp_err(to_host(y), O.conv_fwd(t, p64)) <= 1.0, "fprop"
    dt1, dw, db, dg, dbt = K.fused_nrc_bwd(xd, None, st, bn, pc, to_dev(dy))
    torch.cuda.synchronize()
    dt2, dw_ref, db_ref = O.conv_bwd(t, dy.astype(np.float64), p64)
    dt1_ref = np.where(pre > 0, dt2, 0.0)
    assert ulp_err(to_host(dt1), dt1_ref) <= 1.0, "dt1"
    assert scaled(dw.cpu().numpy(), dw_ref) <= 1e-5, "dw"
    assert scaled(db.cpu().numpy(), db_ref) <= 1e-5, "dbias"
    # the epilogue sums are those of the STORED dt1, with xhat = fmaf(x, inv, -mean*inv)
    dt1_h = to_host(dt1).astype(np.float64)
    xh = f32fma(x, i32, (-m32 * i32).astype(np.float32)).astype(np.float64)
    assert scaled(dbt.cpu().numpy(), dt1_h.sum((0, 2, 3))) <= 1e-5, "sum dt1"
    assert scaled(dg.cpu().numpy(), (dt1_h * xh).sum((0, 2, 3))) <= 1e-5, "sum dt1*xhat"
