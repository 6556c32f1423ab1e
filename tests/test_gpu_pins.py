"""The reference's own edge pins, on the device kernels.

  * one-pass statistics: constant input clamps the variance to 0
    (test_ops.py:187-190) and the mean-1e3 / sd-1 cancellation case stays within
    1e-2 of two-pass (test_ops.py:192-198) -- for the standalone sub-BN1 sums
    (bn_stats_onepass) and for the conv-epilogue statistics (fused_conv_stats_fwd);
  * BN backward with constant dy: dbeta = 4g, dgamma = 0, dx = 0 (test_ops.py:253-261);
  * fused == sequential over 100 random seeds (test_fused_kernels.py:314-354), with
    the reference's own tolerances, through the fused kernels of kernels.py.  Channel
    counts below the kernels' 16-byte granule are zero-padded (zero input channels,
    zero gamma/beta, zero weight rows/columns: the padded channels stay exactly 0).

fp32 mode throughout (the reference's arithmetic); the pins that are meaningful in
bf16 storage (constant clamp, constant dy) run in both modes.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ops as O  # noqa: E402
from paper_1807_01702_b200 import kernels as K  # noqa: E402
from paper_1807_01702_b200.params import BNParams, ChannelStats, ConvParams  # noqa: E402

DT = {"f32": torch.float32, "bf16": torch.bfloat16}


def to_dev(a, dt="f32"):
    return torch.from_numpy(np.ascontiguousarray(a.transpose(0, 2, 3, 1))).to("cuda", DT[dt])


def to_host(t):
    return t.float().permute(0, 3, 1, 2).contiguous().cpu().numpy()


def rel_err(a, b, floor=1e-6):
    """test_ops.py's rel_err: max|a-b| / max(max|b|, floor)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), floor))


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_onepass_constant_clamps_to_zero(dt):
    c = 4 if dt == "f32" else 8
    st = K.bn_stats_onepass(to_dev(np.full((2, c, 4, 4), 1.234, np.float32), dt))
    var = st.var.cpu().numpy()
    assert np.all(var >= 0.0)
    assert np.allclose(var, 0.0)


def test_onepass_adversarial_cancellation():
    rng = np.random.default_rng(9)
    x = (rng.normal(size=(4, 4, 16, 16)) + 1000.0).astype(np.float32)
    one = K.bn_stats_onepass(to_dev(x))
    two = O.stats_twopass(x)
    assert rel_err(one.var.cpu().numpy(), two.var) < 1e-2
    dev_two = K.bn_stats_twopass(to_dev(x))
    assert rel_err(dev_two.var.cpu().numpy(), two.var) < 1e-5


@pytest.mark.parametrize("k", [1, 3])
def test_conv_epilogue_stats_cancellation(k):
    """The same pin on the sub-BN1 statistics fused into the conv epilogue: an identity
    conv (centre tap 1) with bias 1000 writes x + 1000; its one-pass moments stay within
    1e-2 of the two-pass variance of what was written."""
    rng = np.random.default_rng(10)
    c = 8
    x = rng.normal(size=(4, c, 16, 16)).astype(np.float32)
    w = np.zeros((c, c, k, k), np.float32)
    for i in range(c):
        w[i, i, k // 2, k // 2] = 1.0
    p = ConvParams(c, c, k, k, pad=k // 2, weights=w, bias=np.full(c, 1000.0, np.float32), name="id")
    out = torch.empty((4, 16, 16, c), dtype=torch.float32, device="cuda")
    st = K.fused_conv_stats_fwd(to_dev(x), p, out)
    y = to_host(out)
    assert rel_err(st.var.cpu().numpy(), O.stats_twopass(y).var) < 1e-2
    assert rel_err(st.mean.cpu().numpy(), O.stats_twopass(y).mean) < 1e-6


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_bn_bwd_constant_dy(dt):
    """x = [1, 2, 3, 4] per channel, dy = g everywhere: dbeta = 4g, dgamma = 0, dx = 0."""
    g = 0.7 if dt == "f32" else 0.703125  # bf16-exact
    c = 4 if dt == "f32" else 8
    x = np.tile(np.array([1.0, 2.0, 3.0, 4.0], np.float32).reshape(1, 1, 2, 2), (1, c, 1, 1))
    bn = BNParams(gamma=np.ones(c, np.float32), beta=np.zeros(c, np.float32))
    xd = to_dev(x, dt)
    st = K.bn_stats_twopass(xd)
    dx, dg, db = K.bn_bwd(xd, to_dev(np.full_like(x, g), dt), st, bn)
    torch.cuda.synchronize()
    assert np.allclose(db.cpu().numpy(), 4 * g, rtol=1e-6)
    assert np.allclose(dg.cpu().numpy(), 0.0, atol=1e-6)
    assert np.allclose(to_host(dx), 0.0, atol=1e-6)


def _pad4(c):
    return (c + 3) // 4 * 4


@pytest.mark.parametrize("seed", range(100))
def test_fused_equals_sequential_100_seeds(seed):
    """test_fused_kernels.py:314-354 on the device: same shape generator, same
    tolerances, the sequential side computed by the oracle's unfused ops."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 5))
    c = int(rng.integers(1, 9))
    hw = int(rng.integers(2, 9))
    oc = int(rng.integers(1, 9))
    k = int(rng.choice([1, 3]))
    pad = 1 if k == 3 else 0
    x = rng.normal(size=(n, c, hw, hw)).astype(np.float32)
    gamma = rng.uniform(0.5, 1.5, c).astype(np.float32)
    beta = rng.uniform(-0.5, 0.5, c).astype(np.float32)
    w = rng.normal(size=(oc, c, k, k)).astype(np.float32)
    rng.choice([2048, 65536, 256 * 1024])  # the reference draws a tile budget here
    p = ConvParams(in_c=c, out_c=oc, kh=k, kw=k, pad=pad, weights=w, name="c")
    bn = BNParams(gamma=gamma, beta=beta)

    # device operands, zero-padded to 16-byte channel rows
    cp, ocp = _pad4(c), _pad4(oc)
    xp = np.zeros((n, cp, hw, hw), np.float32)
    xp[:, :c] = x
    wp = np.zeros((ocp, cp, k, k), np.float32)
    wp[:oc, :c] = w
    pp = ConvParams(in_c=cp, out_c=ocp, kh=k, kw=k, pad=pad, weights=wp, name="c")
    bnp = BNParams(gamma=np.pad(gamma, (0, cp - c)), beta=np.pad(beta, (0, cp - c)))
    xd = to_dev(xp)

    # fused_conv_stats_fwd vs conv + two-pass stats
    out = torch.empty((n, hw, hw, ocp), dtype=torch.float32, device="cuda")
    stats = K.fused_conv_stats_fwd(xd, pp, out)
    ref = O.conv_fwd(x.astype(np.float64), p)
    ref_stats = O.stats_twopass(ref)
    assert rel_err(to_host(out)[:, :oc], ref, floor=1e-5) < 1e-5
    assert rel_err(stats.var.cpu().numpy()[:oc], ref_stats.var, floor=1e-4) < 1e-4

    # fused_norm_relu_conv_fwd vs conv(relu(bn_fwd(x)))
    in_stats = K.bn_stats_onepass(xd)
    host_stats = O.stats_onepass(x)
    out2 = torch.empty((n, hw, hw, ocp), dtype=torch.float32, device="cuda")
    saved = torch.empty_like(xd)
    K.fused_norm_relu_conv_fwd(xd, in_stats, bnp, pp, out2, saved)
    t2 = O.relu_fwd(O.bn_apply(x, host_stats, bn))
    assert rel_err(to_host(out2)[:, :oc], O.conv_fwd(t2, p), floor=1e-4) < 1e-4

    # fused_nrc_bwd vs conv_bwd -> relu_bwd -> bn_bwd
    dy = rng.normal(size=(n, oc, hw, hw)).astype(np.float32)
    dyp = np.zeros((n, ocp, hw, hw), np.float32)
    dyp[:, :oc] = dy
    dt1, dw, db, dgamma, dbeta = K.fused_nrc_bwd(xd, saved, in_stats, bnp, pp, to_dev(dyp))
    torch.cuda.synchronize()
    dt2_ref, dw_ref, db_ref = O.conv_bwd(t2, dy.astype(np.float64), p)
    dt1_ref = O.relu_bwd(O.bn_apply(x, host_stats, bn), dt2_ref)
    _, dgamma_ref, dbeta_ref = O.bn_bwd(x, dt1_ref, host_stats, bn)
    assert rel_err(dw.cpu().numpy()[:oc, :c], dw_ref, floor=1e-3) < 1e-3
    assert rel_err(db.cpu().numpy()[:oc], db_ref, floor=1e-3) < 1e-3
    assert rel_err(to_host(dt1)[:, :c], dt1_ref, floor=1e-3) < 1e-3
    assert rel_err(dgamma.cpu().numpy()[:c], dgamma_ref, floor=1e-3) < 1e-3
    assert rel_err(dbeta.cpu().numpy()[:c], dbeta_ref, floor=1e-3) < 1e-3
