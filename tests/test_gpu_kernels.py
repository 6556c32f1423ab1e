"""Kernel-level GPU parity (reference-named API in kernels.py) vs the oracle.

Mirrors the reference's component tests (pkg/tests/test_fused_kernels.py):
conv fwd/bwd over a shape sweep, fused conv+stats, fused norm-relu-conv
(saved bitwise in fp32), fused NRC backward incl. the deferred dx, the
composite conv1-BN-ReLU-conv2 backward, split + deferred, the gamma=0/beta=1
and beta=-1e6 golden cases, and missing-stats -> StateError.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ops as O  # noqa: E402
from paper_1807_01702_b200 import kernels as K  # noqa: E402
from paper_1807_01702_b200.errors import StateError  # noqa: E402
from paper_1807_01702_b200.params import BNParams, ConvParams  # noqa: E402

DT = {"f32": torch.float32, "bf16": torch.bfloat16}
TOL = {"f32": 1e-4, "bf16": 5e-3}


def to_dev(a, dt):
    return torch.from_numpy(np.ascontiguousarray(a.transpose(0, 2, 3, 1))).to("cuda", DT[dt])


def to_host(t):
    return t.float().permute(0, 3, 1, 2).contiguous().cpu().numpy()


def scaled(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


def rounded(a, dt):
    """host copy rounded like the device storage (bf16 inputs are exact bf16 values)."""
    if dt == "bf16":
        return torch.from_numpy(a).to(torch.bfloat16).float().numpy().astype(np.float64)
    return a.astype(np.float64)


SHAPES = [  # n, c, hw, oc, k, stride, pad
    (2, 64, 16, 64, 1, 1, 0), (8, 64, 32, 64, 1, 1, 0), (8, 64, 32, 64, 3, 1, 1),
    (4, 128, 14, 32, 3, 1, 1), (2, 96, 8, 128, 1, 1, 0), (2, 32, 9, 48, 3, 2, 1),
    (2, 8, 32, 16, 7, 2, 3), (3, 256, 7, 256, 1, 1, 0), (1, 16, 5, 16, 3, 1, 1),
    (16, 64, 28, 128, 1, 1, 0),
]


@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_conv_fwd_bwd_sweep(dt, shape):
    n, c, hw, oc, k, s, pad = shape
    rng = np.random.default_rng(sum(shape))
    x = rounded(rng.uniform(-1, 1, (n, c, hw, hw)).astype(np.float32), dt)
    w = rounded(rng.uniform(-0.5, 0.5, (oc, c, k, k)).astype(np.float32), dt)
    p = ConvParams(c, oc, k, k, s, pad, weights=w.astype(np.float32), name="c")
    p64 = ConvParams(c, oc, k, k, s, pad, weights=w, name="c")
    y_ref = O.conv_fwd(x, p64)
    dy = rounded(rng.normal(size=y_ref.shape).astype(np.float32), dt)
    dx_ref, dw_ref, db_ref = O.conv_bwd(x, dy, p64)
    xd = to_dev(x.astype(np.float32), dt)
    y = K.conv2d_fwd(xd, p)
    assert scaled(to_host(y), y_ref) < TOL[dt], "fprop"
    dx, dw, db = K.conv2d_bwd(xd, to_dev(dy.astype(np.float32), dt), p)
    torch.cuda.synchronize()
    assert scaled(to_host(dx), dx_ref) < TOL[dt], "dgrad"
    assert scaled(dw.cpu().numpy(), dw_ref) < TOL[dt], "wgrad"
    assert scaled(db.cpu().numpy(), db_ref) < TOL[dt], "dbias"


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_fused_conv_stats(dt):
    rng = np.random.default_rng(1)
    x = rounded(rng.normal(size=(4, 32, 12, 12)).astype(np.float32), dt)
    w = rng.normal(size=(64, 32, 3, 3)).astype(np.float32) * 0.1
    p = ConvParams(32, 64, 3, 3, pad=1, weights=w, name="c")
    y_ref, st_ref = O.conv_stats_fwd(x, ConvParams(32, 64, 3, 3, pad=1, weights=rounded(w, dt)))
    out = torch.empty((4, 12, 12, 64), dtype=DT[dt], device="cuda")
    st = K.fused_conv_stats_fwd(to_dev(x.astype(np.float32), dt), p, out)
    assert scaled(to_host(out), y_ref) < TOL[dt]
    assert scaled(st.mean.cpu().numpy(), st_ref.mean) < TOL[dt] * 3
    assert scaled(st.var.cpu().numpy(), st_ref.var) < TOL[dt] * 3


def test_fused_nrc_saved_bitwise_f32():
    """saved == relu(bn_fwd(x)) bitwise (test_fused_kernels.py:91-103)."""
    rng = np.random.default_rng(4)
    x = rng.normal(size=(2, 8, 5, 5)).astype(np.float32)
    st_ref = O.stats_onepass(x)
    bn = BNParams(rng.uniform(0.5, 1.5, 8).astype(np.float32), rng.uniform(-.5, .5, 8).astype(np.float32))
    p = ConvParams(8, 16, 3, 3, pad=1, weights=rng.normal(size=(16, 8, 3, 3)).astype(np.float32))
    xd = to_dev(x, "f32")
    st = K.bn_stats_onepass(xd)
    saved = torch.empty_like(xd)
    out = torch.empty((2, 5, 5, 16), dtype=torch.float32, device="cuda")
    K.fused_norm_relu_conv_fwd(xd, st, bn, p, out, saved)
    # bitwise against relu(bn_fwd(x)) evaluated with the SAME (device-reduced) statistics
    from paper_1807_01702_b200.params import ChannelStats
    st_host = ChannelStats(st.sum_x.cpu().numpy(), st.sum_x2.cpu().numpy(), st.count,
                           st.mean.cpu().numpy(), st.var.cpu().numpy())
    assert scaled(st_host.mean, st_ref.mean) < 1e-6
    want = O.relu_fwd(O.bn_apply(x, st_host, bn))
    assert np.array_equal(to_host(saved), want)
    assert scaled(to_host(out), O.conv_fwd(want, p)) < 1e-5


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_gamma0_beta1_and_huge_negative_beta(dt):
    rng = np.random.default_rng(2)
    x = rng.normal(size=(2, 8, 4, 4)).astype(np.float32)
    xd = to_dev(x, dt)
    st = K.bn_stats_onepass(xd)
    idc = ConvParams(8, 8, 1, 1, weights=np.eye(8, dtype=np.float32).reshape(8, 8, 1, 1))
    out = torch.empty_like(xd)
    K.fused_norm_relu_conv_fwd(xd, st, BNParams(np.zeros(8, np.float32), np.ones(8, np.float32)),
                               idc, out)
    assert np.allclose(to_host(out), 1.0)
    idc.bias = np.linspace(-1, 1, 8).astype(np.float32)
    K.fused_norm_relu_conv_fwd(xd, st, BNParams(np.ones(8, np.float32),
                                                np.full(8, -1e6, np.float32)), idc, out)
    got = to_host(out)
    for ch in range(8):
        assert np.allclose(got[:, ch], idc.bias[ch], atol=1e-2 if dt == "bf16" else 1e-7)


def test_missing_stats_state_error():
    xd = torch.zeros((1, 2, 2, 8), device="cuda")
    with pytest.raises(StateError):
        K.fused_norm_relu_conv_fwd(xd, None, BNParams(np.ones(8), np.zeros(8)),
                                   ConvParams(8, 8, 1, 1), torch.empty_like(xd))


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_composite_block_backward(dt):
    """conv1 -> BN -> ReLU -> conv2 with the BN gradient handed to conv1 as a deferred
    package applied in its dgrad/wgrad prologues (test_fused_kernels.py:258-289)."""
    rng = np.random.default_rng(20)
    x1 = rng.normal(size=(2, 16, 10, 10)).astype(np.float32)
    p1 = ConvParams(16, 32, 3, 3, pad=1, weights=(rng.normal(size=(32, 16, 3, 3)) * .2).astype(np.float32))
    bn = BNParams(rng.uniform(0.5, 1.5, 32).astype(np.float32), rng.uniform(-.5, .5, 32).astype(np.float32))
    p2 = ConvParams(32, 16, 3, 3, pad=1, weights=(rng.normal(size=(16, 32, 3, 3)) * .2).astype(np.float32))
    x1r = rounded(x1, dt)
    t0 = O.conv_fwd(x1r, p1)
    st = O.stats_onepass(t0)
    t2 = O.relu_fwd(O.bn_apply(t0, st, bn))
    y = O.conv_fwd(t2, p2)
    dy = rng.normal(size=y.shape).astype(np.float32)
    dt2, dw2_ref, _ = O.conv_bwd(t2, dy.astype(np.float64), p2)
    dt1_ref = O.relu_bwd(O.bn_apply(t0, st, bn), dt2)
    dt0_ref, dg_ref, db_ref = O.bn_bwd(t0, dt1_ref, st, bn)
    dx1_ref, dw1_ref, _ = O.conv_bwd(x1r, dt0_ref, p1)

    xd = to_dev(x1, dt)
    t0d = torch.empty((2, 10, 10, 32), dtype=DT[dt], device="cuda")
    std = K.fused_conv_stats_fwd(xd, p1, t0d)
    yd = torch.empty((2, 10, 10, 16), dtype=DT[dt], device="cuda")
    K.fused_norm_relu_conv_fwd(t0d, std, bn, p2, yd)
    dt1, dw2, _, dg, dbt, table = K.fused_nrc_bwd(t0d, None, std, bn, p2, to_dev(dy, dt), return_table=True)
    dx1, dw1, _ = K.fused_conv_stats_bwd(t0d, xd, p1, dt1, dg, dbt, std, bn.gamma, bn.eps, table=table)
    torch.cuda.synchronize()
    tol = 1e-4 if dt == "f32" else 1.5e-1  # bf16: BN-backward cancellation on 200 px/channel
    assert scaled(dw2.cpu().numpy(), dw2_ref) < tol
    assert scaled(dg.cpu().numpy(), dg_ref) < tol
    assert scaled(dbt.cpu().numpy(), db_ref) < tol
    assert scaled(dw1.cpu().numpy(), dw1_ref) < tol
    assert scaled(to_host(dx1), dx1_ref) < tol


def test_split_with_deferred_f32():
    rng = np.random.default_rng(21)
    x = rng.normal(size=(2, 8, 4, 4)).astype(np.float32)
    st_ref = O.stats_onepass(x)
    bn = BNParams(rng.uniform(0.5, 1.5, 8).astype(np.float32), np.zeros(8, np.float32))
    dt1 = rng.normal(size=x.shape).astype(np.float32)
    xh = O.xhat(x, st_ref, bn.eps)
    dgamma, dbeta = (dt1 * xh).sum((0, 2, 3)), dt1.sum((0, 2, 3))
    other = rng.normal(size=x.shape).astype(np.float32)
    xd = to_dev(x, "f32")
    st = K.bn_stats_onepass(xd)
    inv = st.inv_std(bn.eps)
    m = st.count
    table = (st.mean.float(), inv.float(),
             (torch.tensor(dbeta, dtype=torch.float64, device="cuda") / m).float(),
             (torch.tensor(dgamma, dtype=torch.float64, device="cuda") / m).float(),
             (torch.tensor(bn.gamma, dtype=torch.float64, device="cuda") * inv).float())
    got = K.fused_split_bwd_bn_dx([to_dev(other, "f32"), (to_dev(dt1, "f32"), xd, table)])
    dx_ref, _, _ = O.bn_bwd(x, dt1, st_ref, bn)
    assert scaled(to_host(got), other + dx_ref) < 1e-5


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_bn_ops(dt):
    rng = np.random.default_rng(3)
    x = rounded((rng.normal(size=(4, 16, 9, 9)) * 3 + 1).astype(np.float32), dt)
    dy = rounded(rng.normal(size=x.shape).astype(np.float32), dt)
    bn = BNParams(rng.uniform(0.5, 1.5, 16).astype(np.float32), rng.uniform(-1, 1, 16).astype(np.float32))
    xd, dyd = to_dev(x.astype(np.float32), dt), to_dev(dy.astype(np.float32), dt)
    st2 = K.bn_stats_twopass(xd)
    want = O.stats_twopass(x)
    assert scaled(st2.var.cpu().numpy(), want.var) < 1e-5
    y = K.bn_fwd(xd, st2, bn)
    assert scaled(to_host(y), O.bn_apply(x, want, bn)) < TOL[dt]
    dx, dg, db = K.bn_bwd(xd, dyd, st2, bn)
    rdx, rdg, rdb = O.bn_bwd(x, dy, want, bn)
    tol = 1e-4 if dt == "f32" else 5e-2
    assert scaled(to_host(dx), rdx) < tol and scaled(dg.cpu().numpy(), rdg) < tol
    assert scaled(db.cpu().numpy(), rdb) < tol


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_pool_and_relu(dt):
    rng = np.random.default_rng(5)
    x = rounded(rng.normal(size=(2, 16, 8, 8)).astype(np.float32), dt)
    xd = to_dev(x.astype(np.float32), dt)
    y, st = K.avgpool_fwd(xd, 2, emit_stats=True)
    assert scaled(to_host(y), O.avgpool_fwd(x, 2)) < TOL[dt]
    assert scaled(st.mean.cpu().numpy(), O.stats_onepass(O.avgpool_fwd(x, 2)).mean) < TOL[dt] * 3
    g = rounded(rng.normal(size=(2, 16, 4, 4)).astype(np.float32), dt)
    dx = K.avgpool_bwd(to_dev(g.astype(np.float32), dt), xd.shape, 2)
    assert scaled(to_host(dx), O.avgpool_bwd(g, x.shape, 2)) < TOL[dt]
    r = K.relu_fwd(xd)
    assert np.array_equal(to_host(r), np.maximum(to_host(xd), 0))
    gr = K.relu_bwd(xd, xd)
    assert np.array_equal(to_host(gr), np.where(to_host(xd) > 0, to_host(xd), 0))
