"""Numpy restatement of the reference's per-layer kernels (TEST INFRASTRUCTURE).

Each function follows the cited reference function line by line in *semantics*
(dtype of every intermediate, float64 per-channel sums, clamping, mask
conventions) so the oracle reproduces the reference to rounding; it is
pinned against fixtures generated from the reference itself
(``tests/golden/make_golden.py``).  Arrays are NCHW like the reference.
"""

from __future__ import annotations

import numpy as np

from paper_1807_01702_b200.errors import ShapeError, StateError
from paper_1807_01702_b200.params import BNParams, ChannelStats, ConvParams

# ---------------------------------------------------------------------------
# convolution  (ops.py:151-204, fused.py:36-50)
# ---------------------------------------------------------------------------


def _taps(xp, kh, kw, s, oh, ow):
    return xp[:, :, kh: kh + s * oh: s, kw: kw + s * ow: s]


def conv_fwd(x: np.ndarray, p: ConvParams) -> np.ndarray:
    """y[n,o] = bias[o] + sum_{i,kh,kw} xpad[n,i,..]*w[o,i,kh,kw]  (ops.py:151-175).

    Accumulation in x's dtype, one tap at a time; bias added only when nonzero."""
    n, c, h, w = x.shape
    if c != p.in_c:
        raise ShapeError(f"{p.name}: input has {c} channels, expected {p.in_c}")
    oh, ow = p.out_hw(h, w)
    xp = np.pad(x, ((0, 0), (0, 0), (p.pad, p.pad), (p.pad, p.pad))) if p.pad else x
    wt = p.weights.astype(x.dtype, copy=False)
    acc = np.zeros((n, p.out_c, oh, ow), dtype=x.dtype)
    for kh in range(p.kh):
        for kw in range(p.kw):
            patch = _taps(xp, kh, kw, p.stride, oh, ow)           # (n, i, oh, ow)
            acc += np.tensordot(wt[:, :, kh, kw], patch, axes=([1], [1])).transpose(1, 0, 2, 3)
    if np.any(p.bias):
        acc += p.bias.astype(x.dtype).reshape(1, -1, 1, 1)
    return acc


def conv_bwd(x: np.ndarray, dy: np.ndarray, p: ConvParams):
    """(dx, dw, dbias) adjoints of conv_fwd  (ops.py:178-204)."""
    n, c, h, w = x.shape
    oh, ow = p.out_hw(h, w)
    if dy.shape != (n, p.out_c, oh, ow):
        raise ShapeError(f"{p.name}: dy shape {dy.shape} != {(n, p.out_c, oh, ow)}")
    s, pad = p.stride, p.pad
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad))) if pad else x
    wt = p.weights.astype(x.dtype, copy=False)
    dxp = np.zeros_like(xp)
    dw = np.zeros_like(wt)
    for kh in range(p.kh):
        for kw in range(p.kw):
            patch = _taps(xp, kh, kw, s, oh, ow)
            dw[:, :, kh, kw] = np.tensordot(dy, patch, axes=([0, 2, 3], [0, 2, 3]))
            dxp[:, :, kh: kh + s * oh: s, kw: kw + s * ow: s] += np.tensordot(
                wt[:, :, kh, kw], dy, axes=([0], [1])).transpose(1, 0, 2, 3)
    dx = dxp[:, :, pad: pad + h, pad: pad + w] if pad else dxp
    dbias = dy.sum(axis=(0, 2, 3), dtype=np.float64).astype(x.dtype)
    return np.ascontiguousarray(dx), dw.astype(p.weights.dtype), dbias


# ---------------------------------------------------------------------------
# batch-norm statistics and transforms  (ops.py:212-298)
# ---------------------------------------------------------------------------


def stats_twopass(x: np.ndarray) -> ChannelStats:
    """float64 sums + centred variance (ops.py:212-228)."""
    xd = x.astype(np.float64, copy=False)
    n, c, h, w = xd.shape
    m = n * h * w
    s1 = xd.sum(axis=(0, 2, 3))
    s2 = (xd * xd).sum(axis=(0, 2, 3))
    mean = s1 / m
    d = xd - mean.reshape(1, c, 1, 1)
    return ChannelStats(s1, s2, m, mean, (d * d).sum(axis=(0, 2, 3)) / m)


def stats_onepass(x: np.ndarray) -> ChannelStats:
    """float64 Sigma x, Sigma x^2 -> from_sums (ops.py:231-237)."""
    xd = x.astype(np.float64, copy=False)
    n, c, h, w = xd.shape
    return ChannelStats.from_sums(xd.sum(axis=(0, 2, 3)), (xd * xd).sum(axis=(0, 2, 3)), n * h * w)


def _vec(v, dtype, c):
    return np.asarray(v).astype(dtype).reshape(1, c, 1, 1)


def bn_apply(x: np.ndarray, stats: ChannelStats, p: BNParams) -> np.ndarray:
    """(x - mean) * (gamma*inv) + beta with per-channel factors cast to x.dtype (ops.py:240-254)."""
    c = x.shape[1]
    if stats.mean.shape[0] != c or p.channels != c:
        raise ShapeError(f"{p.name}: stats/params for {stats.mean.shape[0]}/{p.channels} "
                         f"channels, input has {c}")
    inv = stats.inv_std(p.eps)
    y = (x - _vec(stats.mean, x.dtype, c)) * _vec(p.gamma * inv, x.dtype, c)
    y += _vec(p.beta, x.dtype, c)
    return y


def xhat(x: np.ndarray, stats: ChannelStats, eps: float) -> np.ndarray:
    c = x.shape[1]
    return (x - _vec(stats.mean, x.dtype, c)) * _vec(stats.inv_std(eps), x.dtype, c)


def bn_dx(x, dy, stats: ChannelStats, gamma, eps, dgamma, dbeta) -> np.ndarray:
    """gamma*inv*(dy - dbeta/m - xhat*dgamma/m), factors cast to x.dtype (ops.py:283-298)."""
    c, m = x.shape[1], stats.count
    k1 = _vec(np.asarray(dbeta, dtype=np.float64) / m, x.dtype, c)
    k2 = _vec(np.asarray(dgamma, dtype=np.float64) / m, x.dtype, c)
    g = _vec(np.asarray(gamma) * stats.inv_std(eps), x.dtype, c)
    return g * (dy - k1 - xhat(x, stats, eps) * k2)


def bn_bwd(x, dy, stats: ChannelStats, p: BNParams):
    """Full BN adjoint (ops.py:257-280): returns (dx, dgamma, dbeta) in x.dtype."""
    if x.shape != dy.shape:
        raise ShapeError(f"{p.name}: dy shape {dy.shape} != x shape {x.shape}")
    xh = xhat(x, stats, p.eps)
    dbeta = dy.sum(axis=(0, 2, 3), dtype=np.float64)
    dgamma = (dy * xh).sum(axis=(0, 2, 3), dtype=np.float64)
    dx = bn_dx(x, dy, stats, p.gamma, p.eps, dgamma, dbeta)
    return dx, dgamma.astype(x.dtype), dbeta.astype(x.dtype)


def relu_fwd(x):
    return np.maximum(x, x.dtype.type(0))


def relu_bwd(x, dy):
    """dy where x > 0 (subgradient 0 at 0) -- ops.py:314-319."""
    if x.shape != dy.shape:
        raise ShapeError(f"relu_bwd: shape mismatch {x.shape} vs {dy.shape}")
    return np.where(x > 0, dy, x.dtype.type(0))


def avgpool_fwd(x, k: int):
    """Non-overlapping k x k mean, accumulated in x.dtype (ops.py:428-443)."""
    n, c, h, w = x.shape
    oh, ow = h // k, w // k
    if oh < 1 or ow < 1:
        raise ShapeError(f"avgpool: window {k} larger than input {h}x{w}")
    win = x[:, :, : oh * k, : ow * k].reshape(n, c, oh, k, ow, k)
    return win.mean(axis=(3, 5), dtype=x.dtype)


def avgpool_bwd(dy, in_shape, k: int):
    """dy/k^2 spread over each window (ops.py:446-454)."""
    n, c, h, w = in_shape
    oh, ow = dy.shape[2], dy.shape[3]
    dx = np.zeros(in_shape, dtype=dy.dtype)
    dx[:, :, : oh * k, : ow * k] = np.repeat(np.repeat(dy, k, axis=2), k, axis=3) / (k * k)
    return dx


# ---------------------------------------------------------------------------
# fused kernels  (fused.py:79-230) -- same values as the tiled reference
# ---------------------------------------------------------------------------


def conv_stats_fwd(x, conv: ConvParams):
    """conv + float64 output sums (fused.py:79-100) -> (y, ChannelStats)."""
    y = conv_fwd(x, conv)
    y64 = y.astype(np.float64)
    n, _, oh, ow = y.shape
    return y, ChannelStats.from_sums(y64.sum(axis=(0, 2, 3)), (y64 * y64).sum(axis=(0, 2, 3)),
                                     n * oh * ow)


def norm_relu_conv_fwd(x, stats: ChannelStats, bn: BNParams, conv: ConvParams,
                       emit_stats: bool = False):
    """normalize -> ReLU (saved) -> conv, optional output stats (fused.py:103-154).
    Returns (y, saved_postrelu, out_stats|None)."""
    if stats is None:
        raise StateError(f"{conv.name}: no statistics available for normalization input")
    saved = relu_fwd(bn_apply(x, stats, bn))
    if emit_stats:
        y, st = conv_stats_fwd(saved, conv)
        return y, saved, st
    return conv_fwd(saved, conv), saved, None


def nrc_bwd(x, saved, stats: ChannelStats, bn: BNParams, conv: ConvParams, dy):
    """(dt1, dw, dbias, dgamma64, dbeta64) -- fused.py:157-200."""
    if saved is None:
        raise StateError(f"{conv.name}: missing saved post-relu tensor for backward")
    dt, dw, dbias = conv_bwd(saved, dy, conv)
    dt1 = dt * (saved > 0)  # fused.py:184 multiplies by the boolean mask
    dbeta = dt1.sum(axis=(0, 2, 3), dtype=np.float64)
    dgamma = (dt1 * xhat(x, stats, bn.eps)).sum(axis=(0, 2, 3), dtype=np.float64)
    return np.ascontiguousarray(dt1), dw, dbias, dgamma, dbeta


def conv_stats_bwd(x_own, saved_in, conv: ConvParams, dt1, dgamma, dbeta, stats,
                   gamma, eps, clip_input=False):
    """deferred BN dx against the kernel's own output, then conv adjoints (fused.py:203-219)."""
    dy = bn_dx(x_own, dt1, stats, gamma, eps, dgamma, dbeta)
    xe = relu_fwd(saved_in) if clip_input else saved_in
    dx, dw, db = conv_bwd(xe, dy, conv)
    if clip_input:
        dx = np.where(saved_in > 0, dx, saved_in.dtype.type(0))
    return dx, dw, db
