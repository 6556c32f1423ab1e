"""Reference-named functional API over libbnff (device tensors, NHWC).

Mirrors the kernel-level boundary of the reference (``fused.py:79-230`` and
``ops.py:151-454``): same function names, argument order and meaning, same
error types (``ShapeError`` / ``StateError``).  Differences, all of layout
rather than semantics:

* feature maps are NHWC torch tensors on the GPU (bf16 or fp32); ``out`` /
  ``saved_out`` may be channel-offset slices of a larger buffer (a DenseNet
  block buffer), exactly like the reference's strided ``out`` views;
* statistics are returned as ``DevStats`` (float64 device tensors);
* ``budget`` / ``workers`` are accepted and ignored (tiling is the GPU grid).

Every call launches hand-written sm_100a kernels through the C ABI; nothing
here computes on the CPU.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from .errors import ShapeError, StateError
from .params import BNParams, ConvParams

DEFAULT_BUDGET = 256 * 1024


def _ptr(t):
    return 0 if t is None else int(t.data_ptr())


def _dcode(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.BF16
    if t.dtype == torch.float32:
        return _lib.F32
    raise ShapeError(f"unsupported dtype {t.dtype}")


def view(t: torch.Tensor) -> _lib.View:
    if t.dim() != 4 or t.stride(3) != 1:
        raise ShapeError(f"expected an NHWC view with unit channel stride, got {tuple(t.shape)}")
    n, h, w, c = t.shape
    # pixel stride; a contiguous tensor's is c even where size-1 dims carry arbitrary strides
    rs = c if t.is_contiguous() else t.stride(2)
    return _lib.View(_ptr(t), n, h, w, c, rs)


def coef(*arrs) -> _lib.Coef:
    a = list(arrs) + [None] * (5 - len(arrs))
    return _lib.Coef(*(_ptr(x) for x in a))


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _call(fn, *args, what=""):
    _lib.check(fn(*args, _stream()), what)


def _L():
    return _lib.lib()


@dataclass
class DevStats:
    """ChannelStats on the device (ops.py:94-125): float64 sums and moments."""
    sum_x: torch.Tensor
    sum_x2: torch.Tensor
    count: int
    mean: torch.Tensor
    var: torch.Tensor

    def inv_std(self, eps: float) -> torch.Tensor:
        return 1.0 / torch.sqrt(torch.clamp(self.var, min=0.0) + eps)

    def slice(self, lo, hi):
        return DevStats(self.sum_x[lo:hi], self.sum_x2[lo:hi], self.count, self.mean[lo:hi],
                        self.var[lo:hi])


def _new_stats(c, count, device):
    z = lambda: torch.zeros(c, dtype=torch.float64, device=device)  # noqa: E731
    return DevStats(z(), z(), count, z(), z())


def _finalize(part, tiles, st: DevStats):
    _call(_L().bnff_stats_finalize, _ptr(part), tiles, st.mean.shape[0], st.count, _ptr(st.sum_x),
          _ptr(st.sum_x2), _ptr(st.mean), _ptr(st.var), what="stats_finalize")


def _pixels(t):
    return t.shape[0] * t.shape[1] * t.shape[2]


class PackedConv:
    """Device copy of a ConvParams: fp32 master + packed operand layouts."""

    def __init__(self, p: ConvParams, dtype: torch.dtype, device="cuda", cin_store=None,
                 window: bool = True):
        self.p = p
        self.dcode = _lib.BF16 if dtype == torch.bfloat16 else _lib.F32
        self.cin_store = cin_store or p.in_c
        self.w32 = torch.as_tensor(p.weights, dtype=torch.float32).contiguous().to(device)
        self.bias = torch.as_tensor(p.bias, dtype=torch.float32).contiguous().to(device)
        L = _L()
        n = L.bnff_pack_size(self.dcode, p.out_c, self.cin_store, p.kh, p.kw)
        nt = L.bnff_pack_size(self.dcode, self.cin_store, p.out_c, p.kh, p.kw)
        self.wp = torch.zeros(n, dtype=dtype, device=device)
        self.wt = torch.zeros(nt, dtype=dtype, device=device)
        _call(L.bnff_pack_weights, self.dcode, _ptr(self.w32), p.out_c, p.in_c, self.cin_store,
              p.kh, p.kw, _ptr(self.wp), _ptr(self.wt), what="pack_weights")
        # window-shift kernel weights (used when the conv/input qualifies, bf16 only)
        self.wf = self.wd = None
        if window and self.cin_store == p.in_c:
            nf = L.bnff_window_pack_size(self.dcode, p.out_c, p.in_c, p.kh, p.kw, 0)
            nd = L.bnff_window_pack_size(self.dcode, p.out_c, p.in_c, p.kh, p.kw, 1)
            self.wf = torch.zeros(nf, dtype=dtype, device=device)
            self.wd = torch.zeros(nd, dtype=dtype, device=device)
            _call(L.bnff_pack_window, self.dcode, _ptr(self.w32), p.out_c, p.in_c, p.kh, p.kw,
                  _ptr(self.wf), _ptr(self.wd), what="pack_window")


def _packed(conv, x):
    if isinstance(conv, PackedConv):
        return conv
    return PackedConv(conv, x.dtype, x.device, cin_store=x.shape[3])


def _out_like(x, conv: ConvParams, out):
    n, h, w, _ = x.shape
    oh, ow = conv.out_hw(h, w)
    if out is None:
        return torch.empty((n, oh, ow, conv.out_c), dtype=x.dtype, device=x.device)
    if tuple(out.shape) != (n, oh, ow, conv.out_c):
        raise ShapeError(f"{conv.name}: out shape {tuple(out.shape)} != {(n, oh, ow, conv.out_c)}")
    return out


def _fprop(x, pc: PackedConv, out, pro, tables, stat_part):
    p = pc.p
    a = _lib.FpropArgs(_dcode(x), p.kh, p.kw, p.stride, p.pad, view(x), view(out), _ptr(pc.wp),
                       _ptr(pc.bias), pro, coef(*(tables or ())), _ptr(stat_part), _ptr(pc.wf))
    _call(_L().bnff_conv_fprop, C.byref(a), what=f"fprop {p.name}")


def _check_cin(x, conv):
    if x.shape[3] != conv.in_c and x.shape[3] < conv.in_c:
        raise ShapeError(f"{conv.name}: input has {x.shape[3]} channels, expected {conv.in_c}")


# ---------------------------------------------------------------------------
# ops.py equivalents
# ---------------------------------------------------------------------------


def conv2d_fwd(x, p, out=None, clip_input: bool = False):
    """ops.conv2d_fwd (ops.py:151-175); clip_input = RCF clipped read (execute.py:170)."""
    pc = _packed(p, x)
    _check_cin(x, pc.p)
    out = _out_like(x, pc.p, out)
    _fprop(x, pc, out, _lib.PRO_RELU if clip_input else _lib.PRO_NONE, None, None)
    return out


def _wgrad(x, dy, pc, x_pro=_lib.PRO_NONE, x_tables=None, dy_pkg=None):
    p = pc.p
    L = _L()
    n, h, w, _ = x.shape
    oh, ow = p.out_hw(h, w)
    ws_n = L.bnff_wgrad_workspace(n, oh, ow, p.kh, p.kw, x.shape[3], p.out_c, 0)
    ws = torch.empty(ws_n, dtype=torch.float32, device=x.device)
    dw = torch.empty((p.out_c, p.in_c, p.kh, p.kw), dtype=torch.float32, device=x.device)
    db = torch.empty(p.out_c, dtype=torch.float32, device=x.device)
    if dy_pkg is None:
        dyv, dyx, dpro, dcf = view(dy), view(dy), _lib.PRO_NONE, coef()
    else:
        dyv, dyx, dpro, dcf = view(dy_pkg[0]), view(dy_pkg[1]), _lib.PRO_BN_DX, coef(*dy_pkg[2])
    a = _lib.WgradArgs(_dcode(x), p.kh, p.kw, p.stride, p.pad, view(x), x_pro,
                       coef(*(x_tables or ())), dyv, dyx, dpro, dcf, 0, _ptr(ws), _ptr(dw), p.in_c,
                       _ptr(db))
    _call(L.bnff_conv_wgrad, C.byref(a), what=f"wgrad {p.name}")
    return dw, db


def _dgrad(dy, pc, dx_shape_like, epi=_lib.DG_PLAIN, x=None, x_tables=None, stat_part=None,
           dy_pkg=None):
    p = pc.p
    dx = torch.empty(tuple(dx_shape_like.shape), dtype=dx_shape_like.dtype,
                     device=dx_shape_like.device)
    if dy_pkg is None:
        dyv, dyx, dpro, dcf = view(dy), view(dy), _lib.PRO_NONE, coef()
    else:
        dyv, dyx, dpro, dcf = view(dy_pkg[0]), view(dy_pkg[1]), _lib.PRO_BN_DX, coef(*dy_pkg[2])
    xv = view(x) if x is not None else view(dx)
    a = _lib.DgradArgs(_dcode(dx), p.kh, p.kw, p.stride, p.pad, dyv, dyx, dpro, dcf, view(dx), xv,
                       _ptr(pc.wt), epi, coef(*(x_tables or ())), _ptr(stat_part), _ptr(pc.wd))
    _call(_L().bnff_conv_dgrad, C.byref(a), what=f"dgrad {p.name}")
    return dx


def conv2d_bwd(x, dy, p, clip_input: bool = False):
    """ops.conv2d_bwd (ops.py:178-204) -> (dx, dw, dbias); clip_input masks dx by x>0."""
    pc = _packed(p, x)
    n, h, w, _ = x.shape
    oh, ow = pc.p.out_hw(h, w)
    if tuple(dy.shape) != (n, oh, ow, pc.p.out_c):
        raise ShapeError(f"{pc.p.name}: dy shape {tuple(dy.shape)} != {(n, oh, ow, pc.p.out_c)}")
    dx = _dgrad(dy, pc, x, _lib.DG_CLIP if clip_input else _lib.DG_PLAIN, x)
    dw, db = _wgrad(x, dy, pc, _lib.PRO_RELU if clip_input else _lib.PRO_NONE)
    return dx, dw, db


def _sums(mode, x, dy=None, cf=None):
    L = _L()
    src = x if mode == 0 else dy
    tiles = L.bnff_sum_tiles(_pixels(src))
    part = torch.empty((tiles, 2, src.shape[3]), dtype=torch.float64, device=src.device)
    _call(L.bnff_channel_sums, _dcode(src), mode, view(x), view(dy if dy is not None else x),
          cf or coef(), _ptr(part), what="channel_sums")
    return part, tiles


def bn_stats_onepass(x) -> DevStats:
    """ops.bn_stats_onepass (ops.py:231-237): one sweep, float64 sums."""
    part, tiles = _sums(0, x)
    st = _new_stats(x.shape[3], _pixels(x), x.device)
    _finalize(part, tiles, st)
    return st


def bn_stats_twopass(x) -> DevStats:
    """ops.bn_stats_twopass (ops.py:212-228): mean sweep + centred-variance sweep."""
    st = bn_stats_onepass(x)
    L = _L()
    tiles = L.bnff_sum_tiles(_pixels(x))
    part = torch.empty((tiles, 2, x.shape[3]), dtype=torch.float64, device=x.device)
    _call(L.bnff_centered_var, _dcode(x), view(x), _ptr(st.mean), _ptr(part), what="centered_var")
    _call(L.bnff_var_finalize, _ptr(part), tiles, x.shape[3], st.count, _ptr(st.var),
          what="var_finalize")
    return st


def _tables(st: DevStats, bn: BNParams, device):
    c = st.mean.shape[0]
    gam = torch.as_tensor(bn.gamma, dtype=torch.float32).to(device)
    bet = torch.as_tensor(bn.beta, dtype=torch.float32).to(device)
    t = [torch.empty(c, dtype=torch.float32, device=device) for _ in range(4)]
    _call(_L().bnff_bn_coeffs, c, _ptr(st.mean), _ptr(st.var), _ptr(gam), _ptr(bet),
          C.c_float(bn.eps), *(_ptr(v) for v in t), what="bn_coeffs")
    return t  # mean32, scale32, beta32, inv32


def bn_fwd(x, stats: DevStats, p: BNParams, out=None, relu: bool = False):
    """ops.bn_fwd (ops.py:240-254): (x-mean)*(gamma*inv)+beta, factors in storage precision."""
    c = x.shape[3]
    if stats.mean.shape[0] != c or p.channels != c:
        raise ShapeError(f"{p.name}: stats/params for {stats.mean.shape[0]}/{p.channels} "
                         f"channels, input has {c}")
    m32, s32, b32, _ = _tables(stats, p, x.device)
    out = torch.empty_like(x) if out is None else out
    _call(_L().bnff_bn_apply, _dcode(x), view(x), view(out), coef(m32, s32, b32), int(relu),
          what="bn_apply")
    return out


def _dx_table(part, tiles, stats: DevStats, gamma, eps, device):
    c = stats.mean.shape[0]
    f = lambda: torch.empty(c, dtype=torch.float32, device=device)  # noqa: E731
    k1, k2, g, m32, i32, dg32, db32 = (f() for _ in range(7))
    dg64 = torch.empty(c, dtype=torch.float64, device=device)
    db64 = torch.empty(c, dtype=torch.float64, device=device)
    gam = torch.as_tensor(gamma, dtype=torch.float32).to(device)
    _call(_L().bnff_dx_coeffs, c, _ptr(part), tiles, stats.count, _ptr(stats.mean), _ptr(stats.var),
          _ptr(gam), C.c_float(eps), _ptr(dg64), _ptr(db64), _ptr(k1), _ptr(k2), _ptr(g), _ptr(m32),
          _ptr(i32), _ptr(dg32), _ptr(db32), what="dx_coeffs")
    return (m32, i32, k1, k2, g), dg64, db64


def _resolve(dt1, x, table):
    out = torch.empty_like(dt1)
    term = _lib.GradTerm(view(dt1), view(x), 1, coef(*table))
    _call(_L().bnff_grad_sum, _dcode(dt1), view(out), 0, C.byref(term), 1, what="bn_dx")
    return out


def bn_bwd(x, dy, stats: DevStats, p: BNParams):
    """ops.bn_bwd (ops.py:257-280) -> (dx, dgamma, dbeta): reduction sweep + dx sweep."""
    if tuple(x.shape) != tuple(dy.shape):
        raise ShapeError(f"{p.name}: dy shape {tuple(dy.shape)} != x shape {tuple(x.shape)}")
    m32, _, _, i32 = _tables(stats, p, x.device)
    part, tiles = _sums(1, x, dy, coef(m32, i32))
    table, dg64, db64 = _dx_table(part, tiles, stats, p.gamma, p.eps, x.device)
    return _resolve(dy, x, table), dg64.float(), db64.float()


def bn_dx_from_sums(x, dy, stats: DevStats, p: BNParams, dgamma, dbeta, out=None):
    """ops.bn_dx_from_sums (ops.py:283-298): the dx half given (dgamma, dbeta)."""
    c = x.shape[3]
    m = stats.count
    dev = x.device
    inv = stats.inv_std(p.eps)
    table = (stats.mean.float(), inv.float(),
             (torch.as_tensor(dbeta, dtype=torch.float64, device=dev) / m).float(),
             (torch.as_tensor(dgamma, dtype=torch.float64, device=dev) / m).float(),
             (torch.as_tensor(p.gamma, dtype=torch.float64, device=dev) * inv).float())
    if any(t.shape[0] != c for t in table):
        raise ShapeError("bn_dx_from_sums: channel mismatch")
    res = _resolve(dy, x, table)
    if out is not None:
        out.copy_(res)
        return out
    return res


def relu_fwd(x, out=None):
    out = torch.empty_like(x) if out is None else out
    _call(_L().bnff_relu_fwd, _dcode(x), view(x), view(out), what="relu_fwd")
    return out


def relu_bwd(x, dy):
    if tuple(x.shape) != tuple(dy.shape):
        raise ShapeError(f"relu_bwd: shape mismatch {tuple(x.shape)} vs {tuple(dy.shape)}")
    dx = torch.empty_like(x)
    _call(_L().bnff_relu_bwd, _dcode(x), view(x), view(dy), view(dx), what="relu_bwd")
    return dx


def avgpool_fwd(x, k: int, stride: int = None, out=None, emit_stats: bool = False):
    stride = k if stride is None else stride
    if stride != k:
        raise ShapeError(f"avgpool windows must be non-overlapping (stride {stride} != k {k})")
    n, h, w, c = x.shape
    if h // k < 1 or w // k < 1:
        raise ShapeError(f"avgpool: window {k} larger than input {h}x{w}")
    out = torch.empty((n, h // k, w // k, c), dtype=x.dtype, device=x.device) if out is None else out
    part, tiles = None, 0
    if emit_stats:
        tiles = _L().bnff_sum_tiles(_pixels(out))
        part = torch.empty((tiles, 2, c), dtype=torch.float64, device=x.device)
    _call(_L().bnff_avgpool_fwd, _dcode(x), view(x), view(out), k, _ptr(part), what="avgpool")
    if emit_stats:
        st = _new_stats(c, _pixels(out), x.device)
        _finalize(part, tiles, st)
        return out, st
    return out


def avgpool_bwd(dy, in_shape_nhwc, k: int):
    dx = torch.empty(tuple(in_shape_nhwc), dtype=dy.dtype, device=dy.device)
    _call(_L().bnff_avgpool_bwd, _dcode(dy), view(dy), view(dx), k, what="avgpool_bwd")
    return dx


# ---------------------------------------------------------------------------
# fused.py equivalents
# ---------------------------------------------------------------------------


def fused_conv_stats_fwd(x, conv, out, budget: int = DEFAULT_BUDGET, workers: int = 1) -> DevStats:
    """fused.py:79-100 -- conv with per-channel sum/sum^2 in the epilogue (sub-BN1 + MVF)."""
    pc = _packed(conv, x)
    if x.shape[3] < pc.p.in_c:
        raise ShapeError(f"{pc.p.name}: input has {x.shape[3]} channels, expected {pc.p.in_c}")
    out = _out_like(x, pc.p, out)
    mt = _L().bnff_stat_rows()
    part = torch.zeros((mt, 2, pc.p.out_c), dtype=torch.float64, device=x.device)
    _fprop(x, pc, out, _lib.PRO_NONE, None, part)
    st = _new_stats(pc.p.out_c, _pixels(out), x.device)
    _finalize(part, mt, st)
    return st


def fused_norm_relu_conv_fwd(x, stats: DevStats, bn: BNParams, conv, out, saved_out=None,
                             budget: int = DEFAULT_BUDGET, workers: int = 1,
                             emit_stats: bool = False):
    """fused.py:103-154 -- normalize+ReLU in the conv's operand prologue; optional output
    statistics in the epilogue.  ``saved_out`` (post-ReLU input) is written only when given."""
    if stats is None:
        raise StateError(f"{getattr(conv, 'name', 'conv')}: no statistics available for "
                         f"normalization input")
    pc = _packed(conv, x)
    c = x.shape[3]
    if stats.mean.shape[0] != c or bn.channels != c:
        raise ShapeError(f"{pc.p.name}: stats/bn cover {stats.mean.shape[0]}/{bn.channels} "
                         f"channels, input has {c}")
    tb = _tables(stats, bn, x.device)
    if saved_out is not None:
        _call(_L().bnff_bn_apply, _dcode(x), view(x), view(saved_out), coef(tb[0], tb[1], tb[2]),
              1, what="saved_postrelu")
    out = _out_like(x, pc.p, out)
    part, mt = None, 0
    if emit_stats:
        mt = _L().bnff_stat_rows()
        part = torch.zeros((mt, 2, pc.p.out_c), dtype=torch.float64, device=x.device)
    _fprop(x, pc, out, _lib.PRO_BN_RELU, tb[:3], part)
    if emit_stats:
        st = _new_stats(pc.p.out_c, _pixels(out), x.device)
        _finalize(part, mt, st)
        return st
    return None


def fused_nrc_bwd(x, saved_postrelu, stats: DevStats, bn: BNParams, conv, dy, dy_pkg=None,
                  return_table: bool = False):
    """fused.py:157-200 -> (dt1, dw, dbias, dgamma64, dbeta64), the reference's 5-tuple.

    The ReLU mask and the wgrad operand are recomputed from x (``saved_postrelu``
    may be None); dgamma/dbeta ride in the dgrad epilogue.  ``dy_pkg`` =
    (dt1_next, x_next, table) applies an incoming deferred BN dx inline.
    ``return_table=True`` appends the device dx-coefficient table (mean, inv, k1, k2, g)
    that fused_conv_stats_bwd(table=...) consumes without recomputing it."""
    pc = _packed(conv, x)
    tb = _tables(stats, bn, x.device)
    n, h, w, c = x.shape
    mt = _L().bnff_stat_rows()
    part = torch.zeros((mt, 2, c), dtype=torch.float64, device=x.device)
    dt1 = _dgrad(dy, pc, x, _lib.DG_NRC, x, (tb[0], tb[1], tb[2], tb[3]), part, dy_pkg)
    dw, db = _wgrad(x, dy, pc, _lib.PRO_BN_RELU, tb[:3], dy_pkg)
    table, dg64, db64 = _dx_table(part, mt, stats, bn.gamma, bn.eps, x.device)
    if return_table:
        return dt1, dw, db, dg64, db64, table
    return dt1, dw, db, dg64, db64


def fused_conv_stats_bwd(x_own_out, saved_in, conv, dt1, dgamma, dbeta, stats: DevStats,
                         bn_gamma, bn_eps, clip_input=False, table=None):
    """fused.py:203-219 -- deferred BN dx applied inside the conv dgrad/wgrad prologues."""
    pc = _packed(conv, saved_in)
    if table is None:
        bn = BNParams(gamma=bn_gamma, beta=bn_gamma * 0, eps=bn_eps)
        dev = saved_in.device
        inv = stats.inv_std(bn_eps)
        m = stats.count
        table = (stats.mean.float(), inv.float(),
                 (torch.as_tensor(dbeta, dtype=torch.float64, device=dev) / m).float(),
                 (torch.as_tensor(dgamma, dtype=torch.float64, device=dev) / m).float(),
                 (torch.as_tensor(bn.gamma, dtype=torch.float64, device=dev) * inv).float())
    pkg = (dt1, x_own_out, table)
    dx = _dgrad(dt1, pc, saved_in, _lib.DG_CLIP if clip_input else _lib.DG_PLAIN, saved_in,
                dy_pkg=pkg)
    dw, db = _wgrad(saved_in, dt1, pc, _lib.PRO_RELU if clip_input else _lib.PRO_NONE, None, pkg)
    return dx, dw, db


def fused_split_bwd_bn_dx(branch_grads: list, resolve=None) -> torch.Tensor:
    """fused.py:222-230 -- sum of fan-out gradients; each branch is a tensor or a deferred
    package (dt1, x, table) resolved inline in the same sweep.  Any number of branches:
    the first launch writes the sum of up to two, later launches accumulate two more."""
    if len(branch_grads) < 1:
        raise ShapeError("fused_split_bwd_bn_dx: no branches")

    def term(b):
        if isinstance(b, tuple):
            return _lib.GradTerm(view(b[0]), view(b[1]), 1, coef(*b[2])), b[0]
        return _lib.GradTerm(view(b), view(b), 0, coef()), b

    first = term(branch_grads[0])[1]
    out = torch.empty(tuple(first.shape), dtype=first.dtype, device=first.device)
    for i in range(0, len(branch_grads), 2):
        chunk = [term(b)[0] for b in branch_grads[i:i + 2]]
        terms = (_lib.GradTerm * len(chunk))(*chunk)
        _call(_L().bnff_grad_sum, _dcode(first), view(out), 1 if i else 0, terms, len(chunk),
              what="split_bwd")
    return out
