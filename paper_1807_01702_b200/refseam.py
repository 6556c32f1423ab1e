"""The drop-in at the reference's own seam.

Two ways a user of the reference (``bnfuse``) switches to the device path:

1. **Executor entry points with the reference signatures** --
   ``forward(g, inputs, mode="train", ctx=None) -> Activations`` and
   ``backward(g, acts, loss_grads, ctx=None) -> GradBundle`` (``execute.py:513-558``).
   The graph (ours or the reference's: node kinds, slots, ConvParams/BNParams are
   duck-typed) is compiled once into an ``Engine`` (cached on the graph object) and
   run on the device; activations and gradients come back as host NCHW arrays keyed
   exactly like the reference's.

2. **Handler installation** -- ``install(execute)`` rebinds the reference executor's
   own handler functions (``_FWD_HANDLERS`` / ``_BWD_HANDLERS``, ``execute.py:294-307,
   477-490``) to kernel shims with the reference's function names and argument order
   (``fused.py:79-230``, ``ops.py:151-454``) that run every compute call on the
   device kernels of ``kernels.py``.  The reference's handler logic -- ledger records,
   deferred BN-gradient routing, view-concat buffers -- is untouched: only the
   ``fused`` / ``ops`` modules those handlers call (and ``_resolve`` /
   ``_incoming``, which materialise deferred packages) are swapped.
   ``uninstall(execute)`` restores the originals.

The shims take and return the reference's host arrays (NCHW numpy, fp32) and its
``ChannelStats``; each call copies its operands to the device, launches the sm_100a
kernels and copies the results back -- a compatibility seam, not the fast path (the
fast path is option 1 / ``Engine``, which keeps everything resident).
"""

from __future__ import annotations

import types

import numpy as np
import torch

from . import kernels as K

F64 = torch.float64


# ---------------------------------------------------------------------------
# host <-> device conversions.  The device kernels take 16-byte channel rows (fp32:
# multiples of 4); other widths (DenseNet-BC growth 12 -> 30-channel transitions) are
# zero-padded on the way in and stripped on the way out: padded input channels are
# zero, padded BN channels have gamma = beta = 0, padded weight rows/columns are zero,
# so the real channels compute exactly what the unpadded op computes.
# ---------------------------------------------------------------------------
def _p4(c: int) -> int:
    return (c + 3) // 4 * 4


def _dev(a) -> torch.Tensor:
    a = np.asarray(a, np.float32)
    c = a.shape[1]
    if c % 4:
        a = np.concatenate([a, np.zeros((a.shape[0], _p4(c) - c) + a.shape[2:], np.float32)], axis=1)
    return torch.from_numpy(np.ascontiguousarray(a.transpose(0, 2, 3, 1))).to("cuda")


def _host(t: torch.Tensor, c: int | None = None) -> np.ndarray:
    a = t.float().permute(0, 3, 1, 2).contiguous().cpu().numpy()
    return a if c is None else np.ascontiguousarray(a[:, :c])


def _put(out, arr):
    if out is None:
        return arr
    np.copyto(out, arr)
    return out


def _pvec(v, n, dtype=np.float64):
    v = np.asarray(v, dtype)
    return v if v.shape[0] == n else np.concatenate([v, np.zeros(n - v.shape[0], dtype)])


def _pconv(p):
    """ConvParams with in/out channels padded to multiples of 4 (zero weights / bias)."""
    ci, co = _p4(p.in_c), _p4(p.out_c)
    if ci == p.in_c and co == p.out_c:
        return p
    from .params import ConvParams
    w = np.zeros((co, ci, p.kh, p.kw), np.float32)
    w[: p.out_c, : p.in_c] = p.weights
    return ConvParams(ci, co, p.kh, p.kw, p.stride, p.pad, w, _pvec(p.bias, co, np.float32), p.name)


def _pbn(bn, cp):
    from .params import BNParams
    return BNParams(_pvec(bn.gamma, cp, np.float32), _pvec(bn.beta, cp, np.float32), bn.eps, bn.name)


def _dstats(cs, cp=None) -> K.DevStats:
    c = np.asarray(cs.mean).shape[0]
    cp = cp or _p4(c)
    d = lambda v: torch.as_tensor(_pvec(v, cp), dtype=F64, device="cuda")  # noqa: E731
    return K.DevStats(d(cs.sum_x), d(cs.sum_x2), int(cs.count), d(cs.mean), d(cs.var))


def _hstats(ds: K.DevStats, CS, c=None):
    h = lambda t: t.cpu().numpy().astype(np.float64)[:c]  # noqa: E731
    return CS(sum_x=h(ds.sum_x), sum_x2=h(ds.sum_x2), count=int(ds.count), mean=h(ds.mean),
              var=h(ds.var))


# ---------------------------------------------------------------------------
# kernel shims with the reference names (ops.py / fused.py)
# ---------------------------------------------------------------------------
def make_shims(ops_mod, fused_mod):
    """(ops, fused) namespaces: the reference modules with every compute function
    replaced by a device-kernel shim of the same name and signature."""
    CS = ops_mod.ChannelStats
    o = types.SimpleNamespace(**{k: v for k, v in vars(ops_mod).items() if not k.startswith("__")})
    f = types.SimpleNamespace(**{k: v for k, v in vars(fused_mod).items() if not k.startswith("__")})

    def _np(t, c):
        return t.cpu().numpy()[:c]

    def conv2d_fwd(x, p, out=None):  # ops.py:151
        return _put(out, _host(K.conv2d_fwd(_dev(x), _pconv(p)), p.out_c))

    def conv2d_bwd(x, dy, p):  # ops.py:178
        dx, dw, db = K.conv2d_bwd(_dev(x), _dev(dy), _pconv(p))
        return (_host(dx, p.in_c), dw.cpu().numpy()[: p.out_c, : p.in_c].copy(), _np(db, p.out_c))

    def bn_stats_twopass(x):  # ops.py:212
        return _hstats(K.bn_stats_twopass(_dev(x)), CS, x.shape[1])

    def bn_stats_onepass(x):  # ops.py:231
        return _hstats(K.bn_stats_onepass(_dev(x)), CS, x.shape[1])

    def bn_fwd(x, stats, p, out=None):  # ops.py:240
        c = x.shape[1]
        return _put(out, _host(K.bn_fwd(_dev(x), _dstats(stats), _pbn(p, _p4(c))), c))

    def bn_bwd(x, dy, stats, p):  # ops.py:257
        c = x.shape[1]
        dx, dg, db = K.bn_bwd(_dev(x), _dev(dy), _dstats(stats), _pbn(p, _p4(c)))
        return _host(dx, c), _np(dg, c), _np(db, c)

    def bn_dx_from_sums(x, dy, stats, p, dgamma, dbeta, out=None):  # ops.py:283
        c, cp = x.shape[1], _p4(x.shape[1])
        r = K.bn_dx_from_sums(_dev(x), _dev(dy), _dstats(stats), _pbn(p, cp), _pvec(dgamma, cp),
                              _pvec(dbeta, cp))
        return _put(out, _host(r, c))

    def relu_fwd(x, out=None):  # ops.py:306
        return _put(out, _host(K.relu_fwd(_dev(x)), x.shape[1]))

    def relu_bwd(x, dy):  # ops.py:314
        return _host(K.relu_bwd(_dev(x), _dev(dy)), x.shape[1])

    def avgpool_fwd(x, k, stride=None, out=None):  # ops.py:428
        return _put(out, _host(K.avgpool_fwd(_dev(x), k, stride), x.shape[1]))

    def avgpool_bwd(dy, in_shape, k):  # ops.py:446
        n, c, h, w = in_shape
        return _host(K.avgpool_bwd(_dev(dy), (n, h, w, _p4(c)), k), c)

    def fused_conv_stats_fwd(x, conv, out, budget=None, workers=1):  # fused.py:79
        n, _, h, w = x.shape
        oh, ow = conv.out_hw(h, w)
        pc = _pconv(conv)
        yd = torch.empty((n, oh, ow, pc.out_c), dtype=torch.float32, device="cuda")
        st = K.fused_conv_stats_fwd(_dev(x), pc, yd)
        _put(out, _host(yd, conv.out_c))
        return _hstats(st, CS, conv.out_c)

    def fused_norm_relu_conv_fwd(x, stats, bn, conv, out, saved_out, budget=None, workers=1,
                                 emit_stats=False):  # fused.py:103
        n, c, h, w = x.shape
        oh, ow = conv.out_hw(h, w)
        pc = _pconv(conv)
        xd = _dev(x)
        yd = torch.empty((n, oh, ow, pc.out_c), dtype=torch.float32, device="cuda")
        sd = torch.empty_like(xd) if saved_out is not None else None
        st = K.fused_norm_relu_conv_fwd(xd, _dstats(stats), _pbn(bn, _p4(c)), pc, yd, sd,
                                        emit_stats=emit_stats)
        _put(out, _host(yd, conv.out_c))
        if saved_out is not None:
            _put(saved_out, _host(sd, c))
        return _hstats(st, CS, conv.out_c) if emit_stats else None

    def fused_nrc_bwd(x, saved_postrelu, stats, bn, conv, dy):  # fused.py:157
        c = x.shape[1]
        dt1, dw, db, dg, dbt = K.fused_nrc_bwd(_dev(x), None, _dstats(stats), _pbn(bn, _p4(c)),
                                               _pconv(conv), _dev(dy))
        return (_host(dt1, c), dw.cpu().numpy()[: conv.out_c, :c].copy(), _np(db, conv.out_c),
                _np(dg, c), _np(dbt, c))

    def fused_conv_stats_bwd(x_own_out, saved_in, conv, dt1, dgamma, dbeta, stats, bn_gamma,
                             bn_eps, clip_input=False):  # fused.py:203
        co = _p4(conv.out_c)
        dx, dw, db = K.fused_conv_stats_bwd(_dev(x_own_out), _dev(saved_in), _pconv(conv), _dev(dt1),
                                            _pvec(dgamma, co), _pvec(dbeta, co), _dstats(stats, co),
                                            _pvec(bn_gamma, co, np.float32), bn_eps,
                                            clip_input=clip_input)
        return (_host(dx, conv.in_c), dw.cpu().numpy()[: conv.out_c, : conv.in_c].copy(),
                _np(db, conv.out_c))

    def fused_split_bwd_bn_dx(branch_grads, resolve):  # fused.py:222
        arrs = [np.asarray(resolve(b)) for b in branch_grads]
        return _host(K.fused_split_bwd_bn_dx([_dev(a) for a in arrs]), arrs[0].shape[1])

    for fn in (conv2d_fwd, conv2d_bwd, bn_stats_twopass, bn_stats_onepass, bn_fwd, bn_bwd,
               bn_dx_from_sums, relu_fwd, relu_bwd, avgpool_fwd, avgpool_bwd):
        setattr(o, fn.__name__, fn)
    for fn in (fused_conv_stats_fwd, fused_norm_relu_conv_fwd, fused_nrc_bwd, fused_conv_stats_bwd,
               fused_split_bwd_bn_dx):
        setattr(f, fn.__name__, fn)
    f.bn_dx_from_sums = bn_dx_from_sums
    return o, f


# ---------------------------------------------------------------------------
# handler installation into the reference executor
# ---------------------------------------------------------------------------
_SAVED = "__bnff_saved_handlers__"


def install(execute) -> None:
    """Point the reference executor's handler tables at device-backed handlers: the
    reference's own handler code, rebound to the kernel shims."""
    if getattr(execute, _SAVED, None) is not None:
        return
    ops_s, fused_s = make_shims(execute.ops, execute.fused)
    glb = dict(vars(execute))
    glb["ops"] = ops_s
    glb["fused"] = fused_s
    DBG = execute.DeferredBNGrad
    BNP = execute.BNParams

    def _resolve(g, acts):  # execute.py:141 / DeferredBNGrad.materialize on the device
        if isinstance(g, DBG):
            x = acts.get(g.x_slot)[:, g.c_lo:g.c_hi]
            bn = BNP(gamma=g.gamma, beta=np.zeros_like(g.gamma), eps=g.eps)
            return ops_s.bn_dx_from_sums(x, g.dt1, g.stats, bn, g.dgamma, g.dbeta)
        return g

    glb["_resolve"] = _resolve

    def rebind(fn):
        return types.FunctionType(fn.__code__, glb, fn.__name__, fn.__defaults__, fn.__closure__)

    glb["_incoming"] = rebind(execute._incoming)
    saved = (dict(execute._FWD_HANDLERS), dict(execute._BWD_HANDLERS))
    for table in (execute._FWD_HANDLERS, execute._BWD_HANDLERS):
        for kind, fn in list(table.items()):
            table[kind] = rebind(fn)
    setattr(execute, _SAVED, saved)


def uninstall(execute) -> None:
    saved = getattr(execute, _SAVED, None)
    if saved is None:
        return
    execute._FWD_HANDLERS.clear()
    execute._FWD_HANDLERS.update(saved[0])
    execute._BWD_HANDLERS.clear()
    execute._BWD_HANDLERS.update(saved[1])
    setattr(execute, _SAVED, None)


# ---------------------------------------------------------------------------
# executor entry points (execute.py:513-558) on the compiled device engine
# ---------------------------------------------------------------------------
class ExecCtx:
    """execute.ExecCtx: budget/workers/ledger/timings are accepted (tiling is the GPU
    grid); ``dtype`` selects the device precision ("f32" = the reference's arithmetic)."""

    def __init__(self, ledger=None, budget=None, workers=1, timings=None, dtype="f32"):
        self.ledger, self.budget, self.workers, self.timings = ledger, budget, workers, timings
        self.dtype = dtype


class Activations:
    """execute.Activations: slot-indexed values, read back from the device on access."""

    def __init__(self, g, eng):
        self.graph = g
        self.engine = eng
        self.vals: dict = {}
        for sid in g.inputs:
            self.vals[sid] = eng.input_host[sid]
        for sid in g.outputs:
            self.vals[sid] = eng.output(sid)[:, : g.slots[sid].shape[1]]

    def get(self, slot_id):
        if slot_id not in self.vals:
            from .errors import StateError
            eng = self.engine
            if slot_id in eng.acts:
                self.vals[slot_id] = eng.act(slot_id)
            elif slot_id in eng.stats:
                self.vals[slot_id] = eng.stats_of(slot_id)
            else:
                raise StateError(f"slot {slot_id} was never produced (missing saved activation?)")
        return self.vals[slot_id]

    def outputs(self):
        return {sid: self.vals[sid] for sid in self.graph.outputs}


class GradBundle:
    """execute.GradBundle: parameter gradients by name plus graph-input gradients."""

    def __init__(self, params=None, inputs=None):
        self.params = params or {}
        self.inputs = inputs or {}


def _arr(v) -> np.ndarray:
    """ndarray, or the reference's Tensor4D (its array is .data)."""
    if isinstance(v, np.ndarray):
        return v
    d = getattr(v, "data", None)
    return np.asarray(d if isinstance(d, np.ndarray) else v)


_CACHE_ATTR = "__bnff_engines__"


def _engine_for(g, dtype):
    from .engine import Engine
    cache = g.__dict__.setdefault(_CACHE_ATTR, {})
    eng = cache.get(dtype)
    if eng is None:
        eng = cache[dtype] = Engine(g, dtype=dtype, input_grad=True)
    return eng


def forward(g, inputs, mode: str = "train", ctx: ExecCtx | None = None) -> Activations:
    """execute.forward (execute.py:513-531) on the device."""
    from .errors import ShapeError, StateError
    if mode != "train":
        raise StateError(f"only train mode is supported, got {mode!r}")
    ctx = ctx or ExecCtx()
    if not isinstance(inputs, dict):  # one array / Tensor4D for a single-input graph
        if len(g.inputs) != 1:
            raise ShapeError(f"graph has {len(g.inputs)} inputs, got a single tensor")
        inputs = {g.inputs[0]: inputs}
    eng = _engine_for(g, getattr(ctx, "dtype", "f32"))
    eng.input_host = {}
    for sid, val in inputs.items():
        arr = _arr(val)
        if arr.shape != tuple(g.slots[sid].shape):
            raise ShapeError(f"input slot {sid}: shape {arr.shape} != declared {g.slots[sid].shape}")
        eng.input_host[sid] = arr
    eng.set_input(eng.input_host[g.inputs[0]])
    eng.forward()
    torch.cuda.synchronize()
    return Activations(g, eng)


def backward(g, acts: Activations, loss_grads: dict, ctx: ExecCtx | None = None) -> GradBundle:
    """execute.backward (execute.py:534-558) on the device."""
    from .errors import ShapeError
    eng = acts.engine
    for sid in g.outputs:
        if sid not in loss_grads:
            raise ShapeError(f"loss gradient missing for output slot {sid}")
        arr = _arr(loss_grads[sid])
        if arr.shape != tuple(g.slots[sid].shape):
            raise ShapeError(f"loss grad slot {sid}: shape {arr.shape} != {g.slots[sid].shape}")
    eng.set_loss_grad(_arr(loss_grads[g.outputs[0]]))
    eng.gflat.zero_()
    eng.backward()
    torch.cuda.synchronize()
    gb = GradBundle(params=eng.param_grads())
    for sid in g.inputs:
        gb.inputs[sid] = eng.input_grad_nchw(sid)
    return gb
