"""Numpy restatement of the reference executor (TEST INFRASTRUCTURE).

Walks a ``paper_1807_01702_b200.graph.Graph`` (any fusion level) forward and
backward with the semantics of ``pkg/src/bnfuse/execute.py``: per-kind
handlers (execute.py:167-490), the ``DeferredBNGrad`` hand-off whose dx
transform is applied by the next gradient reader (execute.py:93-126), Concat
slicing of packages (execute.py:426-444) and Split summation with inline
resolution (execute.py:447-458).  Values are NCHW numpy arrays.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_1807_01702_b200 import graph as G
from paper_1807_01702_b200.errors import ShapeError, StateError
from paper_1807_01702_b200.params import ChannelStats, concat_stats

from . import ops


@dataclass
class Deferred:
    """Gradient at the normalized position awaiting BN's dx transform."""

    dt1: np.ndarray
    dgamma: np.ndarray
    dbeta: np.ndarray
    stats: ChannelStats
    gamma: np.ndarray
    eps: float
    x_slot: int
    c_lo: int
    c_hi: int

    def slice(self, lo, hi):
        return Deferred(self.dt1[:, lo:hi], self.dgamma[lo:hi], self.dbeta[lo:hi],
                        self.stats.slice(lo, hi), self.gamma[lo:hi], self.eps, self.x_slot,
                        self.c_lo + lo, self.c_lo + hi)

    def materialize(self, vals):
        x = vals[self.x_slot][:, self.c_lo: self.c_hi]
        return ops.bn_dx(x, self.dt1, self.stats, self.gamma, self.eps, self.dgamma, self.dbeta)


@dataclass
class Result:
    vals: dict
    node_stats: dict = field(default_factory=dict)

    def outputs(self, g):
        return {s: self.vals[s] for s in g.outputs}


def _get(vals, sid):
    try:
        return vals[sid]
    except KeyError:
        raise StateError(f"slot {sid} was never produced") from None


def forward(g: G.Graph, inputs) -> Result:
    if isinstance(inputs, np.ndarray):
        inputs = {g.inputs[0]: inputs}
    vals = dict(inputs)
    res = Result(vals)
    for node in g.nodes:
        try:
            _FWD[node.kind](node, g, res)
        except ShapeError as e:
            raise ShapeError(f"node {node.id} ({node.kind} {node.name}): {e}") from e
    return res


def _fwd_conv(node, g, r):
    at = node.attrs
    x = _get(r.vals, node.inputs[0])
    xe = ops.relu_fwd(x) if at.clip_input else x
    if node.kind == G.FUSED_CONV_STATS:
        y, st = ops.conv_stats_fwd(xe, at.conv)
        r.vals[node.outputs[1]] = st
    else:
        y = ops.conv_fwd(xe, at.conv)
    r.vals[node.outputs[0]] = y


def _fwd_bn(node, g, r):
    x = _get(r.vals, node.inputs[0])
    st = ops.stats_onepass(x) if node.attrs.onepass else ops.stats_twopass(x)
    r.node_stats[node.id] = st
    r.vals[node.outputs[0]] = ops.bn_apply(x, st, node.attrs.bn)


def _fwd_relu(node, g, r):
    r.vals[node.outputs[0]] = ops.relu_fwd(_get(r.vals, node.inputs[0]))


def _fwd_subbn1(node, g, r):
    r.vals[node.outputs[0]] = ops.stats_onepass(_get(r.vals, node.inputs[0]))


def _fwd_subbn2(node, g, r):
    x, st = _get(r.vals, node.inputs[0]), _get(r.vals, node.inputs[1])
    r.vals[node.outputs[0]] = ops.bn_apply(x, st, node.attrs.bn)


def _fwd_nrc(node, g, r):
    at = node.attrs
    x, st = _get(r.vals, node.inputs[0]), _get(r.vals, node.inputs[1])
    y, saved, ost = ops.norm_relu_conv_fwd(x, st, at.bn, at.conv, emit_stats=at.emit_stats)
    r.vals[node.outputs[0]] = y
    r.vals[node.outputs[1]] = saved
    if at.emit_stats:
        r.vals[node.outputs[2]] = ost


def _fwd_concat(node, g, r):
    r.vals[node.outputs[0]] = np.concatenate([_get(r.vals, s) for s in node.inputs], axis=1)


def _fwd_concat_stats(node, g, r):
    feat = [s for s in node.inputs if g.slots[s].kind == "feature"]
    stat = [s for s in node.inputs if g.slots[s].kind == "stats"]
    r.vals[node.outputs[0]] = np.concatenate([_get(r.vals, s) for s in feat], axis=1)
    r.vals[node.outputs[1]] = concat_stats([_get(r.vals, s) for s in stat])


def _fwd_split(node, g, r):
    x = _get(r.vals, node.inputs[0])
    for o in node.outputs:
        r.vals[o] = x


def _fwd_ews(node, g, r):
    a, b = _get(r.vals, node.inputs[0]), _get(r.vals, node.inputs[1])
    y = a.copy()
    if node.attrs.pad_channels:
        y[:, : b.shape[1]] += b
    else:
        if a.shape != b.shape:
            raise ShapeError(f"EltwiseSum operands {a.shape} vs {b.shape}")
        y += b
    r.vals[node.outputs[0]] = y


def _fwd_pool(node, g, r):
    y = ops.avgpool_fwd(_get(r.vals, node.inputs[0]), node.attrs.k)
    r.vals[node.outputs[0]] = y
    if node.attrs.emit_stats:
        r.vals[node.outputs[1]] = ops.stats_onepass(y)


_FWD = {
    G.CONV: _fwd_conv, G.FUSED_CONV_STATS: _fwd_conv, G.BN: _fwd_bn, G.RELU: _fwd_relu,
    G.SUBBN1: _fwd_subbn1, G.SUBBN2: _fwd_subbn2, G.FUSED_NRC: _fwd_nrc,
    G.CONCAT: _fwd_concat, G.FUSED_CONCAT_STATS: _fwd_concat_stats, G.SPLIT: _fwd_split,
    G.EWS: _fwd_ews, G.POOL: _fwd_pool,
}

# ---------------------------------------------------------------------------
# backward
# ---------------------------------------------------------------------------


class Grads:
    def __init__(self):
        self.params: dict = {}
        self.inputs: dict = {}

    def add(self, name, g):
        self.params[name] = self.params[name] + g if name in self.params else g


def _resolve(gv, vals):
    return gv.materialize(vals) if isinstance(gv, Deferred) else gv


def _accum(grads, sid, gv):
    cur = grads.get(sid)
    if cur is None:
        grads[sid] = gv
        return
    if isinstance(cur, Deferred) or isinstance(gv, Deferred):
        raise StateError(f"slot {sid}: deferred gradient cannot be accumulated")
    grads[sid] = cur + gv


def _incoming(grads, sid, vals):
    gv = grads.get(sid)
    if gv is None:
        raise StateError(f"no gradient arrived at slot {sid}")
    return _resolve(gv, vals)


def backward(g: G.Graph, res: Result, loss_grads: dict) -> Grads:
    grads: dict = {}
    for sid in g.outputs:
        if sid not in loss_grads:
            raise ShapeError(f"loss gradient missing for output slot {sid}")
        grads[sid] = np.asarray(loss_grads[sid])
    out = Grads()
    for node in reversed(g.nodes):
        try:
            _BWD[node.kind](node, g, res, grads, out)
        except ShapeError as e:
            raise ShapeError(f"node {node.id} ({node.kind} {node.name}): {e}") from e
    for sid in g.inputs:
        gv = grads.get(sid)
        out.inputs[sid] = _resolve(gv, res.vals) if gv is not None else None
    return out


def _bwd_conv(node, g, r, grads, out):
    at = node.attrs
    raw = grads.get(node.outputs[0])
    x = _get(r.vals, node.inputs[0])
    if isinstance(raw, Deferred):
        y = _get(r.vals, raw.x_slot)[:, raw.c_lo: raw.c_hi]
        dx, dw, db = ops.conv_stats_bwd(y, x, at.conv, raw.dt1, raw.dgamma, raw.dbeta, raw.stats,
                                        raw.gamma, raw.eps, clip_input=at.clip_input)
    else:
        dy = _incoming(grads, node.outputs[0], r.vals)
        dx, dw, db = ops.conv_bwd(ops.relu_fwd(x) if at.clip_input else x, dy, at.conv)
        if at.clip_input:
            dx = np.where(x > 0, dx, x.dtype.type(0))
    out.add(f"{at.conv.name}.weight", dw)
    out.add(f"{at.conv.name}.bias", db)
    _accum(grads, node.inputs[0], dx)


def _bwd_bn(node, g, r, grads, out):
    st = r.node_stats.get(node.id)
    if st is None:
        raise StateError(f"node {node.id}: backward before forward")
    dy = _incoming(grads, node.outputs[0], r.vals)
    dx, dg, db = ops.bn_bwd(_get(r.vals, node.inputs[0]), dy, st, node.attrs.bn)
    out.add(f"{node.attrs.bn.name}.gamma", dg)
    out.add(f"{node.attrs.bn.name}.beta", db)
    _accum(grads, node.inputs[0], dx)


def _bwd_relu(node, g, r, grads, out):
    dy = _incoming(grads, node.outputs[0], r.vals)
    _accum(grads, node.inputs[0], ops.relu_bwd(_get(r.vals, node.inputs[0]), dy))


def _bwd_subbn1(node, g, r, grads, out):
    if node.attrs.defer_backward:
        return
    pending = grads.get(node.inputs[0])
    if isinstance(pending, Deferred):
        grads[node.inputs[0]] = pending.materialize(r.vals)


def _bwd_subbn2(node, g, r, grads, out):
    at = node.attrs
    dy = _incoming(grads, node.outputs[0], r.vals)
    x, st = _get(r.vals, node.inputs[0]), _get(r.vals, node.inputs[1])
    xh = ops.xhat(x, st, at.bn.eps)
    dbeta = dy.sum(axis=(0, 2, 3), dtype=np.float64)
    dgamma = (dy * xh).sum(axis=(0, 2, 3), dtype=np.float64)
    out.add(f"{at.bn.name}.gamma", dgamma.astype(x.dtype))
    out.add(f"{at.bn.name}.beta", dbeta.astype(x.dtype))
    _accum(grads, node.inputs[0],
           Deferred(dy, dgamma, dbeta, st, at.bn.gamma, at.bn.eps, node.inputs[0], 0, x.shape[1]))


def _bwd_nrc(node, g, r, grads, out):
    at = node.attrs
    dy = _incoming(grads, node.outputs[0], r.vals)
    x, st = _get(r.vals, node.inputs[0]), _get(r.vals, node.inputs[1])
    saved = _get(r.vals, node.outputs[1])
    dt1, dw, db, dgamma, dbeta = ops.nrc_bwd(x, saved, st, at.bn, at.conv, dy)
    out.add(f"{at.conv.name}.weight", dw)
    out.add(f"{at.conv.name}.bias", db)
    out.add(f"{at.bn.name}.gamma", dgamma.astype(x.dtype))
    out.add(f"{at.bn.name}.beta", dbeta.astype(x.dtype))
    _accum(grads, node.inputs[0],
           Deferred(dt1, dgamma, dbeta, st, at.bn.gamma, at.bn.eps, node.inputs[0], 0, x.shape[1]))


def _bwd_concat(node, g, r, grads, out):
    dy = grads.get(node.outputs[0])
    if dy is None:
        raise StateError(f"no gradient arrived at concat output {node.outputs[0]}")
    off = 0
    for s in (s for s in node.inputs if g.slots[s].kind == "feature"):
        c = g.slots[s].shape[1]
        _accum(grads, s, dy.slice(off, off + c) if isinstance(dy, Deferred)
               else dy[:, off: off + c])
        off += c


def _bwd_split(node, g, r, grads, out):
    total = None
    for o in node.outputs:
        if grads.get(o) is None:
            raise StateError(f"no gradient arrived at split branch {o}")
        a = _resolve(grads[o], r.vals)
        total = a.copy() if total is None else total + a
    _accum(grads, node.inputs[0], total)


def _bwd_ews(node, g, r, grads, out):
    dy = _incoming(grads, node.outputs[0], r.vals)
    _accum(grads, node.inputs[0], dy)
    cb = g.slots[node.inputs[1]].shape[1]
    _accum(grads, node.inputs[1], dy[:, :cb] if node.attrs.pad_channels else dy)


def _bwd_pool(node, g, r, grads, out):
    dy = _incoming(grads, node.outputs[0], r.vals)
    _accum(grads, node.inputs[0], ops.avgpool_bwd(dy, g.slots[node.inputs[0]].shape, node.attrs.k))


_BWD = {
    G.CONV: _bwd_conv, G.FUSED_CONV_STATS: _bwd_conv, G.BN: _bwd_bn, G.RELU: _bwd_relu,
    G.SUBBN1: _bwd_subbn1, G.SUBBN2: _bwd_subbn2, G.FUSED_NRC: _bwd_nrc,
    G.CONCAT: _bwd_concat, G.FUSED_CONCAT_STATS: _bwd_concat, G.SPLIT: _bwd_split,
    G.EWS: _bwd_ews, G.POOL: _bwd_pool,
}


def sgd(params: dict, grads: dict, lr: float) -> dict:
    """Post-step weights w - lr*g (no reference optimizer exists)."""
    return {k: (v - np.asarray(lr, v.dtype) * grads[k].astype(v.dtype)) if k in grads else v
            for k, v in params.items()}


def train_step(g: G.Graph, x: np.ndarray, dy_out: np.ndarray):
    """One forward + backward on the oracle; returns (Result, Grads)."""
    res = forward(g, {g.inputs[0]: x})
    return res, backward(g, res, {g.outputs[0]: dy_out})
