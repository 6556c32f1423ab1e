"""Device executor: runs a (rewritten) layer graph on B200 through libbnff.

Counterpart of the reference executor ``pkg/src/bnfuse/execute.py`` (forward
/ backward handler tables, Activations with shared block buffers, the
DeferredBNGrad hand-off).  The difference is *when* dispatch happens: the
graph is walked ONCE at construction time ("compile"), every handler emits
launch thunks with prebuilt C-ABI argument structs and statically placed
device buffers, and a training step is then a flat replay of those thunks on
one CUDA stream -- capturable as a single CUDA graph (``capture()``).

Device layout:
  * feature maps NHWC in bf16 or fp32; in view-concat mode every slot with a
    ``buffer`` annotation is a channel-offset view of one (N,H,W,C_total)
    block buffer, so Concat is free and producers write in place;
  * per-channel statistics float64, placed at the same channel offsets of a
    per-block stats array, so FusedConcatStats (concat_stats) is free too;
  * gradients NHWC; a deferred BN gradient is (dt1, x, coefficient table) and
    its dx transform runs inside whichever kernel reads it next (conv dgrad /
    wgrad operand prologue, or the Split gradient-sum kernel);
  * parameters: one flat fp32 master buffer in reference layout, one flat
    fp32 gradient buffer (NCCL all-reduce target), packed bf16/fp32 copies of
    the conv weights ([co][tap][ci] and [ci][tap][co]) refreshed after SGD.
  * FusedNormReluConv does not materialise ``saved_postrelu`` unless asked:
    backward recomputes relu(bn(x)) from x (bitwise identical in fp32 mode).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import graph as G
from .errors import ShapeError, StateError
from .params import ConvParams

# ---------------------------------------------------------------------------
# small helpers
# ---------------------------------------------------------------------------


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def view_of(t: torch.Tensor) -> _lib.View:
    """NHWC torch tensor (possibly a channel slice) -> bnff_view."""
    if t.dim() != 4 or t.stride(3) != 1:
        raise ShapeError(f"expected an NHWC view with unit channel stride, got {tuple(t.shape)}")
    n, h, w, c = t.shape
    # pixel stride; a contiguous tensor's is c even where size-1 dims carry arbitrary strides
    rs = c if t.is_contiguous() else t.stride(2)
    return _lib.View(_ptr(t), n, h, w, c, rs)


def coef_of(a=None, b=None, c=None, d=None, e=None) -> _lib.Coef:
    return _lib.Coef(_ptr(a), _ptr(b), _ptr(c), _ptr(d), _ptr(e))


def _nb(*ts) -> int:
    """bytes of the logical elements of NHWC views (channel slices count their own channels)."""
    return sum(int(t.numel()) * t.element_size() for t in ts if t is not None)


def _vec_of(dtype_code: int) -> int:
    return 8 if dtype_code == _lib.BF16 else 4


def _round_up(v: int, m: int) -> int:
    return (v + m - 1) // m * m


@dataclass
class Stats:
    """Device ChannelStats: float64 sums/moments (possibly views into a block array)."""
    sum: torch.Tensor
    sumsq: torch.Tensor
    mean: torch.Tensor
    var: torch.Tensor
    count: int

    def slice(self, lo, hi):
        return Stats(self.sum[lo:hi], self.sumsq[lo:hi], self.mean[lo:hi], self.var[lo:hi],
                     self.count)


@dataclass
class Deferred:
    """Device DeferredBNGrad (execute.py:93-126): gradient dt1 at the normalized
    position + per-channel table (mean, invstd, k1, k2, g) + the tensor x the
    normalization was applied to."""
    dt1: torch.Tensor
    x: torch.Tensor
    mean: torch.Tensor
    inv: torch.Tensor
    k1: torch.Tensor
    k2: torch.Tensor
    g: torch.Tensor
    affine: bool = False  # ICF fold: dt1 is the block gradient buffer, g = 1, (k1, k2) = (A, B)

    def slice(self, lo, hi):
        return Deferred(self.dt1[..., lo:hi], self.x[..., lo:hi], self.mean[lo:hi],
                        self.inv[lo:hi], self.k1[lo:hi], self.k2[lo:hi], self.g[lo:hi], self.affine)

    def coef(self):
        return coef_of(self.mean, self.inv, self.k1, self.k2, self.g)


@dataclass
class Plain:
    t: torch.Tensor


@dataclass
class Folded:
    """A split branch whose gradient was folded into the block gradient buffer by the
    consumer's dgrad epilogue (BNFF_DG_NRC_ACC/SET); the sibling branch carries it."""
    into: int  # the sibling slot now holding the combined gradient


# ---------------------------------------------------------------------------
# engine
# ---------------------------------------------------------------------------


class Engine:
    """Compile a graph for the device and run training steps on it.

    Parameters
    ----------
    g : Graph (any fusion level; ``fusion.plan`` output)
    dtype : "bf16" (tensor-core bf16, perf mode) or "f32" (3xTF32 parity mode)
    input_grad : also produce the gradient w.r.t. the graph input (reference
        ``GradBundle.inputs``); off for training throughput runs.
    save_postrelu : materialise FusedNormReluConv's saved post-ReLU tensor
        (reference schedule) instead of recomputing it in backward.
    """

    def __init__(self, g: G.Graph, dtype: str = "bf16", device="cuda", input_grad: bool = True,
                 save_postrelu: bool = False, lr: float = 0.0, use_window: bool = True,
                 sync_bn: bool = False, group=None, side_wgrad: bool = True, fold_icf: bool = True,
                 dp_buckets: bool | None = None, bucket_bytes: int = 4 << 20):
        self.L = _lib.lib()
        self.g = g
        self.dcode = _lib.BF16 if dtype == "bf16" else _lib.F32
        self.tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.vec = _vec_of(self.dcode)
        self.dev = torch.device(device)
        self.input_grad = input_grad
        self.save_postrelu = save_postrelu
        self.lr = float(lr)
        # SyncBN: BN statistics (and the dx reductions) over the global batch of all
        # data-parallel replicas -- 2*C float64 all-reduces per BN in each pass
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.sync_bn = bool(sync_bn) and self.world > 1
        if self.sync_bn and any(n.kind == G.BN and not n.attrs.onepass for n in g.nodes):
            raise _lib.UnsupportedError("sync_bn needs one-pass statistics (fusion level rcf+mvf or above)")
        self.use_window = bool(use_window)
        self.side_wgrad = bool(side_wgrad)
        # data parallel: the gradient SUM all-reduce is issued in reverse-layer buckets from
        # inside backward, on a communication stream, as soon as a bucket's gradients are
        # final (overlapping the rest of backward; captured in the step's CUDA graph)
        self.dp_buckets = (self.world > 1) if dp_buckets is None else bool(dp_buckets)
        self.bucket_bytes = int(bucket_bytes)
        self._comm = None
        self.buckets: list = []  # (lo, hi) ranges of the flat gradient, in issue order
        import os
        self.fuse_finalize = os.environ.get("BNFF_FUSE_FINALIZE", "1") != "0"
        self.fuse_nrp = os.environ.get("BNFF_FUSE_NRP", "1") != "0"  # sub-BN2 -> ReLU -> pool chains
        self.wide_fallback = os.environ.get("BNFF_WIDE_FALLBACK", "1") != "0"  # see _f_FusedNormReluConv
        self.col_strided = os.environ.get("BNFF_COL_STRIDED", "1") != "0"  # see _col_conv
        # CUDA stream priorities of the captured step (lower = higher priority): the side
        # stream carries the weight gradients, the capture stream the dgrad chain
        self.side_prio = int(os.environ.get("BNFF_SIDE_PRIO", "0"))
        self.main_prio = int(os.environ.get("BNFF_MAIN_PRIO", "0"))
        # a deferred BN dx at least this wide (channels) feeding a conv with more than two N
        # tiles of input channels is materialised once: every N tile of the dgrad (M tile of
        # the wgrad) would otherwise stream both wide operands (dt1 and the BN input) again
        # (0: never; C5 sweep / D121 / R50 A/B in DESIGN.md)
        self.wide_dx = int(os.environ.get("BNFF_WIDE_DX", "512"))
        # measurement only: launch every (idempotent) forward coefficient kernel N times, to price
        # one such launch on the critical path
        self.coef_reps = max(1, int(os.environ.get("BNFF_COEF_REPS", "1")))
        self._nrp: dict = {}  # ReLU / AvgPool node id -> the sub-BN2 node heading its fused chain
        self._wide_saved: dict = {}  # NRC node id -> materialised relu(bn(x)) (wide-N fallback)
        self._nrp_done: set = set()
        # ICF block-gradient fold: 1x1 NRC dgrads accumulate scale*dt1 straight
        # into the block gradient buffer; the per-channel remainder rides in (A, B) arrays
        self.fold_icf = bool(fold_icf)
        self.fold = {}  # block group -> dict(A, B, ones, m32, i32, started)
        self._side = None  # side stream of the weight-gradient launches
        self.wpacks = {}  # conv name -> (window fwd pack, window dgrad pack, conv)
        self.cols = {}  # conv name -> (1x1 conv over col, col buffer, dw scratch, kpad, strided)
        self.col_src = {}  # 1x1 col conv name -> (fp32 (co, kpad) weights, stem conv, kpad)
        self.use_shared = any(n.kind == G.FUSED_CONCAT_STATS or
                              (n.kind == G.CONCAT and not n.attrs.physical) for n in g.nodes)
        self.fold_icf = self.fold_icf and not self.sync_bn and any(
            n.kind == G.FUSED_CONCAT_STATS for n in g.nodes)
        self.fwd: list = []
        self.bwd: list = []
        self.opt: list = []
        self.launch_counts = {"fwd": 0, "bwd": 0, "opt": 0}
        self._cur = None
        self._keep: list = []  # ctypes structs referenced by thunks
        self._bufs: list = []  # device buffers referenced by thunks
        self._alloc_params()
        self._alloc_acts()
        self._compile_forward()
        self._compile_backward()
        self._compile_optimizer()
        self.graph_exec = None

    # ------------------------------------------------------------------ alloc
    # every device buffer is owned by the engine: thunks hold raw pointers, so a
    # buffer must never return to the caching allocator while the engine lives
    def _empty(self, shape, dtype=None):
        t = torch.empty(shape, dtype=dtype or self.tdt, device=self.dev)
        self._bufs.append(t)
        return t

    def _zeros(self, shape, dtype=None):
        t = torch.zeros(shape, dtype=dtype or self.tdt, device=self.dev)
        self._bufs.append(t)
        return t

    def _alloc_params(self):
        g = self.g
        self.param_names = list(g.params)
        sizes = [int(np.asarray(g.params[k]).size) for k in self.param_names]
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        total = int(offs[-1])
        host = np.concatenate([np.asarray(g.params[k], np.float32).reshape(-1)
                               for k in self.param_names]) if total else np.zeros(0, np.float32)
        self.wflat = torch.from_numpy(host).to(self.dev)
        self.gflat = self._zeros((total,), torch.float32)
        self.poff = {k: (int(offs[i]), int(sizes[i])) for i, k in enumerate(self.param_names)}
        self.packs = {}  # conv name -> (wpack, wpack_t, cin_store)

    def param(self, name):
        o, n = self.poff[name]
        return self.wflat[o:o + n]

    def grad(self, name):
        o, n = self.poff[name]
        return self.gflat[o:o + n]

    def _store_c(self, c: int) -> int:
        return _round_up(c, self.vec)

    def _alloc_acts(self):
        g = self.g
        self.acts: dict = {}
        self.group_buf: dict = {}
        self.group_stats: dict = {}
        if self.use_shared:
            for grp, (ct, h, w) in g.buffer_groups.items():
                n = next(s.shape[0] for s in g.slots.values() if s.buffer and s.buffer[0] == grp)
                if ct % self.vec:
                    raise _lib.UnsupportedError(
                        f"block buffer {grp}: {ct} channels not a multiple of {self.vec}")
                self.group_buf[grp] = self._zeros((n, h, w, ct))
                self.group_stats[grp] = [self._zeros((ct,), torch.float64) for _ in range(4)]
        # graph input: channel-padded NHWC
        for sid in g.inputs:
            n, c, h, w = g.slots[sid].shape
            self.acts[sid] = self._zeros((n, h, w, self._store_c(c)))
        self.input_c = {sid: g.slots[sid].shape[1] for sid in g.inputs}

    def _feature(self, sid) -> torch.Tensor:
        """Device storage for a feature slot produced by a node (allocated on first use)."""
        if sid in self.acts:
            return self.acts[sid]
        s = self.g.slots[sid]
        n, c, h, w = s.shape
        if c % self.vec:
            raise _lib.UnsupportedError(
                f"slot {sid} ({s.name}): {c} channels not a multiple of {self.vec}")
        if self.use_shared and s.buffer is not None:
            grp, off = s.buffer
            t = self.group_buf[grp][..., off:off + c]
        else:
            t = self._empty((n, h, w, c))
        self.acts[sid] = t
        return t

    def _stats_for(self, feat_sid: int, c: int, count: int) -> Stats:
        s = self.g.slots[feat_sid]
        if self.use_shared and s.buffer is not None:
            grp, off = s.buffer
            arrs = [a[off:off + c] for a in self.group_stats[grp]]
        else:
            arrs = [self._zeros((c,), torch.float64) for _ in range(4)]
        return Stats(*arrs, count=count)

    # ------------------------------------------------------------ emit helpers
    def _emit(self, fn, *args, what="", nbytes=0, flops=0, launches=1, side=False):
        """Append a launch thunk calling fn(*args, stream).  ``nbytes``/``flops`` are the
        launch's ALGORITHMIC HBM bytes / FLOPs (each tensor counted once), used by the
        live roofline in bench.py."""
        check = _lib.check
        self._keep.append(args)

        def thunk(stream):
            check(fn(*args, stream), what)
        thunk.what = what
        thunk.kind = what.split(" ")[0]
        thunk.nbytes = int(nbytes)
        thunk.flops = int(flops)
        thunk.launches = launches  # kernels this C-ABI call launches
        thunk.side = bool(side)    # runs on the side stream (forked/joined by _run)
        thunk.node_id = getattr(self, "_cur_node", -1)  # the graph node that emitted it
        self._cur.append(thunk)

    def _emit_allreduce(self, *tensors, what="allreduce"):
        import torch.distributed as dist
        grp = self.group

        def _ar(stream, ts=tensors):
            for t in ts:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=grp)
        _ar.what, _ar.kind, _ar.nbytes, _ar.flops, _ar.launches = what, "allreduce", 0, 0, 0
        self._cur.append(_ar)

    def _emit_stats_finalize(self, part, tiles, c, count, st: Stats):
        if not self.sync_bn:
            # deferred: the next consumer's coefficient table launch finalizes it in the same
            # kernel (bnff_stats_finalize_coeffs); anything else flushes it first
            self._pending_fin.append((part, tiles, c, count, st))
            if not self.fuse_finalize:
                self._flush_pending()
            return
        # SyncBN: local float64 sums -> all-reduce -> moments over the global count
        self._emit(self.L.bnff_stats_finalize, _ptr(part), tiles, c, count, _ptr(st.sum),
                   _ptr(st.sumsq), None, None, what="stats_finalize")
        self._emit_allreduce(st.sum, st.sumsq, what="syncbn_fwd_allreduce")
        st.count = count * self.world
        self._emit(self.L.bnff_stats_from_sums, c, st.count, _ptr(st.sum), _ptr(st.sumsq),
                   _ptr(st.mean), _ptr(st.var), what="stats_finalize")

    def _pack(self, conv, cin_store, hw=None):
        key = conv.name
        if key not in self.packs:
            n = self.L.bnff_pack_size(self.dcode, conv.out_c, cin_store, conv.kh, conv.kw)
            nt = self.L.bnff_pack_size(self.dcode, cin_store, conv.out_c, conv.kh, conv.kw)
            self.packs[key] = (self._zeros((n,)), self._zeros((nt,)), cin_store, conv)
            # window-shift kernel weights (bf16 stride-1 1x1/3x3 convs)
            h, w = hw if hw is not None else (0, 0)
            # patch-matrix GEMMs: plain fprop operand, plain dgrad epilogue (dy may be deferred)
            tables = _lib.WT_DGRAD_PRO if key in self.col_src else _lib.WT_ALL
            if self.use_window and cin_store == conv.in_c and self.L.bnff_window_ok_ex(
                    self.dcode, conv.in_c, conv.out_c, conv.kh, conv.kw, conv.stride, conv.pad, h, w, tables):
                nf = self.L.bnff_window_pack_size(self.dcode, conv.out_c, conv.in_c, conv.kh, conv.kw, 0)
                nd = self.L.bnff_window_pack_size(self.dcode, conv.out_c, conv.in_c, conv.kh, conv.kw, 1)
                self.wpacks[key] = (self._zeros((nf,)), self._zeros((nd,)), conv)
        return self.packs[key]

    def _gpack(self, conv, t):
        """generic packed weights, or NULL for a window-layout conv (the optimizer only
        repacks its window layout: a rejected window launch must fail, not read stale packs)"""
        return 0 if conv.name in self.wpacks else _ptr(t)

    def _wwin(self, conv, which):
        wp = self.wpacks.get(conv.name)
        return 0 if wp is None else _ptr(wp[which])

    def _flush_pending(self, keep=None):
        """Emit the deferred statistics finalisations (all but `keep`)."""
        rest = []
        for pf in self._pending_fin:
            if pf is keep:
                rest.append(pf)
                continue
            part, tiles, c, count, st = pf
            self._emit(self.L.bnff_stats_finalize, _ptr(part), tiles, c, count, _ptr(st.sum),
                       _ptr(st.sumsq), _ptr(st.mean), _ptr(st.var), what="stats_finalize")
        self._pending_fin = rest

    def _bn_tables(self, st: Stats, bn, tag):
        """fp32 (mean, scale, beta, inv) for a normalize prologue (bn_fwd ops.py:246-249).
        A pending finalisation of a piece inside `st` (the channels a producer just wrote)
        is fused into the same launch."""
        c = st.mean.shape[0]
        mean32, scale32, beta32, inv32 = (self._zeros((c,), torch.float32) for _ in range(4))
        gam = self.param(f"{bn.name}.gamma")
        bet = self.param(f"{bn.name}.beta")
        lo = st.mean.data_ptr()
        hi = lo + 8 * c
        inside = [pf for pf in self._pending_fin
                  if lo <= pf[4].mean.data_ptr() and pf[4].mean.data_ptr() + 8 * pf[2] <= hi]
        merge = inside[-1] if inside else None
        self._flush_pending(keep=merge)
        if merge is None:
            self._emit(self.L.bnff_bn_coeffs, c, _ptr(st.mean), _ptr(st.var), _ptr(gam), _ptr(bet),
                       C.c_float(bn.eps), _ptr(mean32), _ptr(scale32), _ptr(beta32), _ptr(inv32),
                       what=f"bn_coeffs {tag}")
            return mean32, scale32, beta32, inv32
        self._pending_fin = []
        part, tiles, cn, count, ps = merge
        off = (ps.mean.data_ptr() - lo) // 8
        for _ in range(self.coef_reps):
            self._emit(self.L.bnff_stats_finalize_coeffs, _ptr(part), tiles, cn, count, _ptr(ps.sum),
                       _ptr(ps.sumsq), _ptr(ps.mean), _ptr(ps.var), off, c, _ptr(st.mean), _ptr(st.var),
                       _ptr(gam), _ptr(bet), C.c_float(bn.eps), _ptr(mean32), _ptr(scale32), _ptr(beta32),
                       _ptr(inv32), what=f"bn_coeffs {tag}")
        return mean32, scale32, beta32, inv32

    def _channel_stats(self, x: torch.Tensor, st: Stats, tag):
        pixels = x.shape[0] * x.shape[1] * x.shape[2]
        tiles = self.L.bnff_sum_tiles(pixels)
        part = self._empty((tiles, 2, x.shape[3]), torch.float64)
        self._emit(self.L.bnff_channel_sums, self.dcode, 0, view_of(x), view_of(x), coef_of(),
                   _ptr(part), what=f"channel_sums {tag}", nbytes=_nb(x))
        self._emit_stats_finalize(part, tiles, x.shape[3], pixels, st)

    # ---------------------------------------------------------------- forward
    def _compile_forward(self):
        self._cur = self.fwd
        self._pending_fin = []
        self.node_stats: dict = {}   # BN node id -> Stats (two/one-pass, baseline)
        self.node_tables: dict = {}  # node id -> fp32 tables
        self.stats: dict = {}        # stats slot id -> Stats
        for node in self.g.nodes:
            self._cur_node = node.id
            try:
                getattr(self, "_f_" + node.kind)(node)
            except ShapeError as e:
                raise ShapeError(f"node {node.id} ({node.kind} {node.name}): {e}") from e
        self._cur_node = -1
        self._flush_pending()
        self.launch_counts["fwd"] = len(self.fwd)

    def _col_conv(self, conv, x, pro=None):
        """Convolutions the window kernels cannot run directly go through a patch matrix and
        a 1x1 window GEMM over it (csrc/stem.cu): the channel-poor stem conv (the 3-channel
        image, stored with 8; pro NONE only) and strided convolutions whose channels fill
        16-byte chunks (ResNet's stride-2 3x3s; the operand prologue -- ReLU or BN+ReLU -- is
        applied while the patch matrix is written).  Returns (conv1x1, col, dw2, kpad,
        strided) or None when the conv does not qualify."""
        if conv.name in self.cols:
            return self.cols[conv.name]
        if not self.use_window or pro is None:
            return None
        n, h, w, cs = x.shape
        chunk = 16 // x.element_size()
        stem = cs * x.element_size() == 16 and conv.in_c <= cs and conv.kh * conv.kw > 1 \
            and pro == _lib.PRO_NONE
        strided = not stem and conv.stride > 1 and cs == conv.in_c and cs % chunk == 0 \
            and self.col_strided
        if not (stem or strided):
            return None
        taps_c = conv.kh * conv.kw * conv.in_c
        kpad = _round_up(taps_c, 16)
        oh, ow = conv.out_hw(h, w)
        # the GEMM over the patch matrix runs with a plain operand and a plain epilogue
        if not self.L.bnff_window_ok_ex(self.dcode, kpad, conv.out_c, 1, 1, 1, 0, oh, ow, _lib.WT_DGRAD_PRO):
            return None
        c1 = ConvParams(in_c=kpad, out_c=conv.out_c, kh=1, kw=1, name=conv.name + "#col")
        col = self._zeros((n, oh, ow, kpad)) if kpad != taps_c else self._empty((n, oh, ow, kpad))
        w2 = self._zeros((conv.out_c * kpad,), torch.float32)
        dw2 = self._zeros((conv.out_c * kpad,), torch.float32)
        self.col_src[c1.name] = (w2, conv, kpad)
        self.cols[conv.name] = ent = (c1, col, dw2, kpad, strided)
        return ent

    def _conv_fprop(self, node, x, y, conv, pro, tables, stat_part):
        col = self._col_conv(conv, x, pro)
        pname = conv.name
        if col is not None:  # patch matrix (operand prologue applied), then a 1x1 GEMM over it
            c1, colt, _, _, strided = col
            if strided:
                cf = coef_of() if tables is None else coef_of(tables[0], tables[1], tables[2])
                self._emit(self.L.bnff_im2col_s, self.dcode, view_of(x), conv.kh, conv.kw, conv.stride,
                           conv.pad, pro, cf, view_of(colt), what=f"im2col {node.name}",
                           nbytes=_nb(x, colt))
            else:
                self._emit(self.L.bnff_im2col, self.dcode, view_of(x), conv.in_c, conv.kh, conv.kw,
                           conv.stride, conv.pad, view_of(colt), what=f"im2col {node.name}",
                           nbytes=_nb(x, colt))
            x, conv, pro, tables = colt, c1, _lib.PRO_NONE, None
        cin_store = x.shape[3]
        wp, _, _, _ = self._pack(conv, cin_store, (x.shape[1], x.shape[2]))
        if tables is None:
            cf = coef_of()
        else:
            cf = coef_of(tables[0], tables[1], tables[2])
        args = _lib.FpropArgs(self.dcode, conv.kh, conv.kw, conv.stride, conv.pad, view_of(x),
                              view_of(y), self._gpack(conv, wp), _ptr(self.param(f"{pname}.bias")), pro, cf,
                              _ptr(stat_part), self._wwin(conv, 0))
        n_, oh_, ow_, co_ = y.shape
        flops = 2 * n_ * oh_ * ow_ * co_ * conv.kh * conv.kw * cin_store
        self._emit(self.L.bnff_conv_fprop, C.byref(args), what=f"fprop {node.name}",
                   nbytes=_nb(x, y, wp), flops=flops)
        self._keep.append(args)

    def _f_Conv2D(self, node):
        at = node.attrs
        x = self.acts[node.inputs[0]]
        y = self._feature(node.outputs[0])
        pro = _lib.PRO_RELU if at.clip_input else _lib.PRO_NONE
        if node.kind == G.FUSED_CONV_STATS:
            mt = self.L.bnff_stat_rows()
            part = self._zeros((mt, 2, y.shape[3]), torch.float64)
            self._conv_fprop(node, x, y, at.conv, pro, None, part)
            st = self._stats_for(node.outputs[0], y.shape[3], y.shape[0] * y.shape[1] * y.shape[2])
            self._emit_stats_finalize(part, mt, y.shape[3], st.count, st)
            self.stats[node.outputs[1]] = st
        else:
            self._conv_fprop(node, x, y, at.conv, pro, None, None)

    _f_FusedConvStats = _f_Conv2D

    def _f_BatchNorm(self, node):
        x = self.acts[node.inputs[0]]
        y = self._feature(node.outputs[0])
        c = x.shape[3]
        pixels = x.shape[0] * x.shape[1] * x.shape[2]
        st = Stats(*(self._zeros((c,), torch.float64) for _ in range(4)), count=pixels)
        self._channel_stats(x, st, node.name)
        if not node.attrs.onepass:  # two-pass: centred variance overwrites var (ops.py:226-227)
            self._flush_pending()  # the centred pass reads the mean
            tiles = self.L.bnff_sum_tiles(pixels)
            part = self._empty((tiles, 2, c), torch.float64)
            self._emit(self.L.bnff_centered_var, self.dcode, view_of(x), _ptr(st.mean), _ptr(part),
                       what="centered_var", nbytes=_nb(x))
            # var, then the fp32 tables of this BN in the same launch
            tb = tuple(self._zeros((c,), torch.float32) for _ in range(4))
            bn = node.attrs.bn
            self._emit(self.L.bnff_var_finalize_coeffs, _ptr(part), tiles, c, pixels, _ptr(st.var),
                       _ptr(st.mean), _ptr(self.param(f"{bn.name}.gamma")), _ptr(self.param(f"{bn.name}.beta")),
                       C.c_float(bn.eps), *(_ptr(t) for t in tb), what=f"bn_coeffs {node.name}")
        else:
            tb = self._bn_tables(st, node.attrs.bn, node.name)
        self.node_stats[node.id] = st
        self.node_tables[node.id] = tb
        self._emit(self.L.bnff_bn_apply, self.dcode, view_of(x), view_of(y),
                   coef_of(tb[0], tb[1], tb[2]), 0, what="bn_apply", nbytes=_nb(x, y))

    def _f_ReLU(self, node):
        if node.id in self._nrp:  # done by the fused norm-ReLU-pool
            return
        x = self.acts[node.inputs[0]]
        y = self._feature(node.outputs[0])
        self._emit(self.L.bnff_relu_fwd, self.dcode, view_of(x), view_of(y), what="relu_fwd",
                   nbytes=_nb(x, y))

    def _f_FissionSubBN1(self, node):
        x = self.acts[node.inputs[0]]
        st = self._stats_for(node.inputs[0], x.shape[3], x.shape[0] * x.shape[1] * x.shape[2])
        self._channel_stats(x, st, node.name)
        self.stats[node.outputs[0]] = st

    def _nrp_chain(self, node):
        """sub-BN2 -> ReLU -> 2x2 AvgPool with single consumers (the stem): (relu, pool) or None."""
        if not self.fuse_nrp:
            return None
        outs = set(self.g.outputs)
        c1 = self.g.consumers_of(node.outputs[0])
        if len(c1) != 1 or c1[0].kind != G.RELU or node.outputs[0] in outs:
            return None
        relu = c1[0]
        c2 = self.g.consumers_of(relu.outputs[0])
        if len(c2) != 1 or c2[0].kind != G.POOL or relu.outputs[0] in outs or c2[0].attrs.k != 2:
            return None
        return relu, c2[0]

    def _f_FissionSubBN2(self, node):
        x = self.acts[node.inputs[0]]
        st = self.stats.get(node.inputs[1])
        if st is None:
            raise StateError(f"{node.name}: statistics slot {node.inputs[1]} never produced")
        chain = self._nrp_chain(node)
        if chain is not None:  # normalize + ReLU + pool in one pass over the conv output
            relu, pool = chain
            tb = self._bn_tables(st, node.attrs.bn, node.name)
            self.node_tables[node.id] = tb
            y = self._feature(pool.outputs[0])
            pixels = y.shape[0] * y.shape[1] * y.shape[2]
            part, tiles = None, 0
            if pool.attrs.emit_stats:
                tiles = self.L.bnff_sum_tiles(pixels)
                part = self._empty((tiles, 2, y.shape[3]), torch.float64)
            self._emit(self.L.bnff_norm_relu_pool_fwd, self.dcode, view_of(x), view_of(y), pool.attrs.k,
                       coef_of(tb[0], tb[1], tb[2]), _ptr(part), what=f"norm_relu_pool {node.name}",
                       nbytes=_nb(x, y))
            if pool.attrs.emit_stats:
                pst = self._stats_for(pool.outputs[0], y.shape[3], pixels)
                self._emit_stats_finalize(part, tiles, y.shape[3], pixels, pst)
                self.stats[pool.outputs[1]] = pst
            self._nrp[relu.id] = self._nrp[pool.id] = node
            return
        y = self._feature(node.outputs[0])
        tb = self._bn_tables(st, node.attrs.bn, node.name)
        self.node_tables[node.id] = tb
        self._emit(self.L.bnff_bn_apply, self.dcode, view_of(x), view_of(y),
                   coef_of(tb[0], tb[1], tb[2]), 0, what="subbn2", nbytes=_nb(x, y))

    def _f_FusedNormReluConv(self, node):
        at = node.attrs
        x = self.acts[node.inputs[0]]
        st = self.stats.get(node.inputs[1])
        if st is None:
            raise StateError(f"{at.conv.name}: no statistics available for normalization input")
        y = self._feature(node.outputs[0])
        tb = self._bn_tables(st, at.bn, node.name)
        self.node_tables[node.id] = tb
        # cost model: the fused prologue normalises the input once per N tile of the conv; past
        # two N tiles (very wide 1x1s: ResNet expansions, the C5 sweep at C >= 512) one
        # materialising bn_apply pass is cheaper than repeating the transform
        n_tile = 256 if self.dcode == _lib.BF16 else 128
        wide = self.wide_fallback and -(-at.conv.out_c // n_tile) > 2
        if self.save_postrelu or wide:
            saved = self._feature(node.outputs[1])
            self._emit(self.L.bnff_bn_apply, self.dcode, view_of(x), view_of(saved),
                       coef_of(tb[0], tb[1], tb[2]), 1, what="saved_postrelu", nbytes=_nb(x, saved))
        part = None
        if at.emit_stats:
            mt = self.L.bnff_stat_rows()
            part = self._zeros((mt, 2, y.shape[3]), torch.float64)
        if wide:
            self._wide_saved[node.id] = saved
            self._conv_fprop(node, saved, y, at.conv, _lib.PRO_NONE, None, part)
        else:
            self._conv_fprop(node, x, y, at.conv, _lib.PRO_BN_RELU, tb, part)
        if at.emit_stats:
            ost = self._stats_for(node.outputs[0], y.shape[3], y.shape[0] * y.shape[1] * y.shape[2])
            self._emit_stats_finalize(part, mt, y.shape[3], ost.count, ost)
            self.stats[node.outputs[2]] = ost

    def _f_Concat(self, node):
        y = self._feature(node.outputs[0])
        feats = [s for s in node.inputs if self.g.slots[s].kind == "feature"]
        if node.attrs.physical:
            off = 0
            for s in feats:
                piece = self.acts[s]
                c = piece.shape[3]
                self._emit(self.L.bnff_copy, self.dcode, view_of(piece), view_of(y[..., off:off + c]),
                           what="concat_copy", nbytes=2 * _nb(piece))
                off += c
        else:
            off = 0
            for s in feats:  # view mode: producers already wrote in place
                piece = self.acts[s]
                if piece.data_ptr() != y[..., off:].data_ptr():
                    raise StateError(f"{node.name}: view-concat piece {s} not in the block buffer")
                off += piece.shape[3]

    def _f_FusedConcatStats(self, node):
        feat = [s for s in node.inputs if self.g.slots[s].kind == "feature"]
        stat = [s for s in node.inputs if self.g.slots[s].kind == "stats"]
        self._f_Concat(node)
        y = self.acts[node.outputs[0]]
        st = self._stats_for(node.outputs[0], y.shape[3], y.shape[0] * y.shape[1] * y.shape[2])
        if self.sync_bn:  # the pieces' moments are over the global batch (_emit_stats_finalize)
            st.count *= self.world
        off = 0
        for fs, ss in zip(feat, stat):
            piece = self.stats[ss]
            c = piece.mean.shape[0]
            for a, b in zip((st.sum, st.sumsq, st.mean, st.var),
                            (piece.sum, piece.sumsq, piece.mean, piece.var)):
                if a[off:off + c].data_ptr() != b.data_ptr():  # not in place: copy (ops.py:128-143)
                    self._flush_pending()
                    dst = a[off:off + c]
                    def _cp(stream, d=dst, s=b):
                        d.copy_(s)
                    _cp.what, _cp.kind, _cp.nbytes, _cp.flops = "stats_copy", "stats_copy", 0, 0
                    self._cur.append(_cp)
            off += c
        self.stats[node.outputs[1]] = st

    def _f_Split(self, node):
        x = self.acts[node.inputs[0]]
        for o in node.outputs:
            self.acts[o] = x

    def _f_EltwiseSum(self, node):
        a, b = self.acts[node.inputs[0]], self.acts[node.inputs[1]]
        y = self._feature(node.outputs[0])
        if not node.attrs.pad_channels and a.shape != b.shape:
            raise ShapeError(f"EltwiseSum operands {tuple(a.shape)} vs {tuple(b.shape)}")
        self._emit(self.L.bnff_ews_fwd, self.dcode, view_of(a), view_of(b), view_of(y), what="ews",
                   nbytes=_nb(a, b, y))

    def _f_AvgPool(self, node):
        if node.id in self._nrp:
            return
        x = self.acts[node.inputs[0]]
        y = self._feature(node.outputs[0])
        part = None
        pixels = y.shape[0] * y.shape[1] * y.shape[2]
        if node.attrs.emit_stats:
            tiles = self.L.bnff_sum_tiles(pixels)
            part = self._empty((tiles, 2, y.shape[3]), torch.float64)
        self._emit(self.L.bnff_avgpool_fwd, self.dcode, view_of(x), view_of(y), node.attrs.k,
                   _ptr(part), what="avgpool", nbytes=_nb(x, y))
        if node.attrs.emit_stats:
            st = self._stats_for(node.outputs[0], y.shape[3], pixels)
            self._emit_stats_finalize(part, tiles, y.shape[3], pixels, st)
            self.stats[node.outputs[1]] = st

    # --------------------------------------------------------------- backward
    def _compile_backward(self):
        self._cur = self.bwd
        g = self.g
        self.loss_grad = {}
        self.grads: dict = {}
        for sid in g.outputs:
            n, c, h, w = g.slots[sid].shape
            t = self._zeros((n, h, w, c))
            self.loss_grad[sid] = t
            self.grads[sid] = Plain(t)
        # shared split-K workspace (kernels run in stream order)
        ws = 1
        for node in g.nodes:
            conv = getattr(node.attrs, "conv", None)
            if conv is None:
                continue
            xs = g.slots[node.inputs[0]].shape
            oh, ow = conv.out_hw(xs[2], xs[3])
            cin_s = self._store_c(xs[1])
            ws = max(ws, self.L.bnff_wgrad_workspace(xs[0], oh, ow, conv.kh, conv.kw, cin_s,
                                                    conv.out_c, 0))
        for c1, colt, _, _, _ in self.cols.values():  # GEMMs over patch matrices
            n, oh, ow, kp = colt.shape
            ws = max(ws, self.L.bnff_wgrad_workspace(n, oh, ow, 1, 1, kp, c1.out_c, 0))
        self.wg_ws = self._empty((ws,), torch.float32)
        self._side_reads: list = []  # tensors read by side-stream thunks (pending until the join)
        self._done_params: set = set()
        self._bucket_hi = int(self.gflat.numel())
        for node in reversed(g.nodes):
            self._cur_node = node.id
            try:
                getattr(self, "_b_" + node.kind)(node)
            except ShapeError as e:
                raise ShapeError(f"node {node.id} ({node.kind} {node.name}): {e}") from e
            if self.dp_buckets:
                self._done_params.update(self._params_of(node))
                self._maybe_bucket(final=False)
        self._cur_node = -1
        if self.dp_buckets:
            self._maybe_bucket(final=True)
        self.input_grads = {}
        for sid in g.inputs:
            gv = self.grads.get(sid)
            self.input_grads[sid] = self._resolve(gv) if (gv is not None and self.input_grad) else None
        self.launch_counts["bwd"] = len(self.bwd)

    @staticmethod
    def _params_of(node):
        at = node.attrs
        names = []
        conv = getattr(at, "conv", None)
        if conv is not None:
            names += [f"{conv.name}.weight", f"{conv.name}.bias"]
        bn = getattr(at, "bn", None)
        if bn is not None:
            names += [f"{bn.name}.gamma", f"{bn.name}.beta"]
        return names

    def _maybe_bucket(self, final: bool):
        """Emit an all-reduce of the flat-gradient range [lo, hi) once every parameter in it
        has its final gradient and the range holds >= bucket_bytes (the remainder at the end).
        Parameters sit in forward order in the flat buffer and finish in reverse order, so the
        finished ones form a suffix; a range is only issued while that holds."""
        hi = self._bucket_hi
        if final:
            lo = 0
        else:
            done = [self.poff[k] for k in self._done_params if k in self.poff]
            if not done:
                return
            lo = min(o for o, _ in done)
            # every parameter inside [lo, hi) must be final
            if any(o < hi and o + n > lo and k not in self._done_params for k, (o, n) in self.poff.items()):
                return
            if (hi - lo) * 4 < self.bucket_bytes:
                return
        if hi <= lo:
            return
        self._emit_grad_allreduce(lo, hi)
        self._bucket_hi = lo

    def _emit_grad_allreduce(self, lo, hi):
        import torch.distributed as dist
        grp = self.group
        view = self.gflat[lo:hi]
        self.buckets.append((lo, hi))

        def _ar(stream, v=view):
            main = torch.cuda.current_stream(self.dev)
            if self._comm is None:
                self._comm = torch.cuda.Stream(self.dev)
            ev = torch.cuda.Event()
            ev.record(main)
            self._comm.wait_event(ev)
            if self._side is not None:  # the bucket's weight gradients ran on the side stream
                ev2 = torch.cuda.Event()
                ev2.record(self._side)
                self._comm.wait_event(ev2)
            with torch.cuda.stream(self._comm):
                if dist.is_initialized():
                    dist.all_reduce(v, op=dist.ReduceOp.SUM, group=grp)
            self._comm_used = True
        _ar.what = f"grad_allreduce [{lo}, {hi})"
        _ar.kind, _ar.nbytes, _ar.flops, _ar.launches = "grad_allreduce", 0, 0, 0
        self._cur.append(_ar)

    def _fresh_like(self, t):
        return self._empty(tuple(t.shape))

    def _resolve(self, gv) -> torch.Tensor:
        """Materialise a deferred package (DeferredBNGrad.materialize, execute.py:123-126)."""
        if isinstance(gv, Plain):
            return gv.t
        out = self._fresh_like(gv.dt1)
        term = _lib.GradTerm(view_of(gv.dt1), view_of(gv.x), 1, gv.coef())
        self._keep.append(term)
        self._emit(self.L.bnff_grad_sum, self.dcode, view_of(out), 0, C.byref(term), 1,
                   what="bn_dx", nbytes=_nb(gv.dt1, gv.x, out))
        return out

    def _incoming(self, sid) -> torch.Tensor:
        gv = self.grads.get(sid)
        if gv is None:
            raise StateError(f"no gradient arrived at slot {sid}")
        return self._resolve(gv)

    def _add_grad(self, sid, gv):
        cur = self.grads.get(sid)
        if cur is None:
            self.grads[sid] = gv
            return
        if isinstance(cur, Deferred) or isinstance(gv, Deferred):
            raise StateError(f"slot {sid}: deferred gradient cannot be accumulated")
        out = self._fresh_like(cur.t)
        terms = (_lib.GradTerm * 2)(_lib.GradTerm(view_of(cur.t), view_of(cur.t), 0, coef_of()),
                                    _lib.GradTerm(view_of(gv.t), view_of(gv.t), 0, coef_of()))
        self._keep.append(terms)
        self._emit(self.L.bnff_grad_sum, self.dcode, view_of(out), 0, terms, 2, what="grad_add",
                   nbytes=_nb(cur.t, gv.t, out))
        self.grads[sid] = Plain(out)

    def _wants_dx(self, sid):
        return self.input_grad or sid not in self.g.inputs

    def _conv_backward(self, node, conv, x, dy_gv, x_pro, x_tables, dgrad_epi, dgrad_tables,
                       dx_out=None):
        """dgrad (+ epilogue) and wgrad of one conv; returns the dx tensor (or None).
        dx_out: the block gradient view the fold epilogues (DG_NRC_ACC/SET) write into.
        A wide NRC conv whose forward materialised relu(bn(x)) (_f_FusedNormReluConv) takes its
        weight-gradient operand from that tensor instead of re-normalising x per N tile."""
        cin_store = x.shape[3]
        if isinstance(dy_gv, Deferred) and self.wide_dx and dy_gv.dt1.shape[3] >= self.wide_dx \
                and cin_store > 256:
            dy_gv = Plain(self._resolve(dy_gv))
        col = self.cols.get(conv.name)
        if col is None:
            _, wt, _, _ = self._pack(conv, cin_store, (x.shape[1], x.shape[2]))
        if isinstance(dy_gv, Deferred):
            dy, dy_x, dy_pro, dy_coef = dy_gv.dt1, dy_gv.x, _lib.PRO_BN_DX, dy_gv.coef()
        else:
            dy, dy_x, dy_pro, dy_coef = dy_gv.t, dy_gv.t, _lib.PRO_NONE, coef_of()
        xc = coef_of() if x_tables is None else coef_of(x_tables[0], x_tables[1], x_tables[2])
        orig, wconv, wx, wcin, wpro = conv, conv, x, cin_store, x_pro
        saved = self._wide_saved.get(node.id)
        if saved is not None and x_pro == _lib.PRO_BN_RELU:
            wx, wpro, xc = saved, _lib.PRO_NONE, coef_of()
        dw = self.grad(f"{conv.name}.weight")
        if col is not None:  # weight gradient of the 1x1 GEMM over the (transformed) patch matrix
            wconv, wx, dw, wpro, xc = col[0], col[1], col[2], _lib.PRO_NONE, coef_of()
            wcin = wx.shape[3]
        wa = _lib.WgradArgs(self.dcode, wconv.kh, wconv.kw, wconv.stride, wconv.pad, view_of(wx), wpro,
                            xc, view_of(dy), view_of(dy_x), dy_pro, dy_coef, 0, _ptr(self.wg_ws),
                            _ptr(dw), wconv.in_c, _ptr(self.grad(f"{orig.name}.bias")))
        self._keep.append(wa)
        n_, oh_, ow_, co_ = dy.shape
        flops = 2 * n_ * oh_ * ow_ * co_ * wconv.kh * wconv.kw * wcin
        extra = _nb(dy_x) if dy_pro == _lib.PRO_BN_DX else 0
        # the weight gradient is off the critical path: it runs on the side stream, forked
        # before this conv's dgrad (they read the same dy) and joined at the end of backward
        if self.side_wgrad:
            self._side_reads += [dy, dy_x]
        self._emit(self.L.bnff_conv_wgrad, C.byref(wa), what=f"wgrad {node.name}",
                   nbytes=_nb(wx, dy) + extra + 4 * wconv.out_c * wconv.in_c * wconv.kh * wconv.kw,
                   flops=flops, launches=4, side=self.side_wgrad)
        if col is not None:
            self._emit(self.L.bnff_cols_to_weight, _ptr(col[2]), orig.out_c, orig.in_c, orig.kh,
                       orig.kw, col[3], _ptr(self.grad(f"{orig.name}.weight")),
                       what=f"cols_to_weight {node.name}", side=self.side_wgrad)
        dx, part = None, None
        if col is not None and self._wants_dx(node.inputs[0]):
            # input gradient: dgrad of the 1x1 GEMM over the patch matrix (dcol), then a col2im
            # gather (the stem's into the channel-padded image layout; a strided conv's with its
            # dgrad epilogue: ReLU clip or the NRC mask, whose statistics follow from dx)
            c1, colt, _, kpad, strided = col
            dcol = self._empty(tuple(colt.shape))
            _, wt1, _, _ = self._pack(c1, kpad, (colt.shape[1], colt.shape[2]))
            da = _lib.DgradArgs(self.dcode, 1, 1, 1, 0, view_of(dy), view_of(dy_x), dy_pro, dy_coef,
                                view_of(dcol), view_of(colt), self._gpack(c1, wt1), _lib.DG_PLAIN, coef_of(), 0,
                                self._wwin(c1, 1))
            self._keep.append(da)
            n_, h_, w_, _ = dcol.shape
            extra = _nb(dy_x) if dy_pro == _lib.PRO_BN_DX else 0
            self._emit(self.L.bnff_conv_dgrad, C.byref(da), what=f"dgrad {node.name}",
                       nbytes=_nb(dy, dcol, wt1) + extra, flops=2 * n_ * h_ * w_ * kpad * dy.shape[3])
            if not strided:
                dx = self._empty(tuple(x.shape))
                self._emit(self.L.bnff_col2im, self.dcode, view_of(dcol), orig.in_c, orig.kh, orig.kw,
                           orig.stride, orig.pad, view_of(dx), what=f"col2im {node.name}",
                           nbytes=_nb(dcol, dx))
                return dx, None
            if dgrad_epi not in (_lib.DG_PLAIN, _lib.DG_CLIP, _lib.DG_NRC):
                raise StateError(f"{node.name}: dgrad epilogue {dgrad_epi} on a patch-matrix conv")
            dx = self._empty(tuple(x.shape)) if dx_out is None else dx_out
            ecoef = coef_of()
            if dgrad_epi == _lib.DG_NRC:
                m32, s32, b32, i32 = dgrad_tables
                ecoef = coef_of(m32, s32, b32, i32)
            self._emit(self.L.bnff_col2im_s, self.dcode, view_of(dcol), orig.kh, orig.kw, orig.stride,
                       orig.pad, dgrad_epi, view_of(x), ecoef, view_of(dx), what=f"col2im {node.name}",
                       nbytes=_nb(dcol, dx) + (_nb(x) if dgrad_epi != _lib.DG_PLAIN else 0))
            if dgrad_epi == _lib.DG_NRC:  # (sum dt1, sum dt1*xhat) of the stored dt1
                pixels = x.shape[0] * x.shape[1] * x.shape[2]
                tiles = self.L.bnff_sum_tiles(pixels)
                part = self._empty((tiles, 2, x.shape[3]), torch.float64)
                self._emit(self.L.bnff_channel_sums, self.dcode, 1, view_of(x), view_of(dx),
                           coef_of(m32, i32), _ptr(part), what=f"nrc_sums {node.name}", nbytes=_nb(x, dx))
            return dx, part
        if self._wants_dx(node.inputs[0]):
            dx = self._empty(tuple(x.shape)) if dx_out is None else dx_out
            ecoef = coef_of()
            if dgrad_epi >= _lib.DG_NRC:
                part = self._zeros((self.L.bnff_stat_rows(), 2, x.shape[3]), torch.float64)
                m32, s32, b32, i32 = dgrad_tables
                ecoef = coef_of(m32, s32, b32, i32)
            da = _lib.DgradArgs(self.dcode, conv.kh, conv.kw, conv.stride, conv.pad, view_of(dy),
                                view_of(dy_x), dy_pro, dy_coef, view_of(dx), view_of(x), self._gpack(conv, wt),
                                dgrad_epi, ecoef, _ptr(part), self._wwin(conv, 1))
            self._keep.append(da)
            n_, h_, w_, ci_ = dx.shape
            flops = 2 * n_ * h_ * w_ * ci_ * conv.kh * conv.kw * dy.shape[3]
            extra = _nb(dy_x) if dy_pro == _lib.PRO_BN_DX else 0
            extra += _nb(x) if dgrad_epi != _lib.DG_PLAIN else 0
            extra += _nb(dx) if dgrad_epi == _lib.DG_NRC_ACC else 0  # read-modify-write
            self._emit(self.L.bnff_conv_dgrad, C.byref(da), what=f"dgrad {node.name}",
                       nbytes=_nb(dy, dx, wt) + extra, flops=flops)
        return dx, part

    def _b_Conv2D(self, node):
        at = node.attrs
        raw = self.grads.get(node.outputs[0])
        if raw is None:
            raise StateError(f"no gradient arrived at slot {node.outputs[0]}")
        x = self.acts[node.inputs[0]]
        epi = _lib.DG_CLIP if at.clip_input else _lib.DG_PLAIN
        pro = _lib.PRO_RELU if at.clip_input else _lib.PRO_NONE
        dx, _ = self._conv_backward(node, at.conv, x, raw, pro, None, epi, None)
        if dx is not None:
            self._add_grad(node.inputs[0], Plain(dx))

    _b_FusedConvStats = _b_Conv2D

    def _dx_coeffs(self, part, tiles, c, count, st: Stats, bn, tag):
        k1, k2, gg, m32, i32 = (self._zeros((c,), torch.float32) for _ in range(5))
        dg64, db64 = self._zeros((c,), torch.float64), self._zeros((c,), torch.float64)
        if not self.sync_bn:
            self._emit(self.L.bnff_dx_coeffs, c, _ptr(part), tiles, count, _ptr(st.mean),
                       _ptr(st.var), _ptr(self.param(f"{bn.name}.gamma")), C.c_float(bn.eps),
                       _ptr(dg64), _ptr(db64), _ptr(k1), _ptr(k2), _ptr(gg), _ptr(m32), _ptr(i32),
                       _ptr(self.grad(f"{bn.name}.gamma")), _ptr(self.grad(f"{bn.name}.beta")),
                       what=f"dx_coeffs {tag}")
            return m32, i32, k1, k2, gg
        # SyncBN: the replica's own (dbeta, dgamma) sums become its parameter gradients (the
        # data-parallel gradient all-reduce adds them up); the dx coefficients use the
        # all-reduced global sums and the global count.
        self._emit(self.L.bnff_stats_finalize, _ptr(part), tiles, c, count, _ptr(db64), _ptr(dg64),
                   None, None, what=f"dx_coeffs {tag}")
        self._emit(self.L.bnff_sums_to_f32, c, _ptr(dg64), _ptr(db64),
                   _ptr(self.grad(f"{bn.name}.gamma")), _ptr(self.grad(f"{bn.name}.beta")),
                   what=f"dx_coeffs {tag}")
        self._emit_allreduce(db64, dg64, what="syncbn_bwd_allreduce")
        self._emit(self.L.bnff_dx_coeffs_from_sums, c, st.count, _ptr(db64), _ptr(dg64),
                   _ptr(st.mean), _ptr(st.var), _ptr(self.param(f"{bn.name}.gamma")),
                   C.c_float(bn.eps), _ptr(k1), _ptr(k2), _ptr(gg), _ptr(m32), _ptr(i32),
                   what=f"dx_coeffs {tag}")
        return m32, i32, k1, k2, gg

    def _bn_grad_sums(self, x, dy, tables, st, bn, tag):
        """dbeta = sum dy, dgamma = sum dy*xhat (ops.py:271-274) -> backward table."""
        pixels = x.shape[0] * x.shape[1] * x.shape[2]
        tiles = self.L.bnff_sum_tiles(pixels)
        part = self._empty((tiles, 2, x.shape[3]), torch.float64)
        m32, _, _, i32 = tables
        self._emit(self.L.bnff_channel_sums, self.dcode, 1, view_of(x), view_of(dy),
                   coef_of(m32, i32), _ptr(part), what=f"bn_bwd_sums {tag}", nbytes=_nb(x, dy))
        return self._dx_coeffs(part, tiles, x.shape[3], pixels, st, bn, tag)

    def _b_BatchNorm(self, node):
        st = self.node_stats.get(node.id)
        if st is None:
            raise StateError(f"node {node.id}: backward before forward (no saved statistics)")
        dy = self._incoming(node.outputs[0])
        x = self.acts[node.inputs[0]]
        m32, i32, k1, k2, gg = self._bn_grad_sums(x, dy, self.node_tables[node.id], st,
                                                  node.attrs.bn, node.name)
        self._add_grad(node.inputs[0], Plain(self._resolve(Deferred(dy, x, m32, i32, k1, k2, gg))))

    def _b_ReLU(self, node):
        if node.id in self._nrp:
            return
        dy = self._incoming(node.outputs[0])
        x = self.acts[node.inputs[0]]
        dx = self._fresh_like(x)
        self._emit(self.L.bnff_relu_bwd, self.dcode, view_of(x), view_of(dy), view_of(dx),
                   what="relu_bwd", nbytes=_nb(x, dy, dx))
        self._add_grad(node.inputs[0], Plain(dx))

    def _b_FissionSubBN1(self, node):
        if node.attrs.defer_backward:
            return
        pending = self.grads.get(node.inputs[0])
        if isinstance(pending, Deferred):
            self.grads[node.inputs[0]] = Plain(self._resolve(pending))

    def _b_FissionSubBN2(self, node):
        if node.id in self._nrp_done:
            return
        dy = self._incoming(node.outputs[0])
        x = self.acts[node.inputs[0]]
        st = self.stats[node.inputs[1]]
        m32, i32, k1, k2, gg = self._bn_grad_sums(x, dy, self.node_tables[node.id], st,
                                                  node.attrs.bn, node.name)
        self._add_grad(node.inputs[0], Deferred(dy, x, m32, i32, k1, k2, gg))

    def _b_FusedNormReluConv(self, node):
        at = node.attrs
        gv = self.grads.get(node.outputs[0])
        if gv is None:
            raise StateError(f"no gradient arrived at slot {node.outputs[0]}")
        x = self.acts[node.inputs[0]]
        st = self.stats[node.inputs[1]]
        tb = self.node_tables[node.id]
        if not self._wants_dx(node.inputs[0]):
            raise StateError("FusedNormReluConv directly on the graph input is not supported")
        fold = self._fold_plan(node, at.conv, x)
        if fold is not None:
            self._fold_backward(node, at, x, st, tb, gv, *fold)
            return
        dt1, part = self._conv_backward(node, at.conv, x, gv, _lib.PRO_BN_RELU, tb, _lib.DG_NRC, tb)
        mt = part.shape[0]
        m32, i32, k1, k2, gg = self._dx_coeffs(part, mt, x.shape[3], st.count, st, at.bn, node.name)
        self._add_grad(node.inputs[0], Deferred(dt1, x, m32, i32, k1, k2, gg))

    # ------------------------------------------------- ICF block-gradient fold
    def _fold_plan(self, node, conv, x):
        """(target view, sibling slot or None, mode, group, lo) when this consumer's BN dx
        can be folded into the block gradient buffer, else None."""
        if not self.fold_icf or conv.kh != 1 or conv.name not in self.wpacks:
            return None
        if self.dcode == _lib.F32 and x.shape[3] < 64:  # the fp32 fold runs on 32-column TMA tiles
            return None
        sid = node.inputs[0]
        slot = self.g.slots[sid]
        if slot.buffer is None or sid in self.grads:
            return None
        grp, lo = slot.buffer
        if lo != 0:
            return None
        prod = self.g.producer_of(sid)
        if prod is not None and prod.kind == G.SPLIT:
            sib = next(o for o in prod.outputs if o != sid)
            sg = self.grads.get(sib)
            tgt = sg.t if isinstance(sg, Plain) else sg.dt1 if isinstance(sg, Deferred) else None
            if tgt is not None and not self._writable(tgt):
                return None  # the caller's loss gradient, or still read by a side-stream wgrad
            if isinstance(sg, Plain) and tuple(sg.t.shape) == tuple(x.shape):
                return sg.t, sib, _lib.DG_NRC_ACC, grp, lo
            if isinstance(sg, Deferred) and sg.affine and tuple(sg.dt1.shape) == tuple(x.shape):
                return sg.dt1, sib, _lib.DG_NRC_ACC, grp, lo
            return None
        if len(self.g.consumers_of(sid)) != 1:
            return None
        # nothing downstream yet (a transition over the whole block): start a fresh buffer
        return self._empty(tuple(x.shape)), None, _lib.DG_NRC_SET, grp, lo

    def _fold_arrays(self, grp):
        fa = self.fold.get(grp)
        if fa is None:
            ct = self.g.buffer_groups[grp][0]
            fa = {k: self._zeros((ct,), torch.float32) for k in ("A", "B", "m32", "i32")}
            fa["ones"] = torch.ones((ct,), dtype=torch.float32, device=self.dev)
            self._bufs.append(fa["ones"])
            fa["started"] = False
            self.fold[grp] = fa
        return fa

    def _fold_backward(self, node, at, x, st, tb, gv, target, sib, mode, grp, lo):
        """1x1 NRC backward whose BN dx is folded into the block gradient: the dgrad epilogue
        writes target (+)= scale * dt1, dx_coeffs_acc adds g*k1 / g*k2 into (A, B); the
        block gradient is then G - A - B * xhat (a Deferred with g = 1), resolved by the
        channels' producers (bn_dx_from_sums ops.py:283-298, re-associated over consumers)."""
        c = x.shape[3]
        fa = self._fold_arrays(grp)
        sl = slice(lo, lo + c)
        _, part = self._conv_backward(node, at.conv, x, gv, _lib.PRO_BN_RELU, tb, mode, tb,
                                      dx_out=target)
        k1, k2, gg = (self._zeros((c,), torch.float32) for _ in range(3))
        dg64, db64 = self._zeros((c,), torch.float64), self._zeros((c,), torch.float64)
        # a plain (or fresh) target carries no pending remainder: (A, B) restart for its channels
        init = 0 if mode == _lib.DG_NRC_ACC and isinstance(self.grads.get(sib), Deferred) else 1
        self._emit(self.L.bnff_dx_coeffs_acc, c, _ptr(part), part.shape[0], st.count, _ptr(st.mean),
                   _ptr(st.var), _ptr(self.param(f"{at.bn.name}.gamma")), C.c_float(at.bn.eps),
                   _ptr(dg64), _ptr(db64), _ptr(k1), _ptr(k2), _ptr(gg), _ptr(fa["m32"][sl]),
                   _ptr(fa["i32"][sl]), _ptr(self.grad(f"{at.bn.name}.gamma")),
                   _ptr(self.grad(f"{at.bn.name}.beta")), _ptr(fa["A"][sl]), _ptr(fa["B"][sl]), init,
                   what=f"dx_coeffs {node.name}")
        aff = Deferred(target, x, fa["m32"][sl], fa["i32"][sl], fa["A"][sl], fa["B"][sl], fa["ones"][sl],
                       affine=True)
        if sib is not None:
            self.grads[sib] = aff
            self.grads[node.inputs[0]] = Folded(sib)
        else:
            self._add_grad(node.inputs[0], aff)

    def _b_Concat(self, node):
        gv = self.grads.get(node.outputs[0])
        if gv is None:
            raise StateError(f"no gradient arrived at concat output {node.outputs[0]}")
        physical = node.kind == G.CONCAT and node.attrs.physical
        off = 0
        for s in (s for s in node.inputs if self.g.slots[s].kind == "feature"):
            c = self.g.slots[s].shape[1]
            if isinstance(gv, Deferred):
                piece = gv.slice(off, off + c)
            else:
                sl = gv.t[..., off:off + c]
                if physical:  # the reference copies each piece (execute.py:438)
                    cp = self._empty(tuple(sl.shape))
                    self._emit(self.L.bnff_copy, self.dcode, view_of(sl), view_of(cp),
                               what="concat_bwd_copy", nbytes=2 * _nb(sl))
                    sl = cp
                piece = Plain(sl)
            self._add_grad(s, piece)
            off += c

    _b_FusedConcatStats = _b_Concat

    def _b_Split(self, node):
        branches = []
        for o in node.outputs:
            gv = self.grads.get(o)
            if gv is None:
                raise StateError(f"no gradient arrived at split branch {o}")
            if isinstance(gv, Folded):  # already inside the sibling branch's gradient
                continue
            branches.append(gv)
        if len(branches) == 1:
            self._add_grad(node.inputs[0], branches[0])
            return
        # in place into a plain branch's storage when that is safe (a block gradient buffer
        # this backward wrote), else into a fresh buffer
        out = next((b.t for b in branches if isinstance(b, Plain) and self._writable(b.t)), None)
        if out is None:
            out = self._fresh_like(branches[0].dt1)
        if any(isinstance(b, Plain) and b.t is out for b in branches):  # the in-place branch first
            branches.sort(key=lambda b: not (isinstance(b, Plain) and b.t is out))

        def term(b):
            if isinstance(b, Plain):
                return _lib.GradTerm(view_of(b.t), view_of(b.t), 0, coef_of())
            return _lib.GradTerm(view_of(b.dt1), view_of(b.x), 1, b.coef())
        # up to two branches per launch; later launches accumulate into out
        for i in range(0, len(branches), 2):
            part = branches[i:i + 2]
            terms = (_lib.GradTerm * len(part))(*[term(b) for b in part])
            self._keep.append(terms)
            nb = _nb(out) * (2 if i else 1) + sum(_nb(b.t) if isinstance(b, Plain) else _nb(b.dt1, b.x)
                                                  for b in part)
            self._emit(self.L.bnff_grad_sum, self.dcode, view_of(out), 1 if i else 0, terms, len(part),
                       what="split_bwd", nbytes=nb)
        self._add_grad(node.inputs[0], Plain(out))

    @staticmethod
    def _footprint(t):
        """(storage, first channel, last channel + 1, row stride) of an NHWC view."""
        rs = t.stride(2)
        lo = t.storage_offset() % rs if rs else 0
        return t.untyped_storage().data_ptr(), lo, lo + t.shape[3], rs

    def _overlaps(self, a, b):
        sa, la, ha, ra = self._footprint(a)
        sb, lb, hb, rb = self._footprint(b)
        if sa != sb:
            return False
        if ra != rb:
            return True  # differently strided views of one storage: assume they alias
        return la < hb and lb < ha

    def _writable(self, t) -> bool:
        """May backward overwrite t in place?  Not the caller's loss gradient (graph replays
        and repeated backward() read it again), and not a tensor a side-stream weight
        gradient still has to read (the side stream joins only at the end of the pass)."""
        if any(self._overlaps(t, lg) for lg in self.loss_grad.values()):
            return False
        return not any(self._overlaps(t, r) for r in self._side_reads)

    def _b_EltwiseSum(self, node):
        dy = self._incoming(node.outputs[0])
        self._add_grad(node.inputs[0], Plain(dy))
        cb = self.g.slots[node.inputs[1]].shape[1]
        self._add_grad(node.inputs[1], Plain(dy[..., :cb] if node.attrs.pad_channels else dy))

    def _b_AvgPool(self, node):
        head = self._nrp.get(node.id)
        if head is not None:  # pool bwd + ReLU bwd + BN gradient sums in one pass
            dy = self._incoming(node.outputs[0])
            x = self.acts[head.inputs[0]]
            st = self.stats[head.inputs[1]]
            m32, s32, b32, i32 = self.node_tables[head.id]
            dt1 = self._fresh_like(x)
            pixels = x.shape[0] * x.shape[1] * x.shape[2]
            tiles = self.L.bnff_sum_tiles(pixels)
            part = self._empty((tiles, 2, x.shape[3]), torch.float64)
            self._emit(self.L.bnff_pool_relu_bn_bwd, self.dcode, view_of(dy), view_of(x), view_of(dt1),
                       node.attrs.k, coef_of(m32, s32, b32, i32), _ptr(part),
                       what=f"pool_relu_bn_bwd {head.name}", nbytes=_nb(dy, x, dt1))
            mm, ii, k1, k2, gg = self._dx_coeffs(part, tiles, x.shape[3], pixels, st, head.attrs.bn, head.name)
            self._add_grad(head.inputs[0], Deferred(dt1, x, mm, ii, k1, k2, gg))
            self._nrp_done.add(head.id)
            return
        dy = self._incoming(node.outputs[0])
        x = self.acts[node.inputs[0]]
        if not self._wants_dx(node.inputs[0]):
            return
        dx = self._fresh_like(x)
        self._emit(self.L.bnff_avgpool_bwd, self.dcode, view_of(dy), view_of(dx), node.attrs.k,
                   what="avgpool_bwd", nbytes=_nb(dy, dx))
        self._add_grad(node.inputs[0], Plain(dx))

    # -------------------------------------------------------------- optimizer
    def _compile_optimizer(self):
        self._cur = self.opt
        if self.lr != 0.0:
            self._emit(self.L.bnff_sgd, _ptr(self.wflat), _ptr(self.gflat), self.wflat.numel(),
                       C.c_float(self.lr), what="sgd", nbytes=12 * self.wflat.numel())
        self.repack = []
        self._cur = self.repack
        # window-layout convs: one multi-tensor launch (job table resident on the device)
        jobs = []
        max_el = 0
        for name, (wf, wd, conv) in self.wpacks.items():
            if name in self.col_src:  # stem GEMM: (co, ci, kh, kw) -> (co, kpad) first
                w2, orig, kpad = self.col_src[name]
                self._emit(self.L.bnff_weight_to_cols, _ptr(self.param(f"{orig.name}.weight")),
                           orig.out_c, orig.in_c, orig.kh, orig.kw, kpad, _ptr(w2),
                           what="pack_weights")
                src = w2
            else:
                src = self.param(f"{name}.weight")
            jobs.append(_lib.PackJob(_ptr(src), _ptr(wf), _ptr(wd),
                                     conv.out_c, conv.in_c, conv.kh, conv.kw))
            max_el = max(max_el, wf.numel(), wd.numel())
        if jobs:
            arr = (_lib.PackJob * len(jobs))(*jobs)
            raw = bytes(memoryview(arr).cast("B"))
            self.pack_jobs = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(self.dev)
            self._bufs.append(self.pack_jobs)
            self._emit(self.L.bnff_pack_window_multi, self.dcode, len(jobs), _ptr(self.pack_jobs),
                       max_el, what="pack_weights")
        for name, (wp, wt, cin_s, conv) in self.packs.items():
            if name in self.wpacks:  # window kernels serve both passes of this conv
                continue
            self._emit(self.L.bnff_pack_weights, self.dcode, _ptr(self.param(f"{name}.weight")),
                       conv.out_c, conv.in_c, cin_s, conv.kh, conv.kw, _ptr(wp), _ptr(wt),
                       what="pack_weights")
        self._cur = None
        self.launch_counts["opt"] = len(self.opt) + len(self.repack)
        # initial packing of the current weights
        self._run(self.repack)

    # -------------------------------------------------------------------- run
    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)

    def _run(self, thunks):
        """Launch thunks in order on the current stream; side thunks go to the side stream,
        each forked from the current stream's position at that point, and the side stream
        is joined back before returning (also under CUDA-graph capture)."""
        main = torch.cuda.current_stream(self.dev)
        s = C.c_void_p(main.cuda_stream)
        side_used = False
        for t in thunks:
            if getattr(t, "side", False):
                if self._side is None:
                    self._side = torch.cuda.Stream(self.dev, priority=self.side_prio)
                ev = torch.cuda.Event()
                ev.record(main)
                self._side.wait_event(ev)
                t(C.c_void_p(self._side.cuda_stream))
                side_used = True
            else:
                t(s)
        if side_used:
            ev = torch.cuda.Event()
            ev.record(self._side)
            main.wait_event(ev)
        if getattr(self, "_comm_used", False):  # the bucketed gradient all-reduces
            ev = torch.cuda.Event()
            ev.record(self._comm)
            main.wait_event(ev)
            self._comm_used = False

    def set_input(self, x):
        """Graph input: NCHW fp32 (numpy or torch, host or device) -> padded NHWC."""
        sid = self.g.inputs[0]
        n, c, h, w = self.g.slots[sid].shape
        xt = torch.as_tensor(x)
        if tuple(xt.shape) != (n, c, h, w):
            raise ShapeError(f"input slot {sid}: shape {tuple(xt.shape)} != declared {(n, c, h, w)}")
        xt = xt.to(self.dev, torch.float32, non_blocking=True).contiguous()
        _lib.check(self.L.bnff_nchw_to_nhwc(self.dcode, _ptr(xt), n, c, h, w,
                                            view_of(self.acts[sid]), self._stream()), "input")
        self._keep_input = xt

    def set_loss_grad(self, dy):
        sid = self.g.outputs[0]
        n, c, h, w = self.g.slots[sid].shape
        dt = torch.as_tensor(dy).to(self.dev, torch.float32).contiguous()
        if tuple(dt.shape) != (n, c, h, w):
            raise ShapeError(f"loss grad slot {sid}: shape {tuple(dt.shape)} != {(n, c, h, w)}")
        _lib.check(self.L.bnff_nchw_to_nhwc(self.dcode, _ptr(dt), n, c, h, w,
                                            view_of(self.loss_grad[sid]), self._stream()), "dy")
        self._keep_dy = dt

    def forward(self):
        self._run(self.fwd)

    def backward(self):
        self._run(self.bwd)

    def optimizer_step(self):
        self._run(self.opt)
        self._run(self.repack)

    def step(self):
        """One training iteration: forward, backward, SGD (+ weight repack)."""
        if self.graph_exec is not None:
            self.graph_exec.replay()
            return
        self.forward()
        self.backward()
        self.optimizer_step()

    def capture(self, split: bool = False):
        """Capture the step as CUDA graph(s).  split=False: one graph forward+backward+
        SGD+repack (replayed by step()).  split=True: (fwd+bwd graph, optimizer graph),
        so a data-parallel wrapper can all-reduce the gradient buffer in between."""
        s = torch.cuda.Stream(self.dev, priority=self.main_prio)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            self.forward()
            self.backward()  # warm: first launches set kernel attributes
        torch.cuda.current_stream(self.dev).wait_stream(s)
        torch.cuda.synchronize(self.dev)
        if split:
            g1, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(g1):
                self.forward()
                self.backward()
            with torch.cuda.graph(g2):
                self._run(self.opt)
                self._run(self.repack)
            self.graph_parts = (g1, g2)
            return g1, g2
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            self.forward()
            self.backward()
            self._run(self.opt)
            self._run(self.repack)
        self.graph_exec = gr
        return gr

    def all_thunks(self):
        return list(self.fwd) + list(self.bwd) + list(self.opt) + list(self.repack)

    def profile_launches(self, reps: int = 3):
        """Per-launch device time: CUDA events recorded on the launching stream between
        consecutive launches (a separate pass, not the timed region).  Returns
        [(thunk, mean_ms)] in launch order."""
        thunks = self.all_thunks()
        s = self._stream()
        stream = torch.cuda.current_stream(self.dev)
        acc = [0.0] * len(thunks)
        for _ in range(reps):
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(thunks) + 1)]
            evs[0].record(stream)
            for i, t in enumerate(thunks):
                t(s)
                evs[i + 1].record(stream)
            torch.cuda.synchronize(self.dev)
            for i in range(len(thunks)):
                acc[i] += evs[i].elapsed_time(evs[i + 1])
        return [(t, a / reps) for t, a in zip(thunks, acc)]

    def num_launches(self) -> int:
        return (self.launch_counts["fwd"] + self.launch_counts["bwd"] + self.launch_counts["opt"])

    # --------------------------------------------------------------- readback
    def to_nchw(self, t: torch.Tensor, c_real: int | None = None) -> np.ndarray:
        a = t.float().permute(0, 3, 1, 2)
        if c_real is not None:
            a = a[:, :c_real]
        return a.contiguous().cpu().numpy()

    def output(self, sid=None) -> np.ndarray:
        sid = self.g.outputs[0] if sid is None else sid
        return self.to_nchw(self.acts[sid])

    def act(self, sid) -> np.ndarray:
        return self.to_nchw(self.acts[sid], self.g.slots[sid].shape[1])

    def input_grad_nchw(self, sid=None):
        sid = self.g.inputs[0] if sid is None else sid
        t = self.input_grads.get(sid)
        return None if t is None else self.to_nchw(t, self.input_c[sid])

    def param_grads(self) -> dict:
        host = self.gflat.cpu().numpy()
        out = {}
        for k in self.param_names:
            o, n = self.poff[k]
            out[k] = host[o:o + n].reshape(np.asarray(self.g.params[k]).shape)
        return out

    def params_now(self) -> dict:
        host = self.wflat.cpu().numpy()
        return {k: host[o:o + n].reshape(np.asarray(self.g.params[k]).shape)
                for k, (o, n) in self.poff.items()}

    def stats_of(self, stats_sid):
        st = self.stats[stats_sid]
        return {k: getattr(st, k).cpu().numpy() for k in ("sum", "sumsq", "mean", "var")}
