"""Main-memory sweep accounting on the reference's rulebook, next to what the device runs.

The reference charges every node kind a fixed pattern of full-tensor sweeps
(``traffic.py:1-39`` documents it, ``node_sweep_rules`` / ``count_sweeps`` at
``traffic.py:128-231``); a sweep of slot s costs ``numel(s) * bytes_per_elem``.  This
module restates that rulebook as a table (one row per node kind: which slots are read /
written how many times in each pass), so the algorithmic side of every traffic claim here
is the reference's own definition, and adds the two device-side ledgers it is compared
with:

* ``device_ledger(engine)`` -- the bytes each launch of the compiled engine must touch
  (each tensor once per launch, ``Engine._emit``'s ``nbytes``), attributed to the graph
  node that emitted it;
* ``ncu_ledger(csv, engine)`` -- the DRAM bytes ncu measured for those launches, mapped
  launch by launch (tools/ncu_node_ledger.py brackets every thunk with a marker kernel).

``compare(...)`` lines the three up node by node, in the style of ``compare_ledgers``
(``traffic.py:355-365``).  Reports mirror ``bnfuse traffic`` (``cli.py:247-274``): one CSV
per level (node_id, kind, pass, reads, writes, bytes) and a summary JSON.
"""

from __future__ import annotations

import csv
import io
import json
from dataclasses import dataclass, field

from . import graph as G

FWD, BWD = "forward", "backward"

# (pass, slot role, direction, sweeps, role label): slot roles are "in" (inputs[0]),
# "in1" (inputs[1]), "ins" (every input), "out" (outputs[0]), "saved" (outputs[1]),
# "outs" (every output).  Weights are charged separately (conv kinds).
_CONV = ((FWD, "in", "read", 1, "ifmap"), (FWD, "out", "write", 1, "ofmap"),
         (BWD, "out", "read", 2, "grad_out"), (BWD, "in", "read", 1, "saved"),
         (BWD, "in", "write", 1, "grad_in"))
_RULES = {
    G.CONV: _CONV,
    G.FUSED_CONV_STATS: _CONV,
    G.RELU: ((FWD, "in", "read", 1, "ifmap"), (FWD, "out", "write", 1, "ofmap"),
             (BWD, "out", "read", 1, "grad_out"), (BWD, "in", "read", 1, "saved"),
             (BWD, "in", "write", 1, "grad_in")),
    G.SUBBN2: ((FWD, "in", "read", 1, "ifmap"), (FWD, "out", "write", 1, "ofmap"),
               (BWD, "out", "read", 1, "grad_out"), (BWD, "in", "read", 1, "saved")),
    G.FUSED_NRC: ((FWD, "in", "read", 1, "ifmap"), (FWD, "saved", "write", 1, "saved"),
                  (FWD, "out", "write", 1, "ofmap"), (BWD, "out", "read", 2, "grad_out"),
                  (BWD, "saved", "read", 1, "saved"), (BWD, "in", "write", 1, "grad_in")),
    G.SPLIT: ((BWD, "outs", "read", 1, "grad_out"), (BWD, "in", "write", 1, "grad_in")),
    G.EWS: ((FWD, "in", "read", 1, "ifmap"), (FWD, "in1", "read", 1, "ifmap"),
            (FWD, "out", "write", 1, "ofmap")),
    G.POOL: ((FWD, "in", "read", 1, "ifmap"), (FWD, "out", "write", 1, "ofmap"),
             (BWD, "out", "read", 1, "grad_out"), (BWD, "in", "write", 1, "grad_in")),
    G.FUSED_CONCAT_STATS: (),
}
_PHYSICAL_CONCAT = ((FWD, "ins", "read", 1, "ifmap"), (FWD, "out", "write", 1, "ofmap"),
                    (BWD, "out", "read", 1, "grad_out"), (BWD, "ins", "write", 1, "grad_in"))


def _rules(node, concat_physical):
    kind = node.kind
    if kind == G.BN:  # two-pass statistics read x three times, one-pass twice
        reads = 2 if node.attrs.onepass else 3
        return ((FWD, "in", "read", reads, "ifmap"), (FWD, "out", "write", 1, "ofmap"),
                (BWD, "out", "read", 2, "grad_out"), (BWD, "in", "read", 2, "saved"),
                (BWD, "in", "write", 1, "grad_in"))
    if kind == G.SUBBN1:
        if node.attrs.defer_backward:
            return ((FWD, "in", "read", 1, "ifmap"),)
        return ((FWD, "in", "read", 1, "ifmap"), (BWD, "in", "read", 1, "grad_in"),
                (BWD, "in", "read", 1, "saved"), (BWD, "in", "write", 1, "grad_in"))
    if kind == G.CONCAT:
        physical = node.attrs.physical if concat_physical is None else concat_physical
        return _PHYSICAL_CONCAT if physical else ()
    if kind not in _RULES:
        raise ValueError(f"no sweep rule for node kind {kind}")
    return _RULES[kind]


def _slots(node, role):
    return {"in": node.inputs[:1], "in1": node.inputs[1:2], "ins": node.inputs,
            "out": node.outputs[:1], "saved": node.outputs[1:2], "outs": node.outputs}[role]


@dataclass
class Sweep:
    node_id: int
    kind: str
    pass_: str
    slot: int          # -1: weight traffic
    direction: str
    sweeps: int
    bytes: int
    role: str = ""


@dataclass
class Ledger:
    entries: list = field(default_factory=list)

    def total_bytes(self, pass_=None):
        return sum(e.bytes for e in self.entries if pass_ is None or e.pass_ == pass_)

    def weight_bytes(self, pass_=None):
        return sum(e.bytes for e in self.entries if e.role == "weights" and (pass_ is None or e.pass_ == pass_))

    def bytes_by_kind(self):
        out: dict = {}
        for e in self.entries:
            out[e.kind] = out.get(e.kind, 0) + e.bytes
        return out

    def bytes_by_node(self, pass_=None):
        out: dict = {}
        for e in self.entries:
            if pass_ is None or e.pass_ == pass_:
                out[e.node_id] = out.get(e.node_id, 0) + e.bytes
        return out

    def key_map(self):
        """(node, pass, slot, direction) -> sweeps, weight entries excluded (traffic.py:110-118)."""
        out: dict = {}
        for e in self.entries:
            if e.role != "weights":
                k = (e.node_id, e.pass_, e.slot, e.direction)
                out[k] = out.get(k, 0) + e.sweeps
        return out


def count_sweeps(g, concat_physical=None, bytes_per_elem: int = 4) -> Ledger:
    """The reference rulebook applied to every node (traffic.py:222-231); bytes at
    ``bytes_per_elem`` (the reference's 4; the bf16 device path stores 2)."""
    led = Ledger()
    for node in g.nodes:
        for pass_, role_slots, direction, sweeps, role in _rules(node, concat_physical):
            for sid in _slots(node, role_slots):
                slot = g.slots[sid]
                if slot.kind != "feature" or sweeps <= 0:
                    continue
                led.entries.append(Sweep(node.id, node.kind, pass_, sid, direction, sweeps,
                                         sweeps * slot.numel * bytes_per_elem, role))
        conv = getattr(node.attrs, "conv", None)
        if conv is not None and node.kind in G.CONV_GROUP:  # weights: read fwd, read + write bwd
            wb = (conv.weights.size + conv.bias.size) * 4
            led.entries += [Sweep(node.id, node.kind, FWD, -1, "read", 1, wb, "weights"),
                            Sweep(node.id, node.kind, BWD, -1, "read", 1, wb, "weights"),
                            Sweep(node.id, node.kind, BWD, -1, "write", 1, wb, "weights")]
    return led


def compare_ledgers(analytic: Ledger, measured: Ledger) -> list:
    """Node-for-node sweep comparison (traffic.py:355-365): human-readable divergences."""
    a, m = analytic.key_map(), measured.key_map()
    out = []
    for key in sorted(set(a) | set(m)):
        if a.get(key, 0) != m.get(key, 0):
            nid, pass_, slot, direction = key
            out.append(f"node {nid} {pass_} slot {slot} {direction}: analytic {a.get(key, 0)} "
                       f"!= measured {m.get(key, 0)}")
    return out


# ---------------------------------------------------------------------------
# reports (bnfuse traffic, cli.py:247-274)
# ---------------------------------------------------------------------------
CSV_HEADER = ["node_id", "kind", "pass", "reads", "writes", "bytes"]


def to_csv(led: Ledger) -> str:
    agg: dict = {}
    for e in led.entries:
        row = agg.setdefault((e.node_id, e.kind, e.pass_), [0, 0, 0])
        if e.role != "weights":
            row[0 if e.direction == "read" else 1] += e.sweeps
        row[2] += e.bytes
    buf = io.StringIO()
    wr = csv.writer(buf)
    wr.writerow(CSV_HEADER)
    for (nid, kind, pass_), (r, w, b) in sorted(agg.items()):
        wr.writerow([nid, kind, pass_, r, w, b])
    return buf.getvalue()


def summary(led: Ledger, level: str, model: str, baseline: Ledger | None = None) -> dict:
    conv = sum(e.bytes for e in led.entries if e.kind in G.CONV_GROUP)
    relu = led.bytes_by_kind().get(G.RELU, 0)
    out = {"level": level, "model": model, "forward_bytes": led.total_bytes(FWD),
           "backward_bytes": led.total_bytes(BWD), "total_bytes": led.total_bytes(),
           "weight_bytes": led.weight_bytes(), "conv_group_bytes": conv,
           "non_conv_bytes": led.total_bytes() - conv}
    if baseline is not None:
        out["reduction_vs_baseline"] = 1.0 - led.total_bytes() / baseline.total_bytes()
        out["relu_share_of_baseline"] = baseline.bytes_by_kind().get(G.RELU, 0) / baseline.total_bytes()
    out["relu_share"] = relu / max(led.total_bytes(), 1)
    return out


# ---------------------------------------------------------------------------
# device side
# ---------------------------------------------------------------------------
def device_ledger(engine) -> dict:
    """node id -> algorithmic bytes the engine's launches touch (each tensor once per
    launch), per pass; launches not tied to a node (optimizer, repack) under -1."""
    out: dict = {}
    for pass_, thunks in ((FWD, engine.fwd), (BWD, engine.bwd), ("optimizer", engine.opt + engine.repack)):
        for t in thunks:
            nid = getattr(t, "node_id", -1)
            d = out.setdefault(nid, {FWD: 0, BWD: 0, "optimizer": 0})
            d[pass_] += int(getattr(t, "nbytes", 0))
    return out


def ncu_ledger(rows, engine) -> dict:
    """Map an ncu per-kernel list (launch order, each thunk preceded by one
    ``mark_kernel`` launch; tools/ncu_node_ledger.py) to node id -> measured DRAM bytes.
    ``rows``: [(kernel_name, dram_bytes)] in launch order."""
    thunks = engine.all_thunks()
    out: dict = {}
    ti = -1
    for name, nbytes in rows:
        if "mark_kernel" in name:
            ti += 1
            continue
        if ti < 0 or ti >= len(thunks):
            continue
        nid = getattr(thunks[ti], "node_id", -1)
        out[nid] = out.get(nid, 0.0) + float(nbytes)
    return out


def compare(g, analytic: Ledger, device: dict, measured: dict | None = None) -> list:
    """Per node: kind, rulebook bytes, device algorithmic bytes, ncu DRAM bytes."""
    by_node = analytic.bytes_by_node()
    rows = []
    for node in g.nodes:
        dv = device.get(node.id, {})
        rows.append({"node_id": node.id, "kind": node.kind, "name": node.name,
                     "rulebook_bytes": by_node.get(node.id, 0),
                     "device_bytes": dv.get(FWD, 0) + dv.get(BWD, 0),
                     "ncu_bytes": None if measured is None else measured.get(node.id, 0.0)})
    return rows


def to_json(obj) -> str:
    return json.dumps(obj, indent=2, sort_keys=True)
