"""Operator-graph IR for the fused-DAG path (a superset of the reference IR).

The nine reference kinds keep their exact meaning, attributes and shape rules
(/root/reference/pkg/src/dagfuse/graph_ir.py:8-21, 243-314).  Extension kinds
let the north-star CNNs be written down without approximation:

    kind            attrs                                       inputs
    conv2d          + groups (default 1), kernel_h/kernel_w,    1
                      stride_h/stride_w, padding_h/padding_w
    maxpool2d       + padding (default 0; pads with -inf)       1
    avgpool2d       kernel, stride (default kernel), padding,   1
                    count_include_pad (default 1)
    hardswish       -                                           1
    hardsigmoid     -                                           1
    silu            -                                           1
    sigmoid         -                                           1
    channel_scale   -   (C,H,W) x (C,) -> (C,H,W)               2
    gelu            -   exact (erf) GELU                        1
    tokens          weights class_token (C,), pos_embedding     1
                    (1+H*W, C):  (C,H,W) -> (1+H*W, C), row 0 the class
                    token, row 1+h*W+w the pixel (h, w); + pos_embedding
    layernorm       epsilon (default 1e-5); weights gamma,      1
                    beta (C,): normalise over the last axis
    attention       heads:  (L, 3C) packed q|k|v -> (L, C),     1
                    per head softmax(q k^T / sqrt(C/heads)) v
    select_token    index (default 0):  (L, C) -> (C,)          1
    dense           + a rank-2 input (L, fan_in) -> (L, units) (row-wise)

Tensors are single-sample, rank 1, 2 (L, C: token sequences) or 3 (C,H,W);
byte sizes count 32-bit elements exactly like the reference
(graph_ir.py:82-84), so the liveness plan below reproduces
``peak_activation_bytes`` (graph_ir.py:486-512).
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field
from typing import Callable, Iterable, Mapping

import numpy as np

from .errors import CycleDetected, ShapeMismatch

REFERENCE_KINDS = (
    "dense", "conv2d", "relu", "maxpool2d", "batchnorm_inference",
    "residual_add", "global_avg_pool", "flatten", "concat",
)
EXTENSION_KINDS = (
    "avgpool2d", "hardswish", "hardsigmoid", "silu", "sigmoid", "channel_scale",
    "gelu", "tokens", "layernorm", "attention", "select_token",
)
KINDS = REFERENCE_KINDS + EXTENSION_KINDS
ACTIVATION_KINDS = ("relu", "hardswish", "hardsigmoid", "silu", "sigmoid", "gelu")
VARIADIC_KINDS = ("residual_add", "concat")       # >= 2 inputs
BINARY_KINDS = ("channel_scale",)                  # exactly 2 inputs
SINGLE_INPUT_KINDS = tuple(k for k in KINDS if k not in VARIADIC_KINDS + BINARY_KINDS)

DEFAULT_BN_EPSILON = 1e-5
MIB = 1 << 20


def mib_ceil(nbytes: int) -> int:
    return int(math.ceil(nbytes / MIB))


@dataclass(frozen=True)
class TensorSpec:
    """Dims of one single-sample fp32 tensor (graph_ir.py:62-84)."""

    dims: tuple[int, ...]

    def __post_init__(self):
        dims = tuple(int(d) for d in self.dims)
        if len(dims) == 0 or min(dims) < 1:
            raise ValueError(f"dims must be non-empty positive integers, got {self.dims!r}")
        object.__setattr__(self, "dims", dims)

    @property
    def rank(self) -> int:
        return len(self.dims)

    @property
    def element_count(self) -> int:
        n = 1
        for d in self.dims:
            n *= d
        return n

    @property
    def byte_size(self) -> int:
        return 4 * self.element_count


@dataclass(frozen=True)
class OpNode:
    node_id: str
    kind: str
    attrs: Mapping[str, float] = field(default_factory=dict)
    weight_refs: Mapping[str, str] = field(default_factory=dict)
    inputs: tuple[str, ...] = ()

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown node kind {self.kind!r}")
        object.__setattr__(self, "attrs", dict(self.attrs))
        object.__setattr__(self, "weight_refs", dict(self.weight_refs))
        object.__setattr__(self, "inputs", tuple(self.inputs))


class WeightStore:
    """name -> (TensorSpec, read-only flat float32), graph_ir.py:105-149."""

    def __init__(self, tensors: Mapping[str, tuple[TensorSpec, np.ndarray]] | None = None):
        self._t: dict[str, tuple[TensorSpec, np.ndarray]] = {}
        for name, (spec, values) in (tensors or {}).items():
            self.put(name, spec, values)

    def put(self, name: str, spec: TensorSpec, values) -> None:
        flat = np.asarray(values, dtype=np.float32).reshape(-1)
        if flat.size != spec.element_count:
            raise ValueError(f"weight {name!r}: {flat.size} values for shape {spec.dims} "
                             f"({spec.element_count} expected)")
        if flat.flags.writeable:
            flat = flat.view()
            flat.setflags(write=False)
        self._t[name] = (spec, flat)

    def __contains__(self, name) -> bool:
        return name in self._t

    def __len__(self) -> int:
        return len(self._t)

    def names(self) -> list[str]:
        return list(self._t)

    def spec(self, name: str) -> TensorSpec:
        return self._t[name][0]

    def values(self, name: str) -> np.ndarray:
        return self._t[name][1]

    def array(self, name: str) -> np.ndarray:
        spec, flat = self._t[name]
        return flat.reshape(spec.dims)

    def items(self):
        return self._t.items()

    @property
    def byte_size(self) -> int:
        return sum(spec.byte_size for spec, _ in self._t.values())


class ModelGraph:
    """One model: named nodes, an entry fed by the external input, an exit."""

    def __init__(self, model_id: str, nodes: Iterable[OpNode], entry: str, exit: str,
                 input_spec: TensorSpec, output_spec: TensorSpec):
        table: dict[str, OpNode] = {}
        for n in nodes:
            if n.node_id in table:
                raise ValueError(f"duplicate node id {n.node_id!r}")
            table[n.node_id] = n
        self.model_id = model_id
        self.nodes = table
        self.entry, self.exit = entry, exit
        self.input_spec, self.output_spec = input_spec, output_spec

    @property
    def edges(self) -> frozenset[tuple[str, str]]:
        return frozenset((s, n.node_id) for n in self.nodes.values() for s in n.inputs)

    def node_count(self) -> int:
        return len(self.nodes)

    def __repr__(self):
        return f"ModelGraph({self.model_id!r}, {len(self.nodes)} nodes)"


@dataclass(frozen=True)
class Problem:
    code: str
    node_id: str
    message: str

    def __str__(self):
        return f"{self.code}{f' [{self.node_id}]' if self.node_id else ''}: {self.message}"


@dataclass
class ValidationReport:
    model_id: str
    problems: list[Problem]

    @property
    def ok(self) -> bool:
        return not self.problems


# --------------------------------------------------------------------------
# ordering

def topo_order(g) -> list[str]:
    """Kahn's algorithm with a min-heap on node_id strings (graph_ir.py:216-236).

    The string tie-break is part of the contract: the liveness plan and the
    reference plan it must equal are both defined over this exact order.
    """
    pending = {nid: len(n.inputs) for nid, n in g.nodes.items()}
    users: dict[str, list[str]] = {nid: [] for nid in g.nodes}
    for nid, n in g.nodes.items():
        for src in n.inputs:
            if src in users:
                users[src].append(nid)
    heap = [nid for nid, k in pending.items() if k == 0]
    heapq.heapify(heap)
    out: list[str] = []
    while heap:
        nid = heapq.heappop(heap)
        out.append(nid)
        for u in users[nid]:
            pending[u] -= 1
            if pending[u] == 0:
                heapq.heappush(heap, u)
    if len(out) != len(g.nodes):
        raise CycleDetected(g.model_id)
    return out


# --------------------------------------------------------------------------
# per-kind geometry

def hw_attr(attrs: Mapping, name: str, default: int) -> tuple[int, int]:
    """(h, w) pair of a square-or-rectangular attribute (``kernel`` etc.)."""
    base = int(attrs.get(name, default))
    return int(attrs.get(f"{name}_h", base)), int(attrs.get(f"{name}_w", base))


def conv_geometry(attrs: Mapping):
    kh, kw = hw_attr(attrs, "kernel", 1)
    sh, sw = hw_attr(attrs, "stride", 1)
    ph, pw = hw_attr(attrs, "padding", 0)
    return kh, kw, sh, sw, ph, pw


def pool_geometry(attrs: Mapping):
    kh, kw = hw_attr(attrs, "kernel", 1)
    sh, sw = int(attrs.get("stride_h", attrs.get("stride", kh))), \
        int(attrs.get("stride_w", attrs.get("stride", kw)))
    ph, pw = hw_attr(attrs, "padding", 0)
    return kh, kw, sh, sw, ph, pw


def _window_out(extent: int, k: int, s: int, p: int) -> int:
    return (extent + 2 * p - k) // s + 1


def _need_chw(node: OpNode, dims) -> None:
    if len(dims) != 3:
        raise ShapeMismatch(node.node_id, f"{node.kind} expects (C,H,W), got {dims}")


def _shape_dense(node, ins):
    (d,) = ins
    if len(d) not in (1, 2):
        raise ShapeMismatch(node.node_id, f"dense expects a rank-1 (or token rank-2) input, got {d}")
    fan_in = int(node.attrs["fan_in"])
    if d[-1] != fan_in:
        raise ShapeMismatch(node.node_id, f"fan_in {fan_in} but input has {d[-1]} features")
    return tuple(d[:-1]) + (int(node.attrs["units"]),)


def _shape_tokens(node, ins):
    (d,) = ins
    _need_chw(node, d)
    return (1 + d[1] * d[2], d[0])


def _shape_layernorm(node, ins):
    (d,) = ins
    if len(d) not in (1, 2):
        raise ShapeMismatch(node.node_id, f"layernorm expects (C,) or (L, C), got {d}")
    return d


def _shape_attention(node, ins):
    (d,) = ins
    heads = int(node.attrs["heads"])
    if len(d) != 2 or d[1] % 3 or (d[1] // 3) % heads:
        raise ShapeMismatch(node.node_id, f"attention expects (L, 3C) with C % heads == 0, got {d}")
    return (d[0], d[1] // 3)


def _shape_select_token(node, ins):
    (d,) = ins
    idx = int(node.attrs.get("index", 0))
    if len(d) != 2 or not 0 <= idx < d[0]:
        raise ShapeMismatch(node.node_id, f"select_token {idx} of {d}")
    return (d[1],)


def _shape_conv(node, ins):
    (d,) = ins
    _need_chw(node, d)
    kh, kw, sh, sw, ph, pw = conv_geometry(node.attrs)
    groups = int(node.attrs.get("groups", 1))
    cout = int(node.attrs["out_channels"])
    if groups < 1 or d[0] % groups or cout % groups:
        raise ShapeMismatch(node.node_id, f"groups {groups} incompatible with {d[0]}->{cout}")
    oh, ow = _window_out(d[1], kh, sh, ph), _window_out(d[2], kw, sw, pw)
    if oh < 1 or ow < 1:
        raise ShapeMismatch(node.node_id, f"kernel {kh}x{kw} too large for input {d}")
    return (cout, oh, ow)


def _shape_pool(node, ins):
    (d,) = ins
    _need_chw(node, d)
    kh, kw, sh, sw, ph, pw = pool_geometry(node.attrs)
    if ph * 2 > kh or pw * 2 > kw:
        raise ShapeMismatch(node.node_id, "pool padding exceeds half the window")
    oh, ow = _window_out(d[1], kh, sh, ph), _window_out(d[2], kw, sw, pw)
    if oh < 1 or ow < 1:
        raise ShapeMismatch(node.node_id, f"window {kh}x{kw} too large for input {d}")
    return (d[0], oh, ow)


def _shape_same(node, ins):
    return ins[0]


def _shape_add(node, ins):
    first = ins[0]
    for d in ins[1:]:
        if d != first:
            raise ShapeMismatch(node.node_id, f"addend shapes differ: {first} vs {d}")
    return first


def _shape_gap(node, ins):
    (d,) = ins
    _need_chw(node, d)
    return (d[0],)


def _shape_flatten(node, ins):
    n = 1
    for x in ins[0]:
        n *= x
    return (n,)


def _shape_concat(node, ins):
    first = ins[0]
    for d in ins:
        if len(d) != len(first) or d[1:] != first[1:]:
            raise ShapeMismatch(node.node_id, f"concat shapes incompatible: {first} vs {d}")
    return (sum(d[0] for d in ins),) + tuple(first[1:])


def _shape_channel_scale(node, ins):
    x, s = ins
    _need_chw(node, x)
    if s != (x[0],):
        raise ShapeMismatch(node.node_id, f"scale {s} does not match channels of {x}")
    return x


_SHAPE: dict[str, Callable] = {
    "dense": _shape_dense, "conv2d": _shape_conv, "maxpool2d": _shape_pool,
    "avgpool2d": _shape_pool, "batchnorm_inference": _shape_same,
    "residual_add": _shape_add, "global_avg_pool": _shape_gap, "flatten": _shape_flatten,
    "concat": _shape_concat, "channel_scale": _shape_channel_scale,
    "tokens": _shape_tokens, "layernorm": _shape_layernorm, "attention": _shape_attention,
    "select_token": _shape_select_token,
    **{k: _shape_same for k in ACTIVATION_KINDS},
}


def node_output_dims(node: OpNode, input_dims: list[tuple[int, ...]]) -> tuple[int, ...]:
    n = len(input_dims)
    if node.kind in SINGLE_INPUT_KINDS and n != 1:
        raise ShapeMismatch(node.node_id, f"{node.kind} takes exactly one input, got {n}")
    if node.kind in VARIADIC_KINDS and n < 2:
        raise ShapeMismatch(node.node_id, f"{node.kind} takes at least two inputs")
    if node.kind in BINARY_KINDS and n != 2:
        raise ShapeMismatch(node.node_id, f"{node.kind} takes exactly two inputs")
    return tuple(int(x) for x in _SHAPE[node.kind](node, [tuple(d) for d in input_dims]))


def node_input_dims(g, nid: str, shapes: Mapping[str, TensorSpec]) -> list[tuple[int, ...]]:
    if nid == g.entry:
        return [g.input_spec.dims]
    return [shapes[s].dims for s in g.nodes[nid].inputs]


def infer_shapes(g) -> dict[str, TensorSpec]:
    """Output spec of every node, in topo order (graph_ir.py:317-339)."""
    out: dict[str, TensorSpec] = {}
    for nid in topo_order(g):
        node = g.nodes[nid]
        if nid == g.entry:
            if node.inputs:
                raise ShapeMismatch(nid, "entry node must not have predecessors")
            ins = [g.input_spec.dims]
        else:
            unknown = [s for s in node.inputs if s not in g.nodes]
            if unknown:
                raise ShapeMismatch(nid, f"unknown predecessor(s) {unknown}")
            if not node.inputs:
                raise ShapeMismatch(nid, "only the entry node may have no predecessors")
            ins = [out[s].dims for s in node.inputs]
        out[nid] = TensorSpec(node_output_dims(node, ins))
    return out


def expected_weight_shapes(node: OpNode, input_dims) -> dict[str, tuple[tuple[int, ...], bool]]:
    """role -> (dims, required) (graph_ir.py:342-360, plus grouped conv)."""
    a = node.attrs
    if node.kind == "dense":
        u, f = int(a["units"]), int(a["fan_in"])
        return {"weight": ((u, f), True), "bias": ((u,), False)}
    if node.kind == "conv2d":
        kh, kw, *_ = conv_geometry(a)
        cout, groups = int(a["out_channels"]), int(a.get("groups", 1))
        cin = input_dims[0][0]
        return {"weight": ((cout, cin // groups, kh, kw), True), "bias": ((cout,), False)}
    if node.kind == "batchnorm_inference":
        per = ((input_dims[0][0],), True)
        return {"gamma": per, "beta": per, "mean": per, "var": per}
    if node.kind == "layernorm":
        per = ((input_dims[0][-1],), True)
        return {"gamma": per, "beta": per}
    if node.kind == "tokens":
        c, h, w = input_dims[0]
        return {"class_token": ((c,), True), "pos_embedding": ((1 + h * w, c), True)}
    return {}


def validate_graph(g: ModelGraph, w: WeightStore) -> ValidationReport:
    """Structural + weight checks, same problem codes as graph_ir.py:363-462."""
    probs: list[Problem] = []

    def add(code, nid, msg):
        probs.append(Problem(code, nid, msg))

    for role, nid in (("entry", g.entry), ("exit", g.exit)):
        if nid not in g.nodes:
            add(f"missing-{role}", nid, f"{role} node not present")
    if probs:
        return ValidationReport(g.model_id, probs)

    dangling = False
    for nid, node in sorted(g.nodes.items()):
        for src in node.inputs:
            if src not in g.nodes:
                add("dangling-edge", nid, f"input {src!r} is not a node")
                dangling = True
    order = None
    if not dangling:
        try:
            order = topo_order(g)
        except CycleDetected:
            add("cycle", "", "cycle detected")

    for nid, node in sorted(g.nodes.items()):
        k = len(node.inputs)
        if nid == g.entry:
            if k:
                add("entry-arity", nid, "entry node must have no predecessors")
            if node.kind not in SINGLE_INPUT_KINDS:
                add("arity", nid, f"entry consumes one external input; {node.kind} cannot")
        elif node.kind in SINGLE_INPUT_KINDS and k != 1:
            add("arity", nid, f"{node.kind} takes exactly 1 input, has {k}")
        elif node.kind in VARIADIC_KINDS and k < 2:
            add("arity", nid, f"{node.kind} takes >= 2 inputs, has {k}")
        elif node.kind in BINARY_KINDS and k != 2:
            add("arity", nid, f"{node.kind} takes exactly 2 inputs, has {k}")
    if probs:
        return ValidationReport(g.model_id, probs)

    users: dict[str, list[str]] = {nid: [] for nid in g.nodes}
    for nid, node in g.nodes.items():
        for src in node.inputs:
            users[src].append(nid)
    seen = {g.entry}
    for nid in order:
        if nid in seen:
            seen.update(users[nid])
    for nid in sorted(set(g.nodes) - seen):
        add("unreachable", nid, "not reachable from entry")

    try:
        shapes = infer_shapes(g)
    except ShapeMismatch as exc:
        add("shape", exc.node_id, str(exc))
        return ValidationReport(g.model_id, probs)
    if shapes[g.exit].dims != g.output_spec.dims:
        add("output-spec", g.exit,
            f"exit produces {shapes[g.exit].dims}, declared {g.output_spec.dims}")

    for nid in order:
        node = g.nodes[nid]
        expect = expected_weight_shapes(node, node_input_dims(g, nid, shapes))
        for role, ref in sorted(node.weight_refs.items()):
            if role not in expect:
                add("weight-role", nid, f"{node.kind} takes no {role!r} weight")
            elif ref not in w:
                add("weight-missing", nid, f"weight {ref!r} not in store")
            elif w.spec(ref).dims != expect[role][0]:
                add("weight-shape-mismatch", nid,
                    f"{role}={ref!r} has shape {w.spec(ref).dims}, expected {expect[role][0]}")
        for role, (_, required) in sorted(expect.items()):
            if required and role not in node.weight_refs:
                add("weight-ref-missing", nid, f"{node.kind} requires a {role!r} weight ref")
    return ValidationReport(g.model_id, probs)


def node_flops(node: OpNode, input_dims, output_dims) -> int:
    """Multiply-add count (x2) as in graph_ir.py:465-483; grouped conv divides Cin."""
    out = 1
    for d in output_dims:
        out *= int(d)
    a = node.attrs
    if node.kind == "dense":
        return 2 * int(a["fan_in"]) * out          # = 2 * fan_in * units for rank-1
    if node.kind == "attention":                   # q k^T and p v
        seq = int(output_dims[0])
        return 4 * seq * out
    if node.kind == "conv2d":
        kh, kw, *_ = conv_geometry(a)
        cin = input_dims[0][0] // int(a.get("groups", 1))
        return 2 * cin * kh * kw * out
    if node.kind in VARIADIC_KINDS:
        return out * max(len(input_dims) - 1, 1)
    if node.kind == "batchnorm_inference":
        return 4 * out
    if node.kind in ("maxpool2d", "avgpool2d"):
        kh, kw, *_ = pool_geometry(a)
        return kh * kw * out
    if node.kind == "global_avg_pool":
        n = 1
        for d in input_dims[0]:
            n *= int(d)
        return n
    return out


def gemm_flops(g, shapes=None) -> int:
    """Sum of conv2d + dense + attention FLOPs of one graph (the tensor-core work)."""
    shapes = shapes or infer_shapes(g)
    total = 0
    for nid, node in g.nodes.items():
        if node.kind in ("conv2d", "dense", "attention"):
            total += node_flops(node, node_input_dims(g, nid, shapes), shapes[nid].dims)
    return total


# --------------------------------------------------------------------------
# liveness (the reference plan, restated as explicit intervals)

@dataclass(frozen=True)
class LiveInterval:
    """One tensor's lifetime over topo positions, both ends inclusive.

    ``first = -1`` is the external input; ``last = len(order)`` is the exit.
    """

    name: str
    size: int
    first: int
    last: int


def liveness_intervals(g, shapes=None, order=None) -> list[LiveInterval]:
    """Producer -> last-consumer intervals exactly as graph_ir.py:494-506 defines them.

    Entry 0 is the external input, live over [-1, pos(entry)]; every node's
    output is live from its own position to its last consumer's position (or
    its own when unused); the exit output stays live to ``len(order)``.
    """
    shapes = shapes or infer_shapes(g)
    order = order or topo_order(g)
    pos = {nid: i for i, nid in enumerate(order)}
    last = dict(pos)
    for nid, node in g.nodes.items():
        for src in node.inputs:
            if pos[nid] > last[src]:
                last[src] = pos[nid]
    last[g.exit] = len(order)
    ivs = [LiveInterval("<input>", g.input_spec.byte_size, -1, pos[g.entry])]
    ivs += [LiveInterval(nid, shapes[nid].byte_size, pos[nid], last[nid]) for nid in order]
    return ivs


def peak_from_intervals(ivs: list[LiveInterval], n_positions: int) -> int:
    """Peak of the reference sweep (graph_ir.py:503-511) over explicit intervals.

    The sweep adds a tensor at its first position, samples, then frees the
    tensors whose last position is the current one — so at position i the
    live set is {iv : first <= i <= last} plus the input before it is freed.
    Position -1 contributes the input alone.
    """
    delta = np.zeros(n_positions + 2, dtype=np.int64)
    for iv in ivs:
        lo = iv.first + 1
        hi = min(iv.last, n_positions - 1) + 1
        if lo <= hi:
            delta[lo] += iv.size
            delta[hi + 1] -= iv.size
    live = np.cumsum(delta)[: n_positions + 1]
    return int(live.max()) if live.size else 0


def peak_activation_bytes(g, shapes=None) -> int:
    order = topo_order(g)
    return peak_from_intervals(liveness_intervals(g, shapes, order), len(order))
