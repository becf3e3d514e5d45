"""Lowering: one member graph -> a sequence of libdfx kernel launches.

Input: a validated ``ModelGraph`` + ``WeightStore`` (reference IR superset).
Output: a batch-independent ``MemberProgram``:

* **chains** — every launch is an *anchor* node plus the single-consumer
  nodes folded into its epilogue, in this slot order (dfx.h dfx_epilogue):
  ``affine`` (bias, batch-norm) -> ``act1`` -> ``binop`` (residual_add /
  channel_scale with an operand materialised earlier) -> ``act2``.
  Anchors: conv2d/dense -> tcgen05 implicit GEMM; depthwise conv2d ->
  dwconv; pools -> pool; global_avg_pool -> gap; batchnorm / activations /
  residual_add / channel_scale -> elementwise.  flatten is a view; concat is
  zero-copy (producers write at a channel offset of one buffer) with a copy
  launch only for parts that cannot be placed (misaligned offset, the graph
  input, a value already placed elsewhere).
* **buffers** — physical bf16 NHWC tensors (one per materialised value or
  concat group) with launch-index lifetimes for the activation planner.
* **blobs** — packed weights (bf16 GEMM matrices in (r, s, channel-block)
  K order, fp32 epilogue vectors, fp32 depthwise taps) for the weight arena.

Semantics are the reference's per-kind definitions
(/root/reference/pkg/src/dagfuse/executor.py:56-167, extension kinds as in
graph_ir.py).  Folding batch-norm into (alpha, beta) and the bf16 storage of
activations are the only numerical departures; parity is checked against the
oracle within the north-star tolerance.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

from .errors import UnsupportedOnDevice
from .graph_ir import (ACTIVATION_KINDS, conv_geometry, infer_shapes, pool_geometry,
                       topo_order)

GEMM, DWCONV, POOL, GAP, EW, COPY, SE = "gemm", "dwconv", "pool", "gap", "ew", "copy", "se"
DWSE = "dwse"            # depthwise conv -> SE gate -> channel scale, one launch
LN, TOKENS, ATTN = "ln", "tokens", "attn"      # token (ViT) launches, dfx_vit.cu
SE_MAX_C, SE_MAX_CR = 4096, 512          # limits of dfx_fused.cu se_kernel
# fold the gate's channel_scale into the SE launch (DFX_SE_FUSE=0: off, A/B).  With 8-CTA
# clusters this measured slower (EfficientNetV2-L alone 2.73 vs 2.66 ms); with 16-CTA
# clusters and the faster epilogue math it wins: EfficientNetV2-L batch 1 2.22 -> 2.16 ms,
# 4-model batch 32 11.77 -> 11.58 ms (61 launches fewer)
SE_FUSE_SCALE = os.environ.get("DFX_SE_FUSE", "1") == "1"


def round_up(x: int, a: int) -> int:
    return (x + a - 1) // a * a


def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit patterns, round-to-nearest-even (finite inputs)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


PRECISIONS = ("fp16", "bf16", "fp16x2", "bf16x2")
# Split precision (dfx.h DFX_F16X2 / DFX_BF16X2): every activation and GEMM / SE
# weight stored as two 16-bit planes v = hi + lo; GEMMs accumulate
# hi*hi + lo*hi + hi*lo.  The accurate mode: ~22 (fp16x2) / 16 (bf16x2)
# significant bits instead of 11 / 8 (SURVEY.md §7 hard part 2's escape hatch).
SPLIT_PRECISIONS = ("fp16x2", "bf16x2")


def base_precision(precision: str) -> str:
    """The 16-bit type of one plane: "fp16x2" -> "fp16"."""
    return precision[:4]


def planes_of(precision: str) -> int:
    return 2 if precision in SPLIT_PRECISIONS else 1


def pack_bits(a: np.ndarray, precision: str) -> np.ndarray:
    """Stored bits of a weight matrix [rows][k]: 16-bit, or for split precision
    [hi rows; lo rows] with hi = rn16(a), lo = rn16(a - hi)."""
    if precision not in SPLIT_PRECISIONS:
        return to_storage_bits(a, precision)
    b = base_precision(precision)
    a = np.asarray(a, np.float32)
    hi = to_storage_bits(a, b)
    lo = to_storage_bits(a - storage_bits_to_f32(hi, b), b)
    return np.ascontiguousarray(np.concatenate([hi, lo], axis=0))


def to_storage_bits(a: np.ndarray, precision: str) -> np.ndarray:
    """fp32 -> 16-bit storage bit patterns (fp16 saturates at +-65504 like the kernels)."""
    if precision == "bf16":
        return to_bf16_bits(a)
    if precision == "fp16":
        c = np.clip(np.asarray(a, np.float32), -65504, 65504)
        try:                       # torch's converter (F16C): ~15x numpy's on fp16 subnormals
            import torch           # (the lo plane of split weights), same IEEE round-to-nearest-even
            return torch.from_numpy(np.ascontiguousarray(c)).to(torch.float16).numpy().view(np.uint16)
        except ImportError:
            return c.astype(np.float16).view(np.uint16)
    raise ValueError(precision)


def storage_bits_to_f32(b: np.ndarray, precision: str) -> np.ndarray:
    if precision == "bf16":
        return bf16_bits_to_f32(b)
    return b.view(np.float16).astype(np.float32)


@dataclass
class Buffer:
    bid: int
    h: int
    w: int
    c: int                  # channels of the whole buffer
    pitch: int              # round_up(c, 8)
    name: str
    first: int = 10 ** 9    # launch index of first write
    last: int = -1          # launch index of last read
    is_input: bool = False
    planes: int = 1         # 2: split precision, hi and lo planes of a pixel side by side

    @property
    def phys_pitch(self) -> int:
        """Elements per pixel in memory (both planes for split precision)."""
        return self.pitch * self.planes

    def bytes_for(self, n: int) -> int:
        return n * self.h * self.w * self.phys_pitch * 2


@dataclass
class Value:
    """Physical placement of one IR value."""
    buf: int
    coff: int
    h: int
    w: int
    c: int
    flat: bool = False      # logical rank-1 over physical (h, w, c) in CHW order


@dataclass
class Epi:
    alpha: np.ndarray | None = None
    beta: np.ndarray | None = None
    act1: str | None = None
    binop: int = 0          # 0 none, 1 add, 2 scale
    other: str | None = None   # IR node id of the binop operand
    act2: str | None = None

    def affine_open(self) -> bool:
        return self.act1 is None and self.binop == 0 and self.act2 is None


@dataclass
class Launch:
    kind: str
    nodes: list[str]                    # IR nodes covered (anchor first)
    src: str                            # IR value read as the main operand
    dst: str                            # IR value written
    epi: Epi = field(default_factory=Epi)
    geom: dict = field(default_factory=dict)
    blobs: dict = field(default_factory=dict)     # role -> blob key
    index: int = -1
    pre: Epi | None = None              # GEMM A prologue transform (a folded EW producer)
    se: "Launch | None" = None          # DWSE: the absorbed SE launch (its blobs / geometry)
    pre_nodes: list = field(default_factory=list)


@dataclass
class MemberProgram:
    model_id: str
    input_dims: tuple
    output_dims: tuple
    launches: list[Launch]
    values: dict[str, Value]
    buffers: list[Buffer]
    blobs: dict[str, np.ndarray]        # key -> uint16 (bf16) or float32 array
    exit_value: str
    input_value: str = "<input>"
    gemm_flops_per_sample: int = 0
    precision: str = "fp16"
    input_im2col: tuple | None = None   # (kh, kw, sh, sw, ph, pw): input stored im2col'ed
    input_split: int = 0                # > 0: im2col'ed input as [hi | hi | lo] blocks of this width

    def weight_bytes(self) -> int:
        return sum(b.nbytes for b in self.blobs.values())


# ------------------------------------------------------------------------------------------

def _act_or_none(kind):
    return kind if kind in ACTIVATION_KINDS else None


class _Lowerer:
    def __init__(self, g, w):
        self.g, self.w = g, w
        self.shapes = infer_shapes(g)
        self.order = topo_order(g)
        self.pos = {nid: i for i, nid in enumerate(self.order)}
        self.users: dict[str, list[str]] = {nid: [] for nid in g.nodes}
        for nid in self.order:
            for s in g.nodes[nid].inputs:
                if nid not in self.users[s]:
                    self.users[s].append(nid)
        self.absorbed: dict[str, str] = {}      # node -> anchor
        self.launches: list[Launch] = []
        self.values: dict[str, Value] = {}
        self.buffers: list[Buffer] = []
        self.blobs: dict[str, np.ndarray] = {}
        self.acc_owner: dict[str, str] = {}
        self.pending_weights: list = []
        self.pending_se: list = []
        self.pending_vec: list = []             # (launch, node, fp32 weight roles)
        self.precision = "fp16"
        self.keep_f32 = False
        self.input_im2col = self._entry_im2col()
        self.input_split = 0
        self.debug_f32: dict[str, np.ndarray] = {}

    # -------------------------------------------------------------- helpers
    def _entry_im2col(self):
        """(kh, kw, sh, sw, ph, pw) when the entry conv should read an im2col'ed input
        written by the input kernel (dfx_in_params.kh > 0) and run as a 1x1 GEMM over
        kh*kw*C channels: stems with C < 16 input channels (C = 3 would otherwise pad
        every tap's channel block 3 -> 16, 5.3x the MMA work) and patchify convs
        (stride 16 does not fit a TMA element stride)."""
        node = self.g.nodes[self.g.entry]
        d = self.g.input_spec.dims
        if node.kind != "conv2d" or len(d) != 3 or int(node.attrs.get("groups", 1)) != 1:
            return None
        kh, kw, sh, sw, ph, pw = conv_geometry(node.attrs)
        if kh * kw == 1 or (d[0] >= 16 and max(sh, sw) <= 8):
            return None
        ow = (d[2] + 2 * pw - kw) // sw + 1
        window = d[0] * kh * ((min(ow, 256) - 1) * sw + kw) * 4     # dfx_bw.cu in_im2col_kernel smem
        if kh * kw * d[0] > 2048 or window > 219 * 1024:
            return None
        return (kh, kw, sh, sw, ph, pw)

    def dims(self, nid):
        return self.shapes[nid].dims

    def in_dims(self, nid):
        if nid == self.g.entry:
            return self.g.input_spec.dims
        return self.dims(self.g.nodes[nid].inputs[0])

    def src_of(self, nid, k=0):
        return "<input>" if nid == self.g.entry else self.g.nodes[nid].inputs[k]

    def warr(self, node, role):
        return np.asarray(self.w.array(node.weight_refs[role]), dtype=np.float32)

    def single_user(self, nid):
        u = self.users[nid]
        return u[0] if len(u) == 1 and nid != self.g.exit else None

    def bn_affine(self, node):
        eps = np.float32(node.attrs.get("epsilon", 1e-5))
        var = self.warr(node, "var")
        inv = (np.float32(1.0) / np.sqrt(var + eps)).astype(np.float32)
        s = self.warr(node, "gamma").astype(np.float64) * inv
        t = self.warr(node, "beta").astype(np.float64) - self.warr(node, "mean") * s
        return s, t

    # -------------------------------------------------------------- chains
    def materialized(self, nid) -> bool:
        """Is ``nid``'s value stored by some launch (not a folded middle of a chain)?"""
        if nid not in self.absorbed:
            return True
        return any(L.dst == nid for L in self.launches)

    def absorb(self, anchor_id: str, tail: str, epi: Epi, allow_affine: bool, allow_bin: bool):
        """Greedily fold single-consumer successors into the epilogue."""
        nodes = [anchor_id] if anchor_id != tail else [tail]
        while True:
            nxt = self.single_user(tail)
            if nxt is None:
                break
            node = self.g.nodes[nxt]
            k = node.kind
            if k == "batchnorm_inference" and allow_affine and epi.affine_open():
                s, t = self.bn_affine(node)
                a = np.ones_like(s) if epi.alpha is None else epi.alpha.astype(np.float64)
                b = np.zeros_like(s) if epi.beta is None else epi.beta.astype(np.float64)
                epi.alpha = (a * s).astype(np.float32)
                epi.beta = (b * s + t).astype(np.float32)
            elif _act_or_none(k) and epi.binop == 0 and epi.act1 is None:
                epi.act1 = k
            elif _act_or_none(k) and epi.binop != 0 and epi.act2 is None:
                epi.act2 = k
            elif k == "residual_add" and allow_bin and epi.binop == 0 and epi.act2 is None \
                    and len(node.inputs) == 2:
                other = node.inputs[1] if node.inputs[0] == tail else node.inputs[0]
                if other == tail or self.pos[other] >= self.pos[anchor_id] \
                        or not self.materialized(other):
                    break
                epi.binop, epi.other = 1, other
            elif k == "channel_scale" and allow_bin and epi.binop == 0 and epi.act2 is None \
                    and node.inputs[0] == tail:
                other = node.inputs[1]
                if self.pos[other] >= self.pos[anchor_id] or not self.materialized(other):
                    break
                epi.binop, epi.other = 2, other
            else:
                break
            self.absorbed[nxt] = anchor_id
            nodes.append(nxt)
            tail = nxt
        return nodes, tail

    def lower_node(self, nid):
        node = self.g.nodes[nid]
        k = node.kind
        if k in ("conv2d", "dense"):
            return self.lower_gemm_or_dw(nid)
        if k in ("maxpool2d", "avgpool2d"):
            kh, kw, sh, sw, ph, pw = pool_geometry(node.attrs)
            L = Launch(POOL, [nid], self.src_of(nid), nid,
                       geom=dict(kh=kh, kw=kw, sh=sh, sw=sw, ph=ph, pw=pw,
                                 is_max=int(k == "maxpool2d"),
                                 cip=int(node.attrs.get("count_include_pad", 1))))
            self.launches.append(L)
            return
        if k == "global_avg_pool":
            se = self.match_se(nid)
            if se is not None:
                self.launches.append(se)
                return
            self.launches.append(Launch(GAP, [nid], self.src_of(nid), nid))
            return
        if k in ("flatten", "concat"):
            return          # views; handled in placement
        if k == "layernorm":
            sel = self.single_user(nid)
            geom = dict(norm=1, eps=float(node.attrs.get("epsilon", 1e-5)))
            if sel is not None and self.g.nodes[sel].kind == "select_token" \
                    and int(self.g.nodes[sel].attrs.get("index", 0)) == 0:
                self.absorbed[sel] = nid            # normalise only the selected row
                L = Launch(LN, [nid, sel], self.src_of(nid), sel, geom=geom)
            else:
                L = Launch(LN, [nid], self.src_of(nid), nid, geom=geom)
            self.pending_vec.append((L, node, ("gamma", "beta")))
            self.launches.append(L)
            return
        if k == "select_token":
            if int(node.attrs.get("index", 0)) != 0:
                raise UnsupportedOnDevice(nid, "select_token index != 0")
            self.launches.append(Launch(LN, [nid], self.src_of(nid), nid, geom=dict(norm=0, eps=0.0)))
            return
        if k == "tokens":
            L = Launch(TOKENS, [nid], self.src_of(nid), nid)
            self.pending_vec.append((L, node, ("class_token", "pos_embedding")))
            self.launches.append(L)
            return
        if k == "attention":
            heads = int(node.attrs["heads"])
            c = self.dims(nid)[1]
            if c % heads or c // heads != 64:
                raise UnsupportedOnDevice(nid, f"attention head dim {c // max(heads, 1)} (64 only)")
            self.launches.append(Launch(ATTN, [nid], self.src_of(nid), nid,
                                        geom=dict(heads=heads, seq=self.dims(nid)[0], c=c)))
            return
        # elementwise anchors
        epi = Epi()
        src = self.src_of(nid)
        if k == "batchnorm_inference":
            s, t = self.bn_affine(node)
            epi.alpha, epi.beta = s.astype(np.float32), t.astype(np.float32)
        elif k in ACTIVATION_KINDS:
            epi.act1 = k
        elif k == "residual_add":
            ins = node.inputs
            if len(ins) > 2:
                self.lower_multi_add(nid)
                return
            src, epi.binop, epi.other = ins[0], 1, ins[1]
        elif k == "channel_scale":
            src, epi.binop, epi.other = node.inputs[0], 2, node.inputs[1]
        nodes, tail = self.absorb(nid, nid, epi, allow_affine=k in ("batchnorm_inference",)
                                  or k in ACTIVATION_KINDS, allow_bin=True)
        self.launches.append(Launch(EW, nodes, src, tail, epi=epi))

    def lower_multi_add(self, nid):
        """residual_add with k > 2 inputs: left fold (executor.py:153-155) as k-1 adds."""
        ins = self.g.nodes[nid].inputs
        tmp = f"{nid}#acc"
        self.acc_owner[tmp] = nid
        acc = ins[0]
        for i, other in enumerate(ins[1:]):
            dst = nid if i == len(ins) - 2 else tmp
            self.launches.append(Launch(EW, [nid], acc, dst, epi=Epi(binop=1, other=other)))
            acc = dst

    def lower_gemm_or_dw(self, nid):
        node = self.g.nodes[nid]
        idims = self.in_dims(nid)
        a = node.attrs
        epi = Epi()
        bias = self.warr(node, "bias") if "bias" in node.weight_refs else None
        if node.kind == "dense":
            units, fan_in = int(a["units"]), int(a["fan_in"])
            wt = self.warr(node, "weight")
            src = self.src_of(nid)
            geom = dict(cout=units, cin=fan_in, kh=1, kw=1, sh=1, sw=1, ph=0, pw=0,
                        dense=True, tokens=len(idims) == 2)
            wt4 = wt.reshape(units, fan_in, 1, 1)
            kind = GEMM
        else:
            kh, kw, sh, sw, ph, pw = conv_geometry(a)
            cout, groups = int(a["out_channels"]), int(a.get("groups", 1))
            cin = idims[0]
            wt4 = self.warr(node, "weight")
            src = self.src_of(nid)
            if nid == self.g.entry and self.input_im2col is not None:
                # 1x1 conv over the im2col'ed input, K order (r, s, c)
                wt4 = np.ascontiguousarray(wt4.transpose(0, 2, 3, 1)).reshape(cout, kh * kw * cin, 1, 1)
                cin, kh, kw, sh, sw, ph, pw = kh * kw * cin, 1, 1, 1, 1, 0, 0
                kb = self.input_split
                if kb:                     # K = [w_hi | w_lo | w_hi] (see STEM_SPLIT)
                    w2 = wt4.reshape(cout, cin).astype(np.float32)
                    hi = storage_bits_to_f32(to_storage_bits(w2, self.precision), self.precision)
                    lo = storage_bits_to_f32(to_storage_bits(w2 - hi, self.precision), self.precision)
                    t3 = np.zeros((cout, 3 * kb), np.float32)
                    t3[:, :cin], t3[:, kb:kb + cin], t3[:, 2 * kb:2 * kb + cin] = hi, lo, hi
                    wt4, cin = t3.reshape(cout, 3 * kb, 1, 1), 3 * kb
            elif max(sh, sw) > 8:
                raise UnsupportedOnDevice(nid, f"conv stride {sh}x{sw} > 8 (TMA element stride)")
            geom = dict(cout=cout, cin=cin, kh=kh, kw=kw, sh=sh, sw=sw, ph=ph, pw=pw,
                        dense=False)
            if groups == 1:
                kind = GEMM
            elif groups == cin == cout:
                kind = DWCONV
            else:
                raise UnsupportedOnDevice(nid, f"grouped conv with groups={groups} "
                                               f"(only 1 or depthwise)")
        epi.beta = None if bias is None else bias.astype(np.float32)
        nodes, tail = self.absorb(nid, nid, epi, allow_affine=True, allow_bin=(kind == GEMM))
        L = Launch(kind, nodes, src, tail, epi=epi, geom=geom)
        key = f"{nid}.w"
        L.blobs["weight"] = key
        self.pending_weights.append((L, wt4))
        self.launches.append(L)

    # -------------------------------------------------------------- placement
    def new_buffer(self, h, w, c, name):
        b = Buffer(len(self.buffers), h, w, c, round_up(c, 8), name, planes=planes_of(self.precision))
        self.buffers.append(b)
        return b.bid

    def _is_flat_source(self, s):
        node = self.g.nodes[s]
        if node.kind != "flatten":
            return False
        d = self.in_dims(s)
        return len(d) == 3 and d[1] * d[2] > 1

    def resolve(self, name):
        """Placement of a value, creating flatten views on demand."""
        if name in self.values:
            return self.values[name]
        node = self.g.nodes.get(name)
        if node is not None and node.kind == "flatten":
            if len(self.in_dims(name)) == 2:
                raise UnsupportedOnDevice(name, "flatten of a token tensor")
            src = self.resolve(self.src_of(name))
            v = Value(src.buf, src.coff, src.h, src.w, src.c, flat=src.flat or src.h * src.w > 1)
            self.values[name] = v
            return v
        raise UnsupportedOnDevice(name, "value has no placement")

    def place(self):
        g = self.g
        ind = g.input_spec.dims
        h, w = (ind[1], ind[2]) if len(ind) == 3 else (1, 1)
        c = ind[0]
        if self.input_im2col is not None:
            kh, kw, sh, sw, ph, pw = self.input_im2col
            h, w, c = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1, c * kh * kw
            if self.input_split:
                c = 3 * self.input_split
        ib = self.new_buffer(h, w, c, "<input>")
        self.buffers[ib].is_input = True
        self.values["<input>"] = Value(ib, 0, h, w, c)

        produced = {L.dst for L in self.launches}
        # concat groups, outermost first (reverse topo order): parts written in place
        self.copies = []
        for cid in reversed([n for n in self.order if g.nodes[n].kind == "concat"]):
            d = self.dims(cid)
            if any(self._is_flat_source(s) for s in g.nodes[cid].inputs):
                raise UnsupportedOnDevice(cid, "concat of flattened spatial tensors")
            h, w = (d[1], d[2]) if len(d) == 3 else (1, 1)
            if cid not in self.values:
                self.values[cid] = Value(self.new_buffer(h, w, d[0], cid), 0, h, w, d[0])
            base = self.values[cid]
            off = 0
            for s in g.nodes[cid].inputs:
                cs = self.dims(s)[0]
                at = base.coff + off
                if at % 8 == 0 and s not in self.values and \
                        (s in produced or g.nodes[s].kind == "concat"):
                    self.values[s] = Value(base.buf, at, h, w, cs)
                else:
                    self.copies.append((s, cid, at))
                off += cs

        # launch outputs, in launch order (sources resolve lazily through flatten views)
        for L in self.launches:
            if L.dst in self.values:
                continue
            src = self.resolve(L.src)
            if L.dst.endswith("#acc"):
                d = self.dims(self.acc_owner[L.dst])
            else:
                d = self.dims(L.dst)
            if L.kind == EW and src.flat:
                self.values[L.dst] = Value(self.new_buffer(src.h, src.w, src.c, L.dst), 0,
                                           src.h, src.w, src.c, flat=True)
            elif len(d) == 3:
                self.values[L.dst] = Value(self.new_buffer(d[1], d[2], d[0], L.dst), 0,
                                           d[1], d[2], d[0])
            elif len(d) == 2:                    # token rows (L, C) -> view h = 1, w = L
                self.values[L.dst] = Value(self.new_buffer(1, d[0], d[1], L.dst), 0, 1, d[0], d[1])
            else:
                self.values[L.dst] = Value(self.new_buffer(1, 1, d[0], L.dst), 0, 1, 1, d[0])
        for nid in self.order:              # remaining views (e.g. a flatten exit)
            if nid not in self.values and g.nodes[nid].kind == "flatten":
                self.resolve(nid)

    # -------------------------------------------------------------- build
    def run(self) -> MemberProgram:
        if len(self.g.input_spec.dims) == 2 or len(self.dims(self.g.exit)) == 2:
            raise UnsupportedOnDevice(self.g.exit, "token tensor as the model input or output")
        for nid in self.order:
            if nid in self.absorbed:
                continue
            self.lower_node(nid)
        if FUSE_DWSE and self.precision not in SPLIT_PRECISIONS:
            self.fuse_dw_se()
        if FOLD_PRE and self.precision not in SPLIT_PRECISIONS:
            self.fold_pre_transforms()
        self.place()
        for s, cid, off in self.copies:
            self.launches.append(Launch(COPY, [cid], s, f"{cid}@{off}",
                                        geom=dict(coff=off, concat=cid)))
        self.launches.sort(key=lambda L: self.pos[L.geom["concat"]] if L.kind == COPY
                           else self.pos[L.nodes[0]])          # stable: keeps emission order
        for i, L in enumerate(self.launches):
            L.index = i + 1            # 0 is the input conversion
        self.check_and_finish()
        self.pack_weights()
        for L in self.launches:
            if L.kind == DWSE:
                L.blobs.update(L.se.blobs)
        return MemberProgram(self.g.model_id, tuple(self.g.input_spec.dims),
                             tuple(self.g.output_spec.dims), self.launches, self.values,
                             self.buffers, self.blobs, self.g.exit)

    def fuse_dw_se(self):
        """depthwise conv (+ BN/act) -> SE gate -> channel_scale(dw, gate), where the
        depthwise output feeds only the SE and the scale and the gate only the scale:
        ONE dwse launch (dfx_fused.cu dwse_kernel) instead of three."""
        g = self.g
        uses: dict[str, int] = {}
        for L in self.launches:
            uses[L.src] = uses.get(L.src, 0) + 1
            if L.epi.other is not None:
                uses[L.epi.other] = uses.get(L.epi.other, 0) + 1
        for nid in self.order:
            if g.nodes[nid].kind in ("concat", "flatten"):
                for s_ in g.nodes[nid].inputs:
                    uses[s_] = uses.get(s_, 0) + 2
        uses[g.exit] = uses.get(g.exit, 0) + 2
        by_src: dict[str, list] = {}
        for L in self.launches:
            by_src.setdefault(L.src, []).append(L)
        drop = set()
        for D in self.launches:
            if D.kind != DWCONV or D.epi.binop or D.epi.act2 is not None or uses.get(D.dst, 0) != 2:
                continue
            geo = D.geom
            if geo["kh"] > 7 or geo["kw"] > 7 or geo["cout"] % 8 or geo["cout"] > SE_MAX_C:
                continue
            cons = by_src.get(D.dst, [])
            S = next((L for L in cons if L.kind == SE and not L.geom.get("apply")), None)
            E = next((L for L in cons if L.kind == EW and L.epi.binop == 2), None)
            if S is None or E is None or E.epi.other != S.dst or uses.get(S.dst, 0) != 1:
                continue
            e = E.epi
            if e.alpha is not None or e.beta is not None or e.act1 or e.act2:
                continue
            oh, ow = self.dims(D.dst)[1:]
            if dwse_smem(geo["cout"], S.geom["cr"], oh * ow) > SE_SMEM_BUDGET:
                continue
            D.kind, D.se, D.dst = DWSE, S, E.dst
            D.nodes = D.nodes + S.nodes + E.nodes
            D.geom = dict(geo, cr=S.geom["cr"], act1=S.geom["act1"], act2=S.geom["act2"], c=geo["cout"])
            drop.update((id(S), id(E)))
        self.launches = [L for L in self.launches if id(L) not in drop]

    def fold_pre_transforms(self):
        """Fold an elementwise producer into the A operand of the 1x1 conv that is its
        only consumer: DenseNet's pre-activation BN + ReLU on the concat buffer (mode
        1) and the squeeze-excitation channel scale before a projection conv (mode
        2).  The GEMM rewrites each A tile in shared memory before the MMA
        (dfx_epi.cuh pre_transform_stage): one launch and one full activation
        write + read fewer.  1x1 / unpadded only: a transform of padding zeros
        would not stay zero."""
        g = self.g
        uses: dict[str, int] = {}
        for L in self.launches:
            uses[L.src] = uses.get(L.src, 0) + 1
            if L.epi.other is not None:
                uses[L.epi.other] = uses.get(L.epi.other, 0) + 1
        for nid in self.order:
            if g.nodes[nid].kind in ("concat", "flatten"):
                for s in g.nodes[nid].inputs:
                    uses[s] = uses.get(s, 0) + 2          # views / copies: never fold
        uses[g.exit] = uses.get(g.exit, 0) + 2
        producer = {L.dst: L for L in self.launches}
        drop = set()
        for L in self.launches:
            geo = L.geom
            if L.kind != GEMM or geo.get("dense") or geo.get("tokens") or geo["kh"] != 1 or \
                    geo["kw"] != 1 or geo["ph"] or geo["pw"]:
                continue
            E = producer.get(L.src)
            if E is None or E.kind != EW or uses.get(E.dst, 0) != 1 or E.dst.endswith("#acc"):
                continue
            if E.src in g.nodes and g.nodes[E.src].kind == "flatten":
                continue
            e = E.epi
            if e.binop == 0 and e.act2 is None and (e.alpha is not None or e.beta is not None or e.act1):
                pre = Epi(alpha=e.alpha, beta=e.beta, act1=e.act1)
            elif e.binop == 2 and e.alpha is None and e.beta is None and e.act1 is None and e.act2 is None:
                pre = Epi(binop=2, other=e.other)
            else:
                continue
            L.pre, L.pre_nodes, L.src = pre, list(E.nodes), E.src
            geo["pre"] = 1
            drop.add(id(E))
        self.launches = [L for L in self.launches if id(L) not in drop]

    def value_of(self, name):
        return self.resolve(name)

    def check_and_finish(self):
        n_launch = len(self.launches) + 2      # + input conversion (0) + output (last)
        inb = self.values["<input>"].buf
        self.buffers[inb].first = 0

        def touch_write(v, i):
            b = self.buffers[v.buf]
            b.first = min(b.first, i)
            b.last = max(b.last, i)

        def touch_read(v, i):
            b = self.buffers[v.buf]
            b.last = max(b.last, i)

        for L in self.launches:
            i = L.index
            touch_read(self.value_of(L.src), i)
            if L.epi.other is not None:
                touch_read(self.value_of(L.epi.other), i)
            if L.pre is not None and L.pre.other is not None:
                touch_read(self.value_of(L.pre.other), i)
            if L.kind == COPY:
                touch_write(self.value_of(L.geom["concat"]), i)
            else:
                touch_write(self.value_of(L.dst), i)
            # semantic checks for flattened operands
            sv = self.value_of(L.src)
            if sv.flat and L.kind == EW and L.epi.alpha is not None:
                raise UnsupportedOnDevice(L.nodes[0], "per-channel affine on a flattened tensor")
            if sv.flat and L.kind in (POOL, GAP, DWCONV):
                raise UnsupportedOnDevice(L.nodes[0], "spatial op on a flattened tensor")
            if L.kind == GEMM and not L.geom["dense"] and sv.flat:
                raise UnsupportedOnDevice(L.nodes[0], "conv on a flattened tensor")
        exitv = self.value_of(self.g.exit)
        self.buffers[exitv.buf].last = n_launch
        for b in self.buffers:
            if b.first > b.last:        # written but never read (dead-end) -> live at write
                b.last = b.first

    # -------------------------------------------------------------- weights
    def match_se(self, gap_id: str):
        """global_avg_pool -> dense -> [act] -> dense -> [act] (a squeeze-excitation
        gate) with single consumers along the chain: ONE cluster launch."""
        chain = [gap_id]
        cur = gap_id
        fcs, acts = [], [None, None]
        for which in (0, 1):
            nxt = self.single_user(cur)
            if nxt is None or self.g.nodes[nxt].kind != "dense":
                return None
            fcs.append(nxt)
            chain.append(nxt)
            cur = nxt
            a = self.single_user(cur)
            if a is not None and self.g.nodes[a].kind in ACTIVATION_KINDS:
                acts[which] = self.g.nodes[a].kind
                chain.append(a)
                cur = a
        c = self.dims(gap_id)[0]
        cr = int(self.g.nodes[fcs[0]].attrs["units"])
        if int(self.g.nodes[fcs[1]].attrs["units"]) != c or c > SE_MAX_C or cr > SE_MAX_CR:
            return None
        # the gate's only consumer scales the pooled tensor itself: fuse it (apply = 1)
        apply = 0
        sc = self.single_user(cur)
        x = self.src_of(gap_id)
        if SE_FUSE_SCALE and sc is not None and self.g.nodes[sc].kind == "channel_scale" \
                and self.g.nodes[sc].inputs == (x, cur):
            chain.append(sc)
            cur, apply = sc, 1
        for n in chain[1:]:
            self.absorbed[n] = gap_id
        L = Launch(SE, chain, x, cur,
                   geom=dict(c=c, cr=cr, act1=acts[0], act2=acts[1], fc1=fcs[0], fc2=fcs[1],
                             apply=apply))
        self.pending_se.append(L)
        return L

    def pack_weights(self):
        for L, node, roles in self.pending_vec:
            for role in roles:
                v = self.warr(node, role).reshape(-1)
                arr = np.zeros(round_up(len(v), 8), dtype=np.float32)
                arr[:len(v)] = v
                key = f"{node.node_id}.{role}"
                self.blobs[key] = arr
                L.blobs[role] = key
        for L in self.pending_se:
            for role, fc in (("1", L.geom["fc1"]), ("2", L.geom["fc2"])):
                node = self.g.nodes[fc]
                key = f"{fc}.w"
                wt = self.warr(node, "weight")            # (out, in)
                # fc1 is stored transposed ([C][Cr]) so each cluster CTA's channel
                # slice of both FCs is one contiguous block (dfx_fused.cu se_kernel)
                self.blobs[key] = pack_bits(np.ascontiguousarray(wt.T) if role == "1" else wt,
                                            self.precision)
                L.blobs["w" + role] = key
                if "bias" in node.weight_refs:
                    b = self.warr(node, "bias")
                    arr = np.zeros(round_up(len(b), 8), dtype=np.float32)
                    arr[:len(b)] = b
                    self.blobs[f"{fc}.b"] = arr
                    L.blobs["b" + role] = f"{fc}.b"
        for L, wt4 in self.pending_weights:
            geo = L.geom
            if L.kind in (DWCONV, DWSE):
                c = geo["cout"]
                taps = np.ascontiguousarray(wt4[:, 0].transpose(1, 2, 0).reshape(-1, c),
                                            dtype=np.float32)       # [kh*kw][c]
                self.blobs[L.blobs["weight"]] = taps
            else:
                sv = self.resolve(L.src)
                if geo["dense"] and sv.flat:
                    # dense over a flattened (C,H,W): a conv whose kernel is the whole image
                    cin, h, w = sv.c, sv.h, sv.w
                    wt4 = wt4.reshape(geo["cout"], cin, h, w)
                    geo.update(cin=cin, kh=h, kw=w)
                cin = geo["cin"]
                cb = choose_cb(cin)
                cblocks = -(-cin // cb)
                cout = geo["cout"]
                t = np.zeros((cout, geo["kh"], geo["kw"], cblocks * cb), dtype=np.float32)
                t[..., :cin] = wt4.transpose(0, 2, 3, 1)
                packed = pack_bits(t.reshape(cout, -1), self.precision)
                geo.update(cb=cb, cblocks=cblocks, ksteps=geo["kh"] * geo["kw"] * cblocks,
                           k=packed.shape[1])
                self.blobs[L.blobs["weight"]] = packed
                if self.keep_f32:
                    self.debug_f32[L.blobs["weight"]] = t.reshape(cout, -1)
                if L.pre is not None and L.pre.binop == 0:
                    # the transform reads whole 8-channel chunks up to cblocks * cb;
                    # an identity scale where only a shift / an activation is folded
                    for role, v in (("pre_alpha", L.pre.alpha if L.pre.alpha is not None
                                     else np.ones(cin, np.float32)), ("pre_beta", L.pre.beta)):
                        if v is None:
                            continue
                        arr = np.zeros(cblocks * cb, dtype=np.float32)
                        arr[:len(v)] = v
                        key = f"{L.nodes[0]}.{role}"
                        self.blobs[key] = arr
                        L.blobs[role] = key
            for role in ("alpha", "beta"):
                v = getattr(L.epi, role)
                if v is not None:
                    key = f"{L.nodes[0]}.{role}"
                    arr = np.zeros(round_up(len(v), 8), dtype=np.float32)
                    arr[:len(v)] = v
                    self.blobs[key] = arr
                    L.blobs[role] = key
        for L in self.launches:
            if L.kind == EW:
                for role in ("alpha", "beta"):
                    v = getattr(L.epi, role)
                    if v is not None:
                        key = f"{L.nodes[0]}.{role}"
                        arr = np.zeros(round_up(len(v), 8), dtype=np.float32)
                        arr[:len(v)] = v
                        self.blobs[key] = arr
                        L.blobs[role] = key


CB_WASTE = float(os.environ.get("DFX_CB_WASTE", "0.125"))     # A/B knob
# Split-precision stem (the precision escape of SURVEY.md §7 hard part 2): the
# im2col'ed entry conv runs as ONE GEMM over K = [x_hi | x_hi | x_lo] against
# [w_hi | w_lo | w_hi], where v = v_hi + v_lo with both parts 16-bit: the products
# x_hi w_hi + x_hi w_lo + x_lo w_hi carry ~16 mantissa bits of the fp32 input and
# weights.  Measured with the CPU emulator on the calibrated DenseNet161 in bf16:
# the stem's weight rounding alone is 3.1 % of the logits' 4.3 % (weights) and the
# input rounding another ~1 %; the stem is 0.1-1.5 % of a model's FLOPs.
# "bf16" (default): bf16 DAGs only; "all": fp16 too; "off".
STEM_SPLIT = os.environ.get("DFX_STEM_SPLIT", "bf16")


def choose_cb(cin: int) -> int:
    """Channel block for the K loop: the widest of 64/32/16 wasting <= CB_WASTE."""
    for cb in (64, 32):
        if -(-cin // cb) * cb <= cin * (1 + CB_WASTE):
            return cb
    return 16


def lower_member(g, w, keep_f32: bool = False, precision: str = "fp16") -> MemberProgram:
    """``precision``: 16-bit storage/operand type ("fp16" default, or "bf16").
    ``keep_f32`` also keeps the unrounded packed GEMM weights (tests only)."""
    if precision not in PRECISIONS:
        raise ValueError(precision)
    low = _Lowerer(g, w)
    low.keep_f32 = keep_f32
    low.precision = precision
    if low.input_im2col is not None and (STEM_SPLIT == "all" or STEM_SPLIT == precision) and \
            precision not in SPLIT_PRECISIONS:
        kh, kw = low.input_im2col[:2]
        low.input_split = round_up(kh * kw * g.input_spec.dims[0], 8)
    prog = low.run()
    if precision in SPLIT_PRECISIONS:
        for L in prog.launches:
            if L.kind in (LN, TOKENS, ATTN):
                raise UnsupportedOnDevice(L.nodes[0], f"{L.kind} has no split-precision kernel ({precision})")
    prog.debug_f32 = low.debug_f32
    prog.precision = precision
    prog.input_im2col = low.input_im2col
    prog.input_split = low.input_split
    from .graph_ir import gemm_flops
    prog.gemm_flops_per_sample = gemm_flops(g)
    return prog


# ------------------------------------------------------------------------------------------
# per-batch GEMM tiling

def choose_m_tile(n: int, p: int, q: int, sh: int, sw: int):
    """(tn, tp, tq) covering <= 128 output pixels with the best row utilisation."""
    best = None
    if p * q <= 128:
        tq, tp = q, p
        tn = max(1, min(n, 128 // (p * q), 256))
        cands = [(tn, tp, tq)]
    else:
        cands = []
        for tq in range(1, min(q, 128) + 1):
            if tq * sw > 256:
                break
            tp = min(p, 128 // tq)
            if tp < 1 or tp * sh > 256:
                continue
            cands.append((1, tp, tq))
    for tn, tp, tq in cands:
        tiles = math.ceil(n / tn) * math.ceil(p / tp) * math.ceil(q / tq)
        util = (n * p * q) / (tiles * 128)
        score = (round(util, 4), tq)
        if best is None or score > best[0]:
            best = (score, (tn, tp, tq))
    return best[1]


def choose_bn(cout: int) -> tuple[int, int]:
    nt = -(-cout // 256)
    bn = round_up(-(-cout // nt), 16)
    return bn, -(-cout // bn)


GEMM_M2 = os.environ.get("DFX_GEMM_M2", "1") != "0"     # A/B switch for 256-row CTAs
BN_FLOOR_MANY_M = int(os.environ.get("DFX_BN_FLOOR_MANY_M", "64"))   # A/B knob
BN_FLOOR_SUBWAVE_X2 = int(os.environ.get("DFX_BN_FLOOR_SUBWAVE_X2", "128"))   # A/B knob
SPLIT_MIN_STAGES = int(os.environ.get("DFX_SPLIT_MIN_STAGES", "4"))   # K stages per split, at least
# split precision: a stage costs 2-3x the MMAs and twice the operand bytes, so fewer,
# longer splits (measured at batch 1: 4-model fp16x2 3.34 ms at 4, 3.26 at 6, 3.39 at 8)
SPLIT_MIN_STAGES_X2 = int(os.environ.get("DFX_SPLIT_MIN_STAGES_X2", "6"))
# split-K reduction: "kernel" (default) = fp32 workspace + a splitk_kernel launch;
# "cluster" = the splits of a tile form a thread-block cluster and reduce over DSMEM
# inside the GEMM (dfx_gemm.cu, <= 8 splits; removes 245 of 928 launches at batch 1
# but measured no faster: 2.651 vs 2.635 ms fused, 4.539 vs 4.617 ms sequential --
# the splitk launch overlaps the GEMM tail under PDL, cluster co-scheduling does not);
# "fixup" = last-arriving CTA reduces (A/B, 2.28 -> 3.11 ms); "auto" (default) = cluster
# at batch <= 2 in DAGs of <= 4 members (4-model batch 1 2.27 -> 2.23 ms; with 8
# concurrent members the clusters wait for free GPC slices: 2.71 -> 3.12 ms), kernel else
SPLITK_MODE = os.environ.get("DFX_SPLITK", "auto")
# fuse depthwise conv -> SE -> channel scale into one dwse launch (DFX_FUSE_DWSE=1: on, A/B).
# Off by default: one 16-CTA cluster per image starves the depthwise phase of SMs
# (EfficientNetV2-L alone, batch 1: 2.85 vs 2.29 ms; batch 32: 7.54 vs 6.95 ms)
FUSE_DWSE = os.environ.get("DFX_FUSE_DWSE", "0") == "1"
SE_SMEM_BUDGET = 190 * 1024          # dfx_common.cuh kSeSmemBudget


def dwse_smem(c: int, cr: int, hwo: int) -> int:
    """dwse_kernel dynamic smem with staged FC slices (dfx_common.cuh dwse_smem_bytes)."""
    cs = -(-c // 128) * 8
    return 2 * round_up(cs * cr * 2, 16) + round_up(hwo * cs * 2, 16)


# fold elementwise producers into the A operand of 1x1 convs (DFX_FOLD_PRE=1: on, A/B).
# Off by default: the in-smem rewrite serialises each pipeline stage behind 4-6
# transform warps and measured slower than the separate bandwidth-bound pass
# (4-model batch 1 2.72 vs 2.52 ms, batch 32 17.1 vs 12.5 ms, 150 launches fewer)
FOLD_PRE = os.environ.get("DFX_FOLD_PRE", "0") == "1"
SPLITK_CLUSTER_MAX = int(os.environ.get("DFX_SPLITK_CLUSTER_MAX", "16"))   # > 8: non-portable cluster sizes


def gemm_tiling(geom: dict, n: int, p: int, q: int, sm_count: int = 148, cluster_ok: bool = False,
                max_splits: int = 0, planes: int = 1) -> dict:
    tn, tp, tq = choose_m_tile(n, p, q, geom["sh"], geom["sw"])
    mt = (math.ceil(n / tn), math.ceil(p / tp), math.ceil(q / tq))
    bn, nt = choose_bn(geom["cout"])
    m_tiles = mt[0] * mt[1] * mt[2]
    # small-M layers: narrower N tiles first (more CTAs, no extra kernel), split-K second
    # (with many M tiles -- batched layers -- N stays >= BN_FLOOR_MANY_M: an N = 64 MMA
    # costs what an N = 128 one does, so split-K keeps the tensor pipe denser)
    bn_floor = BN_FLOOR_MANY_M if m_tiles >= 8 else 64
    if planes > 1 and n <= 2 and 8 <= m_tiles < sm_count:
        # split precision at batch 1-2, sub-wave M (56x56 / 28x28 maps): wide N tiles,
        # since an N = 2bn MMA costs what an N = bn one does up to 128 (4-model batch 1
        # fp16x2 2.960 -> 2.947 ms; at batch 32 the same rule cost 17.19 -> 17.53 ms)
        bn_floor = max(bn_floor, BN_FLOOR_SUBWAVE_X2)
    while m_tiles * nt < sm_count and bn > bn_floor:
        bn = max(bn_floor, round_up(bn // 2, 16))
        nt = -(-geom["cout"] // bn)
    kpack = 64 // geom["cb"]
    stages = math.ceil(geom["ksteps"] / kpack)
    base = m_tiles * nt
    splits = 1
    min_st = SPLIT_MIN_STAGES_X2 if planes > 1 else SPLIT_MIN_STAGES
    if base < sm_count and stages >= 2 * min_st:
        splits = min(math.ceil(sm_count / base), stages // min_st)
    if max_splits:
        splits = min(splits, max_splits)
    sps = math.ceil(stages / max(splits, 1))
    splits = math.ceil(stages / sps)
    # m2: 256-row CTAs (two M tiles sharing each weight stage) once the grid still
    # fills the GPU -- halves B bytes per MAC for the fill-rate-bound large layers
    # (a 256-row CTA takes ~1.6x a 128-row one: only when the wave count drops enough)
    waves1 = math.ceil(m_tiles * nt / sm_count)
    waves2 = math.ceil(math.ceil(m_tiles / 2) * nt / sm_count)
    # (short-K layers go to the persistent kernel instead, whose overlapped epilogue
    # matters more there than the halved weight traffic: measured on 3x3 64->256 at
    # batch 32, 115 us m2 vs 80 us persistent; VGG's K=4608 layers keep m2)
    m2 = int(GEMM_M2 and planes == 1 and splits == 1 and bn >= 128 and m_tiles >= 2 and stages >= 24
             and not geom.get("pre")
             and math.ceil(m_tiles / 2) * nt >= sm_count and waves2 * 1.6 < waves1)
    tiles = (math.ceil(m_tiles / 2) if m2 else m_tiles) * nt * splits
    # cluster split-K when the splits fit one portable cluster; wider splits keep the
    # workspace + splitk_kernel reduction
    csplit = int((SPLITK_MODE == "cluster" or (SPLITK_MODE == "auto" and n <= 2 and cluster_ok))
                 and 1 < splits <= SPLITK_CLUSTER_MAX)
    return dict(tn=tn, tp=tp, tq=tq, mt_n=mt[0], mt_p=mt[1], mt_q=mt[2], bn=bn, nt=nt, csplit=csplit,
                kpack=kpack, stages=stages, splits=splits, sps=sps, m2=m2,
                tiles=tiles)
