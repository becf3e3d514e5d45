"""Activation planner: liveness intervals -> offsets in one shared arena.

Two artefacts come out of here.

* The **reference plan** (``member_plan``): the per-node intervals of the
  reference liveness rule (/root/reference/pkg/src/dagfuse/graph_ir.py:486-512),
  with fp32 single-sample byte sizes.  Its peak equals
  ``peak_activation_bytes`` bit-exactly; offsets are assigned by a
  deterministic first-fit so that the peak is realised as a real arena.
  ``fused_arena`` stacks member plans in member order into disjoint
  segments — the Σ that the reference's fused memory estimate charges
  (/root/reference/pkg/src/dagfuse/costmodel.py:264-266) — or, in the
  sequential-reuse variant, overlays them (max).

* The **device plan** (built by ``lower.py`` with ``first_fit``): the same
  rule over the buffers the kernels actually materialise (bf16, NHWC,
  batched, after epilogue fusion and zero-copy concat), which is smaller.
"""

from __future__ import annotations

from dataclasses import dataclass

from .graph_ir import LiveInterval, infer_shapes, liveness_intervals, peak_from_intervals, topo_order


@dataclass(frozen=True)
class Placement:
    name: str
    size: int
    first: int
    last: int
    offset: int


@dataclass(frozen=True)
class MemberPlan:
    model_id: str
    order: tuple[str, ...]
    placements: tuple[Placement, ...]
    peak: int            # max live bytes (== peak_activation_bytes for the reference plan)
    arena_bytes: int     # extent of the first-fit assignment (>= peak)

    def offset_of(self, name: str) -> int:
        for p in self.placements:
            if p.name == name:
                return p.offset
        raise KeyError(name)


def _align(x: int, a: int) -> int:
    return (x + a - 1) // a * a


def first_fit(intervals: list[LiveInterval], align: int = 1) -> list[Placement]:
    """Deterministic first-fit: intervals in (first, name) order; each takes the
    lowest aligned offset that does not overlap (in bytes) any already-placed
    interval whose [first, last] range intersects its own."""
    placed: list[Placement] = []
    for iv in sorted(intervals, key=lambda v: (v.first, v.name)):
        busy = sorted((p.offset, p.offset + p.size) for p in placed
                      if p.first <= iv.last and iv.first <= p.last and p.size > 0)
        at = 0
        for lo, hi in busy:
            if at + iv.size <= lo:
                break
            at = max(at, _align(hi, align))
        placed.append(Placement(iv.name, iv.size, iv.first, iv.last, at))
    return placed


def check_disjoint(placements) -> None:
    """Raise if two time-overlapping placements overlap in bytes."""
    ps = list(placements)
    for i, a in enumerate(ps):
        for b in ps[i + 1:]:
            if a.first <= b.last and b.first <= a.last and a.size and b.size:
                if a.offset < b.offset + b.size and b.offset < a.offset + a.size:
                    raise AssertionError(f"{a.name} and {b.name} overlap")


def plan_from_intervals(model_id: str, order, intervals, n_positions: int,
                        align: int = 1) -> MemberPlan:
    places = first_fit(intervals, align)
    extent = max((p.offset + p.size for p in places), default=0)
    return MemberPlan(model_id, tuple(order), tuple(places),
                      peak_from_intervals(intervals, n_positions), extent)


def member_plan(g, align: int = 1) -> MemberPlan:
    """Reference plan of one model (fp32, single sample, reference topo order)."""
    shapes = infer_shapes(g)
    order = topo_order(g)
    ivs = liveness_intervals(g, shapes, order)
    return plan_from_intervals(g.model_id, order, ivs, len(order), align)


@dataclass(frozen=True)
class FusedArena:
    mode: str                          # "sum" (disjoint segments) or "max" (overlay)
    segments: tuple[tuple[str, int, int], ...]   # (model_id, offset, bytes)
    total_bytes: int
    plans: tuple[MemberPlan, ...]


def fused_arena(plans: list[MemberPlan], mode: str = "sum", align: int = 256) -> FusedArena:
    """Member arenas in member order: disjoint (Σ) or overlaid (max)."""
    if mode not in ("sum", "max"):
        raise ValueError(mode)
    segs, at = [], 0
    for p in plans:
        if mode == "sum":
            segs.append((p.model_id, at, p.arena_bytes))
            at = _align(at + p.arena_bytes, align)
        else:
            segs.append((p.model_id, 0, p.arena_bytes))
            at = max(at, _align(p.arena_bytes, align))
    return FusedArena(mode, tuple(segs), at, tuple(plans))
