"""Memory accounting of the fused DAG (the subset of the reference cost model on
the hot path) plus the measured replacements.

``profile_graph`` / ``estimate_memory`` reproduce the reference arithmetic
exactly (/root/reference/pkg/src/dagfuse/costmodel.py:252-274, 358-373) so
``FusedDag.total_mem_estimate_mib`` is identical to the reference's.  The
calibration/replay machinery of the reference (Table IV, scenario replays)
is out of scope: on B200 the swap-in time and peak HBM are *measured*
(``device.WeightArena.upload``; cudaMemGetInfo samples in the bench and the
manager), not simulated.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Sequence

from .graph_ir import infer_shapes, mib_ceil, node_flops, node_input_dims, peak_activation_bytes, topo_order

MIB = 1 << 20
UNFUSED = "unfused"
FUSED = "fused"
MODES = (UNFUSED, FUSED)

# per-kind ms per MFLOP of the reference's analytic latency (costmodel.py:83-93)
_DEFAULT_OP_MS_PER_MFLOP = {
    "dense": 0.05, "conv2d": 0.05, "relu": 0.01, "maxpool2d": 0.02, "batchnorm_inference": 0.02,
    "residual_add": 0.01, "global_avg_pool": 0.01, "flatten": 0.001, "concat": 0.005,
}


@dataclass(frozen=True)
class CostTable:
    """Memory constants of the reference's default table (costmodel.py:116-121)."""
    context_base_mib: float = 500.0
    per_model_overhead_mib: float = 34.0
    dedup_saving_mib_per_extra_model: float = 34.0
    op_latency_ms_per_mflop: dict = field(default_factory=lambda: dict(_DEFAULT_OP_MS_PER_MFLOP))

    def op_latency_ms(self, kind: str, flops: int) -> float:
        return self.op_latency_ms_per_mflop.get(kind, 0.01) * (flops / 1e6)


DEFAULT_COST_TABLE = CostTable()


@dataclass(frozen=True)
class MemoryEstimate:
    context_mib: float
    weights_mib: float
    activations_mib: float
    overhead_mib: float

    @property
    def peak_mib(self) -> float:
        return self.context_mib + self.weights_mib + self.activations_mib + self.overhead_mib


@dataclass(frozen=True)
class GraphProfile:
    mem_required_mib: int
    iter_latency_ms: float
    weight_bytes: int
    peak_activation_bytes: int


def profile_graph(graph, weights, ct: CostTable = DEFAULT_COST_TABLE) -> GraphProfile:
    shapes = infer_shapes(graph)
    wbytes = weights.byte_size
    act = peak_activation_bytes(graph, shapes)
    mem = mib_ceil(wbytes + act) + int(math.ceil(ct.per_model_overhead_mib))
    lat = 0.0
    for nid in topo_order(graph):
        node = graph.nodes[nid]
        lat += ct.op_latency_ms(node.kind, node_flops(node, node_input_dims(graph, nid, shapes),
                                                      shapes[nid].dims))
    return GraphProfile(mem, lat, wbytes, act)


def estimate_memory(manifests: Sequence, mode: str, ct: CostTable = DEFAULT_COST_TABLE) -> MemoryEstimate:
    """Reference peak-memory estimate (costmodel.py:252-274)."""
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
    n = len(manifests)
    if n == 0:
        return MemoryEstimate(0.0, 0.0, 0.0, 0.0)
    weights = sum(m.weight_bytes for m in manifests) / MIB
    wa = sum(max(m.mem_required_mib - ct.per_model_overhead_mib, 0.0) for m in manifests)
    acts = max(wa - weights, 0.0)
    if mode == UNFUSED:
        over = n * ct.per_model_overhead_mib
    else:
        over = max(n * ct.per_model_overhead_mib - (n - 1) * ct.dedup_saving_mib_per_extra_model,
                   ct.per_model_overhead_mib)
    return MemoryEstimate(ct.context_base_mib, weights, acts, over)

