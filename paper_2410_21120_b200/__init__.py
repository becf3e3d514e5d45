"""B200-native fused multi-CNN DAG (FusedInf, arXiv 2410.21120).

Drop-in for the reference ``dagfuse`` build/load/query path
(/root/reference/pkg/src/dagfuse/__init__.py:10-57): the same names, argument
meanings and error types, with the query path running on sm_100a through
``libdfx`` (include/dfx.h).  Submodules are imported lazily so that the IR,
file formats and planner work without a GPU.
"""

from __future__ import annotations

import importlib

__version__ = "0.1.0"

_EXPORTS = {
    # graph IR
    "ModelGraph": "graph_ir", "OpNode": "graph_ir", "TensorSpec": "graph_ir",
    "ValidationReport": "graph_ir", "WeightStore": "graph_ir", "infer_shapes": "graph_ir",
    "topo_order": "graph_ir", "validate_graph": "graph_ir",
    # executor surface (GPU-backed)
    "Tensor": "executor", "run": "executor", "run_batch": "executor",
    # fusion compiler
    "FusedDag": "fuse", "InitPreamble": "fuse", "SubGraph": "fuse", "execute_fused": "fuse",
    "fuse_models": "fuse", "swap_subgraph": "fuse", "load_fused": "fuse", "unload": "fuse", "nonfinite_outputs": "fuse",
    # repository (read side)
    "Repository": "repo", "ModelManifest": "repo",
    # memory / load accounting
    "estimate_memory": "costmodel", "FUSED": "costmodel", "UNFUSED": "costmodel",
    "MemoryEstimate": "costmodel", "CostTable": "costmodel",
    # errors
    **{n: "errors" for n in (
        "DagfuseError", "ShapeMismatch", "CycleDetected", "MissingWeight", "DuplicateModelId",
        "ValidationFailed", "NotFound", "UnknownSubgraph", "MissingInput", "Unschedulable",
        "BudgetExceeded", "WeightsFormatError", "ModelFormatError", "DeviceError",
        "UnsupportedOnDevice")},
}

__all__ = sorted(_EXPORTS)


def __getattr__(name):
    mod = _EXPORTS.get(name)
    if mod is None:
        raise AttributeError(name)
    return getattr(importlib.import_module(f".{mod}", __name__), name)
