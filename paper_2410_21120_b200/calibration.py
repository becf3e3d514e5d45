"""B200 recalibration of the reference's loading cost model.

The reference prices swap-in with a calibrated table of per-function totals
for an N-model episode in both modes, plus memory constants and per-kind op
latencies (/root/reference/pkg/src/dagfuse/costmodel.py:51-140, file format
:391-474, paper table in calibration/paper_tableIV.cfg).  ``measure`` runs
that episode on the B200 with this package's real loaders and returns a
``CostTable`` of measured numbers; ``dump_cost_table`` writes it in the
reference's own "key = value" format, so the reference's ``load_cost_table``
(and with it ``plan_batches`` / ``simulate_load`` / ``simulate_swap``) runs on
B200 numbers unchanged.  ``simulate_load`` / ``simulate_swap`` here restate
the reference's scaling rules (costmodel.py:145-330) so a calibration can be
checked against held-out measured loads.

What each priced function is on this system:

* ``cudaMalloc``: unfused = one cudaMalloc per weight tensor (``PerTensorArena``);
  fused = the arena's one cudaMalloc;
* ``cudaMemcpyAsync``: unfused = one copy per tensor from pageable memory; fused =
  the one pinned H2D of the packed arena; ``calibration_weight_bytes`` = the
  episode's fp32 weight bytes (the reference's volume unit);
* ``get_schema``: unfused = per member, graph JSON parse + lowering + packing;
  fused = reading the DAG's packed-arena header + program table once (pack_io);
* the device queries (cuDeviceGet ... cudaStreamIsCapturing): timed through
  libcudart / libcuda, called once per member unfused and once fused;
* ``op_latency_ms_per_mflop``: measured device time per MFLOP of each IR kind
  at batch 1 (a launch's time is charged to its anchor node's kind);
* ``context_base_mib``: device memory the CUDA context holds (cudaMemGetInfo);
  ``per_model_overhead_mib``: measured per-member instance memory beyond
  weights (activation arena + I/O + descriptors) of the unfused images.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field
from pathlib import Path

from . import costmodel
from .costmodel import FUSED, MIB, MODES, UNFUSED

DEVICE_FUNCTIONS = ("cuDeviceGet", "cuDeviceGetCount", "cuDriverGetVersion", "cudaGetDevice",
                    "cudaGetDeviceCount", "cudaSetDevice", "cudaStreamIsCapturing")
MALLOC_FUNCTION, MEMCPY_FUNCTION, SCHEMA_FUNCTION = "cudaMalloc", "cudaMemcpyAsync", "get_schema"
INIT_FUNCTIONS = DEVICE_FUNCTIONS + (MALLOC_FUNCTION, MEMCPY_FUNCTION, SCHEMA_FUNCTION)


@dataclass(frozen=True)
class FunctionCost:                        # costmodel.py:103-113
    unfused_total_ms: float
    fused_total_ms: float


@dataclass(frozen=True)
class CostTable(costmodel.CostTable):
    """The reference CostTable's fields (costmodel.py:116-192) over this
    package's memory CostTable (so ``estimate_memory`` / the planner take it)."""
    init_call_costs: dict = field(default_factory=dict)
    calibration_models: int = 7
    calibration_weight_bytes: int = 1
    teardown_ms: float = 0.0

    @property
    def function_names(self) -> tuple[str, ...]:
        return tuple(self.init_call_costs)

    def one_member_cost_ms(self, name: str) -> float:
        return self.init_call_costs[name].unfused_total_ms / self.calibration_models

    def function_cost_ms(self, name: str, members: int, mode: str) -> float:
        """Unfused: linear through the origin; fused: the line through one member's
        cost and the calibration total, clamped at zero (costmodel.py:152-166)."""
        cost, cal = self.init_call_costs[name], self.calibration_models
        if mode == UNFUSED:
            return cost.unfused_total_ms * members / cal
        single = self.one_member_cost_ms(name)
        if members == 1:
            return single
        return max(single + (cost.fused_total_ms - single) / (cal - 1) * (members - 1), 0.0)

    def marginal_fused_cost_ms(self, name: str) -> float:
        cost = self.init_call_costs[name]
        return max((cost.fused_total_ms - self.one_member_cost_ms(name)) / (self.calibration_models - 1), 0.0)

    def memcpy_ms(self, weight_bytes: int, mode: str) -> float:
        t = self.init_call_costs[MEMCPY_FUNCTION]
        return (t.unfused_total_ms if mode == UNFUSED else t.fused_total_ms) * weight_bytes / \
            self.calibration_weight_bytes


def simulate_load(manifests, mode: str, ct: CostTable) -> dict[str, float]:
    """Phase times of loading a member set (costmodel.py:277-305): init, malloc, memcpy."""
    if mode not in MODES or not manifests:
        raise ValueError("simulate_load needs a mode and at least one member")
    n, wb = len(manifests), sum(m.weight_bytes for m in manifests)
    ft = {name: (ct.memcpy_ms(wb, mode) if name == MEMCPY_FUNCTION else ct.function_cost_ms(name, n, mode))
          for name in ct.function_names}
    init = sum(v for k, v in ft.items() if k not in (MALLOC_FUNCTION, MEMCPY_FUNCTION))
    return dict(init=init, malloc=ft.get(MALLOC_FUNCTION, 0.0), memcpy=ft.get(MEMCPY_FUNCTION, 0.0),
                teardown=ct.teardown_ms, total=init + ft.get(MALLOC_FUNCTION, 0.0)
                + ft.get(MEMCPY_FUNCTION, 0.0) + ct.teardown_ms)


def simulate_swap(incoming, mode: str, ct: CostTable) -> dict[str, float]:
    """One member swapped into a loaded set (costmodel.py:308-338)."""
    ft = {}
    for name in ct.function_names:
        if name == MEMCPY_FUNCTION:
            ft[name] = ct.memcpy_ms(incoming.weight_bytes, mode)
        else:
            ft[name] = ct.one_member_cost_ms(name) if mode == UNFUSED else ct.marginal_fused_cost_ms(name)
    init = sum(v for k, v in ft.items() if k not in (MALLOC_FUNCTION, MEMCPY_FUNCTION))
    return dict(init=init, malloc=ft[MALLOC_FUNCTION], memcpy=ft[MEMCPY_FUNCTION],
                total=init + ft[MALLOC_FUNCTION] + ft[MEMCPY_FUNCTION] + ct.teardown_ms)


# ------------------------------------------------------------------ file format (costmodel.py:391-474)
_UNIT_MS = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1000.0}


def _fmt(ms: float) -> tuple[float, str]:
    if ms < 1e-2:
        return ms * 1e6, "ns"
    if ms >= 1000.0:
        return ms / 1000.0, "s"
    return ms, "ms"


def dump_cost_table(ct: CostTable, path, header: str = "") -> None:
    lines = ["# Device cost calibration measured on NVIDIA B200 (paper_2410_21120_b200.calibration):",
             f"# per-function initialization totals for a {ct.calibration_models}-model episode,",
             "# memory constants and transfer volume, in the reference's cost-table format."]
    lines += [f"# {h}" for h in header.splitlines()] + [""]
    lines += [f"calibration_models = {ct.calibration_models}",
              f"calibration_weight_bytes = {ct.calibration_weight_bytes}",
              f"context_base_mib = {ct.context_base_mib!r}",
              f"per_model_overhead_mib = {ct.per_model_overhead_mib!r}",
              f"dedup_saving_mib_per_extra_model = {ct.dedup_saving_mib_per_extra_model!r}",
              f"teardown_ms = {ct.teardown_ms!r}", ""]
    for name in ct.function_names:
        c = ct.init_call_costs[name]
        for mode, ms in ((UNFUSED, c.unfused_total_ms), (FUSED, c.fused_total_ms)):
            v, u = _fmt(ms)
            lines.append(f"init.{name}.{mode}_{u} = {v!r}")
    lines.append("")
    for kind, v in sorted(ct.op_latency_ms_per_mflop.items()):
        lines.append(f"op_latency_ms_per_mflop.{kind} = {v!r}")
    Path(path).write_text("\n".join(lines) + "\n")


def load_cost_table(path) -> CostTable:
    scalars, init, ops = {}, {}, {}
    for lineno, line in enumerate(Path(path).read_text().splitlines(), 1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        key, raw = (p.strip() for p in line.split("=", 1))
        if key.startswith("init."):
            _, fn, tail = key.split(".")
            mode, _, unit = tail.rpartition("_")
            init.setdefault(fn, {})[mode] = float(raw) * _UNIT_MS[unit]
        elif key.startswith("op_latency_ms_per_mflop."):
            ops[key.split(".", 1)[1]] = float(raw)
        else:
            scalars[key] = float(raw)
    return CostTable(context_base_mib=scalars["context_base_mib"],
                     per_model_overhead_mib=scalars["per_model_overhead_mib"],
                     dedup_saving_mib_per_extra_model=scalars["dedup_saving_mib_per_extra_model"],
                     op_latency_ms_per_mflop=ops,
                     init_call_costs={k: FunctionCost(v[UNFUSED], v[FUSED]) for k, v in init.items()},
                     calibration_models=int(scalars["calibration_models"]),
                     calibration_weight_bytes=int(scalars["calibration_weight_bytes"]),
                     teardown_ms=scalars.get("teardown_ms", 0.0))


# ------------------------------------------------------------------ measurement (GPU)
def _device_query_ms(reps: int) -> dict[str, float]:
    """Wall ms of one call of each device query, median of ``reps``."""
    import statistics
    cudart = C.CDLL("libcudart.so") if _has("libcudart.so") else None
    cuda = C.CDLL("libcuda.so.1")
    i, dev = C.c_int(), C.c_int()
    cap = C.c_int()
    calls = {
        "cuDeviceGet": lambda: cuda.cuDeviceGet(C.byref(dev), 0),
        "cuDeviceGetCount": lambda: cuda.cuDeviceGetCount(C.byref(i)),
        "cuDriverGetVersion": lambda: cuda.cuDriverGetVersion(C.byref(i)),
    }
    if cudart is not None:
        calls.update({
            "cudaGetDevice": lambda: cudart.cudaGetDevice(C.byref(i)),
            "cudaGetDeviceCount": lambda: cudart.cudaGetDeviceCount(C.byref(i)),
            "cudaSetDevice": lambda: cudart.cudaSetDevice(0),
            "cudaStreamIsCapturing": lambda: cudart.cudaStreamIsCapturing(None, C.byref(cap)),
        })
    cuda.cuInit(0)
    out = {}
    for name in DEVICE_FUNCTIONS:
        f = calls.get(name)
        if f is None:
            out[name] = 0.0
            continue
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            f()
            ts.append((time.perf_counter() - t0) * 1e3)
        out[name] = statistics.median(ts)
    return out


def _has(lib: str) -> bool:
    try:
        C.CDLL(lib)
        return True
    except OSError:
        return False


def measure(models, workdir, precision: str = "fp16", device: int = 0) -> tuple[CostTable, dict]:
    """Run the calibration episode for ``models`` [(graph, weights)] on the GPU and
    return (CostTable, report).  ``workdir`` receives the graph / packed files.
    The episode books cudaMalloc explicitly and reads per-model overheads from
    cudaMemGetInfo deltas, so arenas use plain cudaMalloc here (the retained
    arena pool would hide both)."""
    from . import device as _dev
    saved = _dev.ARENA_POOL
    _dev.ARENA_POOL = False
    try:
        return _measure(models, workdir, precision, device)
    finally:
        _dev.ARENA_POOL = saved


def _measure(models, workdir, precision: str = "fp16", device: int = 0) -> tuple[CostTable, dict]:
    from . import fuse, model_io, pack_io, runtime as rt
    from .device import DeviceDag, PerTensorArena, WeightArena, program_for
    from .lower import lower_member
    rt.init_device(device)
    workdir = Path(workdir)
    workdir.mkdir(parents=True, exist_ok=True)
    n = len(models)
    free_ctx, total = rt.mem_info()
    context_mib = (total - free_ctx) / MIB
    wbytes = sum(w.byte_size for _, w in models)
    # get_schema: unfused = parse + lower + pack per member; fused = one packed header
    for g, _ in models:
        model_io.save_graph(g, workdir / f"{g.model_id}.graph.json")
    t_unf = 0.0
    for g, w in models:
        t0 = time.perf_counter()
        g2 = model_io.load_graph(workdir / f"{g.model_id}.graph.json")
        lower_member(g2, w, precision=precision)
        t_unf += time.perf_counter() - t0
    dag = fuse.fuse_models(models)
    pack_io.save_packed(dag, workdir / "episode.dfxpack", precision=precision)
    t0 = time.perf_counter()
    pack_io.read_header(workdir / "episode.dfxpack")
    t_fus = time.perf_counter() - t0
    programs = [program_for(g, w, precision) for g, w in models]
    # cudaMalloc / cudaMemcpyAsync: per-tensor unfused vs one arena fused (median of 3)
    unf, fus = [], []
    for _ in range(3):
        pt = PerTensorArena(programs, device)
        unf.append((pt.malloc_ms, pt.memcpy_ms))
        pt.free()
        wa = WeightArena(programs, device)
        wa.upload()
        fus.append((wa.malloc_ms, wa.memcpy_ms))
        wa.free()
    unf.sort(key=lambda t: sum(t))
    fus.sort(key=lambda t: sum(t))
    q = _device_query_ms(50)
    costs = {name: FunctionCost(q[name] * n, q[name]) for name in DEVICE_FUNCTIONS}
    costs[MALLOC_FUNCTION] = FunctionCost(unf[1][0], min(fus[1][0], unf[1][0]))
    costs[MEMCPY_FUNCTION] = FunctionCost(unf[1][1], min(fus[1][1], unf[1][1]))
    costs[SCHEMA_FUNCTION] = FunctionCost(t_unf * 1e3, min(t_fus * 1e3, t_unf * 1e3))
    # memory: per-member instance overhead of the unfused images (beyond weights + activations)
    overheads, ops = [], {}
    for (g, w), prog in zip(models, programs):
        f0, _ = rt.mem_info()
        img = DeviceDag([(g, w)], device, programs=[prog], precision=precision)
        inst = img.acquire((1,))
        f1, _ = rt.mem_info()
        act = costmodel.profile_graph(g, w).peak_activation_bytes
        overheads.append(max((f0 - f1 - prog.weight_bytes() - act) / MIB, 0.0))
        for r in inst.profile_nodes(reps=4):
            kind = g.nodes[r["node"]].kind if r.get("node") in g.nodes else None
            if kind and r["flops"]:
                a = ops.setdefault(kind, [0.0, 0.0])
                a[0] += r["ms"]
                a[1] += r["flops"] / 1e6
        img.free()
    per_model = float(sum(overheads) / n)
    ct = CostTable(context_base_mib=round(context_mib, 1), per_model_overhead_mib=round(per_model, 1),
                   dedup_saving_mib_per_extra_model=round(per_model, 1),
                   op_latency_ms_per_mflop={k: (ms / mf) for k, (ms, mf) in sorted(ops.items())},
                   init_call_costs=costs, calibration_models=n, calibration_weight_bytes=int(wbytes))
    report = dict(models=[g.model_id for g, _ in models], weight_bytes=wbytes, context_mib=context_mib,
                  per_model_overhead_mib=overheads, unfused_malloc_memcpy_ms=unf, fused_malloc_memcpy_ms=fus,
                  schema_ms={"unfused": t_unf * 1e3, "fused": t_fus * 1e3}, device_query_ms=q)
    return ct, report
