"""``Tensor`` and the single-model query surface, executed on the B200.

Same names and semantics as the reference executor surface
(/root/reference/pkg/src/dagfuse/executor.py:22-46, 187-201): ``run`` evaluates
one model on one input, ``run_batch`` maps over a list preserving order.
Here both go through the fused-DAG device path (a one-member DAG, resident
on GPU 0 and cached per (graph, weights) object pair); ``run_batch`` sends
the whole list as ONE batched graph launch.  There is no CPU fallback: without
libdfx or a B200 the call raises ``DeviceError``.
"""

from __future__ import annotations

import threading
import weakref
from dataclasses import dataclass

import numpy as np

from .errors import ShapeMismatch
from .graph_ir import TensorSpec

F32 = np.float32


@dataclass(frozen=True)
class Tensor:
    """Spec + flat read-only fp32 values (executor.py:22-46)."""

    spec: TensorSpec
    values: np.ndarray

    def __post_init__(self):
        arr = np.asarray(self.values, dtype=F32).reshape(-1)
        if arr.size != self.spec.element_count:
            raise ValueError(f"{arr.size} values for shape {self.spec.dims}")
        if arr.flags.writeable:
            arr = arr.view()
            arr.setflags(write=False)
        object.__setattr__(self, "values", arr)

    @staticmethod
    def from_array(arr) -> "Tensor":
        a = np.asarray(arr, dtype=F32)
        return Tensor(TensorSpec(a.shape), a.reshape(-1))

    @staticmethod
    def zeros(spec: TensorSpec) -> "Tensor":
        return Tensor(spec, np.zeros(spec.element_count, dtype=F32))

    def array(self) -> np.ndarray:
        return self.values.reshape(self.spec.dims)


# (id(g), id(w)) -> (weakref g, weakref w, DeviceDag): the solo device DAG of a
# (graph, weights) pair lives as long as both objects do (a finalizer frees it)
_solo: dict[tuple[int, int], tuple] = {}
_solo_lock = threading.Lock()


def _drop_solo(key) -> None:
    with _solo_lock:
        hit = _solo.pop(key, None)
    if hit is not None:
        hit[2].free()


def _solo_dag(g, w):
    from .device import DeviceDag
    key = (id(g), id(w))
    with _solo_lock:
        hit = _solo.get(key)
        if hit is not None and hit[0]() is g and hit[1]() is w:
            return hit[2]
    d = DeviceDag([(g, w)])
    with _solo_lock:
        old = _solo.get(key)
        _solo[key] = (weakref.ref(g), weakref.ref(w), d)
    if old is not None:
        old[2].free()
    for obj in (g, w):
        weakref.finalize(obj, _drop_solo, key).atexit = False
    return d


def run(g, w, x: Tensor) -> Tensor:
    if x.spec.dims != g.input_spec.dims:
        raise ShapeMismatch(g.entry, f"input {x.spec.dims} vs declared {g.input_spec.dims}")
    (out,) = _solo_dag(g, w).execute([x.values.reshape((1,) + g.input_spec.dims)])
    return Tensor(g.output_spec, out.reshape(-1))


def run_batch(g, w, xs: list[Tensor]) -> list[Tensor]:
    if not xs:
        return []
    for x in xs:
        if x.spec.dims != g.input_spec.dims:
            raise ShapeMismatch(g.entry, f"input {x.spec.dims} vs declared {g.input_spec.dims}")
    batch = np.stack([x.values for x in xs]).reshape((len(xs),) + g.input_spec.dims)
    (out,) = _solo_dag(g, w).execute([batch])
    return [Tensor(g.output_spec, o.reshape(-1)) for o in out]
