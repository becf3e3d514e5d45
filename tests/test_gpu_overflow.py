"""fp16 overflow is visible, never a clamped finite logit.

Half-precision stores round to nearest without saturation (dfx_common.cuh
Elt<__half>::pack2): an activation beyond 65504 becomes inf (a split fp16x2 value
hi + lo becomes NaN), propagates to the member's logits, and the output kernel
counts it (``fuse.nonfinite_outputs`` / ``dfx_nonfinite_count``).  The reference
is fp32 (/root/reference/pkg/src/dagfuse/executor.py:1-8), so such a logit is a
parity failure the tests and the bench now see."""

from pathlib import Path

import numpy as np
import pytest

from oracle.executor_ref import run_faithful
from paper_2410_21120_b200 import fuse, model_io
from paper_2410_21120_b200.executor import Tensor
from paper_2410_21120_b200.graph_ir import WeightStore

pytestmark = pytest.mark.gpu

MODELS = Path(__file__).parent / "golden" / "models"


def _mlp(scale: float):
    g = model_io.load_graph(MODELS / "mlp_m0.graph.json")
    w = model_io.load_weights(MODELS / "mlp_m0.weights.fiwt")
    if scale != 1.0:
        w2 = WeightStore()
        for name in w.names():
            spec, vals = w.spec(name), np.asarray(w.values(name), dtype=np.float32)
            w2.put(name, spec, vals * (scale if name == "n01_dense.weight" else 1.0))
        w = w2
    return g, w


def _run(models, precision):
    dag = fuse.fuse_models(models)
    fuse.load_fused(dag, precision=precision)
    try:
        x = np.full(models[0][0].input_spec.element_count, 3.0, dtype=np.float32)
        out = fuse.execute_fused(dag, {models[0][0].model_id: Tensor(models[0][0].input_spec, x)})
        return x, np.asarray(out[models[0][0].model_id].values)
    finally:
        fuse.unload(dag)


@pytest.mark.parametrize("precision", ["fp16", "fp16x2"])
def test_overflow_reaches_logits_and_is_counted(precision):
    fuse.nonfinite_outputs(reset=True)
    _, y = _run([_mlp(1.0)], precision)
    assert np.isfinite(y).all()
    assert fuse.nonfinite_outputs() == 0
    _, y = _run([_mlp(1e6)], precision)            # first dense layer far beyond 65504
    assert not np.isfinite(y).all(), y
    n = fuse.nonfinite_outputs(reset=True)
    assert n == int((~np.isfinite(y)).sum()) > 0
    assert fuse.nonfinite_outputs() == 0


def test_bf16_range_holds_the_same_values():
    """bf16 has fp32's exponent range: the scaled model stays finite and near the oracle."""
    fuse.nonfinite_outputs(reset=True)
    g, w = _mlp(1e6)
    x, y = _run([(g, w)], "bf16")
    assert np.isfinite(y).all() and fuse.nonfinite_outputs() == 0
    ref = np.asarray(run_faithful(g, w, x), dtype=np.float64).reshape(-1)
    assert np.max(np.abs(y - ref)) <= 6e-2 * np.max(np.abs(ref))
