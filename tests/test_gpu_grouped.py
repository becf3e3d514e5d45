"""Grouped implicit GEMM across members (north-star subsystem 4; dfx_gemm.cu's
ndesc > 1 path): two concurrent members whose GEMM sequences share layer shapes
(ResNet-50 and ResNet-152: stem, layer1, layer2 and the common blocks of layer3/4)
run those layers as ONE gemm_kernel launch over both problems
(device.ExecInstance._pair_chains / _group_launch).

* grouped == ungrouped bitwise (each tile computes exactly what it did alone);
* both against the CPU oracle (fp16x2: the accurate storage, 2e-4);
* the launch count drops by the number of grouped pairs.
The reference evaluates members one after another
(/root/reference/pkg/src/dagfuse/fuse.py:281-290, executor.py:68-92)."""

import numpy as np
import pytest

from oracle.executor_ref import run_fast
from paper_2410_21120_b200 import device, zoo
from paper_2410_21120_b200.device import DeviceDag

pytestmark = pytest.mark.gpu


def _models():
    r50 = zoo.resnet50(model_id="r50s", res=64, classes=10)
    r152 = zoo.resnet152(model_id="r152s", res=64, classes=10)
    return [r50, r152]


@pytest.mark.parametrize("precision,batch", [("fp16x2", (1, 2)), ("fp16", (2, 2))])
def test_grouped_gemm_matches_ungrouped_and_oracle(monkeypatch, precision, batch):
    members = _models()
    rng = np.random.default_rng(5)
    xs = [rng.standard_normal((b,) + tuple(g.input_spec.dims)).astype(np.float32) for b, (g, _) in zip(batch, members)]
    outs, launches, grouped = {}, {}, {}
    for flag in (False, True):
        monkeypatch.setattr(device, "GROUP_GEMM", flag)
        monkeypatch.setattr(device, "GROUP_MIN", 1)
        dd = DeviceDag(members, 0, "concurrent", precision=precision)
        try:
            inst = dd.acquire(tuple(batch))
            launches[flag], grouped[flag] = inst.kernel_nodes, inst.grouped_launches
            dd.release(inst)
            outs[flag] = dd.execute(xs)
        finally:
            dd.free()
    assert grouped[False] == 0 and grouped[True] >= 16
    assert launches[True] == launches[False] - grouped[True]
    for a, b in zip(outs[False], outs[True]):
        assert np.array_equal(a, b)
    if precision != "fp16x2":          # uncalibrated random-init nets: the oracle check
        return                         # is made at the accurate storage
    for (g, w), x, got in zip(members, xs, outs[True]):
        ref = run_fast(g, w, x)
        err = np.abs(got.reshape(len(x), -1) - ref.reshape(len(x), -1)).max(1) / np.abs(ref.reshape(len(x), -1)).max(1)
        assert err.max() <= 2e-4, (g.model_id, err)
