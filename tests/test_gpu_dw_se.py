"""The squeeze-excitation absorbed by the depthwise-epilogue GEMM (dfx_gemm_desc.se,
dfx_epi.cuh se_finish): at batch 1-2 an MBConv block's expand conv, depthwise conv,
SE gate and channel scale are ONE launch whose CTAs meet at one grid-wide barrier.

* EfficientNetV2-L at batch 1 and MobileNetV3-L at batch 2 run with every eligible
  SE absorbed (no SE node left where the depthwise epilogue applies);
* logits against the CPU oracle (fp16: 2e-2; fp16x2: 2e-4) and against the
  unfused-SE graph of the same DAG;
* repeated replays (the barrier's epoch words are reused) give identical logits.
"""

import numpy as np
import pytest

from oracle.executor_ref import run_fast
from paper_2410_21120_b200 import device, runtime as rt, zoo
from paper_2410_21120_b200.device import DeviceDag

pytestmark = pytest.mark.gpu


def _rel(got, ref):
    got, ref = got.reshape(len(got), -1), ref.reshape(len(ref), -1)
    return float((np.abs(got - ref).max(1) / np.abs(ref).max(1)).max())


@pytest.mark.parametrize("name,batch,precision", [("efficientnet_v2_l", 1, "fp16x2"),
                                                  ("efficientnet_v2_l", 1, "fp16"),
                                                  ("mobilenet_v3_large", 2, "fp16x2")])
def test_dw_se_fused(monkeypatch, name, batch, precision):
    g, w = zoo.build(name)
    xs = np.random.default_rng(3).standard_normal((batch,) + tuple(g.input_spec.dims)).astype(np.float32)
    outs, n_se = {}, {}
    for fuse_se in (False, True):
        monkeypatch.setattr(device, "GEMM_DW_SE", fuse_se)
        dd = DeviceDag([(g, w)], precision=precision)
        try:
            inst = dd.acquire((batch,))
            n_se[fuse_se] = sum(1 for op, _, _ in inst.nodes if op == rt.OP_SE)
            fused = inst.se_count
            dd.release(inst)
            outs[fuse_se] = [dd.execute([xs])[0] for _ in range(3)]
        finally:
            dd.free()
    assert fused > 0 and n_se[True] == n_se[False] - fused
    for o in outs[True][1:]:                       # barrier words reused across replays
        assert np.array_equal(o, outs[True][0])
    ref = run_fast(g, w, xs)
    tol = 2e-4 if precision == "fp16x2" else 2e-2
    assert _rel(outs[True][0], ref) <= tol
    assert _rel(outs[True][0], outs[False][0]) <= tol


@pytest.mark.parametrize("name,batch,precision", [("efficientnet_v2_l", 1, "fp16x2"),
                                                  ("efficientnet_v2_l", 2, "fp16"),
                                                  ("mobilenet_v3_large", 1, "fp16")])
def test_dw_squeeze_feeds_se(monkeypatch, name, batch, precision):
    """dfx_se_fuse mode 1 (the default at batch <= 2): the depthwise-epilogue GEMM
    writes its channels' means, the SE launch after it skips its pooling pass."""
    g, w = zoo.build(name)
    xs = np.random.default_rng(4).standard_normal((batch,) + tuple(g.input_spec.dims)).astype(np.float32)
    outs, nsq = {}, {}
    for on in (False, True):
        monkeypatch.setattr(device, "GEMM_DW_SQUEEZE", on)
        dd = DeviceDag([(g, w)], precision=precision)
        try:
            inst = dd.acquire((batch,))
            nsq[on] = sum(1 for _, p, _ in inst.nodes if isinstance(p, rt.SeParams) and p.pooled)
            dd.release(inst)
            outs[on] = [dd.execute([xs])[0] for _ in range(2)]
        finally:
            dd.free()
    assert nsq[False] == 0 and nsq[True] > 0
    assert np.array_equal(outs[True][0], outs[True][1])
    tol = 2e-4 if precision == "fp16x2" else 2e-2
    assert _rel(outs[True][0], run_fast(g, w, xs)) <= tol
    assert _rel(outs[True][0], outs[False][0]) <= tol
