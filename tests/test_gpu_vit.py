"""ViT token kernels on the B200 (dfx_vit.cu + the token-row GEMM fold) vs the oracle.

Tiny ViTs cover the edges of the attention kernel (L = 2: one partial key
block; L = 17; L = 65: two key blocks, second one with a single valid key;
two 64-query tiles) in fp16 and bf16; ViT-B/16 itself is checked at B = 3.
Tolerance: the north-star 2e-2 (per sample ||d||inf / ||ref||inf).
"""

import numpy as np
import pytest

from oracle.executor_ref import run_fast
from paper_2410_21120_b200 import fuse, zoo
from paper_2410_21120_b200.device import DeviceDag
from paper_2410_21120_b200.executor import Tensor

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _rel(got, ref):
    return float((np.abs(got - ref).max(axis=1) / np.abs(ref).max(axis=1)).max())


def _tiny(res, patch):
    return zoo.vit_b_16(model_id=f"vit_tiny_{res}_{patch}", res=res, patch=patch, hidden=128,
                        layers=2, heads=2, mlp=256, classes=10)


@pytest.mark.parametrize("precision", ["fp16", "bf16"])
@pytest.mark.parametrize("res,patch", [(16, 16), (32, 8), (64, 8), (96, 8)])   # L = 2, 17, 65, 145
def test_tiny_vit_parity(res, patch, precision):
    g, w = _tiny(res, patch)
    xs = np.random.default_rng(res).standard_normal((3, 3, res, res)).astype(np.float32)
    dag = DeviceDag([(g, w)], precision=precision)
    try:
        got = dag.execute([xs])[0]
    finally:
        dag.free_instances()
    assert _rel(got, run_fast(g, w, xs)) <= TOL


def test_vit_b16_parity():
    g, w = zoo.build("vit_b_16")
    dag = fuse.fuse_models([(g, w)])
    xs = np.random.default_rng(79).standard_normal((3, 3, 224, 224)).astype(np.float32)
    outs = fuse.execute_fused(dag, {g.model_id: [Tensor(g.input_spec, x) for x in xs]})[g.model_id]
    got = np.stack([t.values for t in outs])
    ref = run_fast(g, w, xs)
    assert _rel(got, ref) <= TOL
    assert np.all(got.argmax(1) == ref.argmax(1))
