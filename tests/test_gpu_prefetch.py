"""L2 prefetch of the next weight blobs from batch-1 GEMMs (dfx_gemm_launch.l2_pf,
device.ExecInstance._set_l2_prefetch): every range lies inside the member's own
weight segment and is exactly the next GEMM's weight blob (or an SE's FC blobs
before it), and the prefetch changes no result bit -- it is a cache hint only.
The chain it shortens is the reference's member-after-member evaluation
(/root/reference/pkg/src/dagfuse/fuse.py:281-290, executor.py:68-92)."""

import numpy as np
import pytest

from paper_2410_21120_b200 import device, runtime as rt, zoo
from paper_2410_21120_b200.device import DeviceDag
from paper_2410_21120_b200.lower import GEMM, SE

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def effnet():
    return [zoo.build("efficientnet_v2_l")]


def _outputs(models, batch, seed=7):
    dd = DeviceDag(models, 0, "concurrent", precision="fp16x2")
    inst = dd.acquire(batch)
    rng = np.random.default_rng(seed)
    xs = [rng.standard_normal((n,) + tuple(g.input_spec.dims)).astype(np.float32)
          for n, (g, _) in zip(batch, models)]
    inst.upload_inputs(xs)
    inst.launch_graph()
    inst.sync()
    return dd, inst, inst.download_outputs()


def test_prefetch_ranges_are_the_next_weight_blobs(effnet):
    dd, inst, _ = _outputs(effnet, (1,))
    prog = dd.programs[0]
    seg_lo, seg_bytes = dd.arena.segment(0)
    weights = {dd.arena.addr(0, L.blobs["weight"]): prog.blobs[L.blobs["weight"]].nbytes
               for L in prog.launches if L.kind == GEMM}
    se_blobs = {dd.arena.addr(0, k) for L in prog.launches if L.kind == SE for k in L.blobs.values()}
    gemms = [p for op, p, _ in inst.nodes if op == rt.OP_GEMM]
    with_pf = [gl for gl in gemms if gl.l2_pf_units]
    assert len(with_pf) >= len(gemms) - 1            # every GEMM but the last prefetches
    for gl in with_pf:
        for r in range(2):
            units = (gl.l2_pf_units >> (16 * r)) & 0xFFFF
            if not units:
                continue
            a, b = gl.l2_pf[r], units * 256
            assert seg_lo <= a and a + b <= seg_lo + seg_bytes
            if r == 0:                                 # the next GEMM's weights, rounded down to 256 B
                assert a in weights and weights[a] - 256 < b <= weights[a]
            else:
                assert a in se_blobs
    dd.free()


def test_prefetch_changes_no_bit(effnet, monkeypatch):
    dd, _, on = _outputs(effnet, (1,))
    dd.free()
    monkeypatch.setattr(device, "L2_PREFETCH", False)
    dd, inst, off = _outputs(effnet, (1,))
    assert all(gl.l2_pf_units == 0 for op, gl, _ in inst.nodes if op == rt.OP_GEMM)
    dd.free()
    for a, b in zip(on, off):
        assert np.array_equal(a, b)
