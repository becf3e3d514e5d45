"""Packed-arena swap-in on the GPU (pack_io.load_packed): one read into pinned
memory + one H2D; outputs bit-equal to the same DAG loaded from FIWT weights,
and swap_subgraph still works on a DAG whose weights live only on disk/GPU."""

from pathlib import Path

import numpy as np
import pytest

from oracle.executor_ref import run_faithful
from paper_2410_21120_b200 import fuse, model_io, pack_io
from paper_2410_21120_b200.executor import Tensor

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden" / "models"


def pair(mid):
    return model_io.load_graph(GOLD / f"{mid}.graph.json"), model_io.load_weights(GOLD / f"{mid}.weights.fiwt")


@pytest.mark.parametrize("pinned", [False, True])
def test_load_packed_matches_fiwt_path(tmp_path, pinned):
    mem = [pair(m) for m in ("zoo_vgg16_bn", "zoo_resnet50", "zoo_mobilenet_v3_large")]
    dag = fuse.fuse_models(mem)
    path = tmp_path / "dag.dfxpack"
    pack_io.save_packed(dag, path)
    packed = pack_io.load_packed(path, pinned=pinned)
    assert packed.total_mem_estimate_mib == dag.total_mem_estimate_mib and packed.model_ids() == dag.model_ids()
    arena = fuse.device_image(packed).arena
    assert arena.read_ms > 0 and arena.memcpy_ms > 0 and arena.total == pack_io.read_header(path)[0]["total"]
    rng = np.random.default_rng(3)
    inputs = {g.model_id: Tensor(g.input_spec, rng.standard_normal(g.input_spec.element_count)) for g, _ in mem}
    want = fuse.execute_fused(dag, inputs)
    got = fuse.execute_fused(packed, inputs)
    for g, w in mem:
        assert np.array_equal(got[g.model_id].values, want[g.model_id].values)
        ref = run_faithful(g, w, inputs[g.model_id].values)
        assert np.abs(got[g.model_id].values - ref).max() <= 2e-2 * np.abs(ref).max()
    with pytest.raises(LookupError):
        packed.subgraphs[0].weight_binding.values(packed.subgraphs[0].weight_binding.names()[0])
    fuse.unload(dag)
    # swap one member of the packed DAG: only the incoming segment is uploaded
    g2, w2 = pair("zoo_densenet161")
    out_id, keep_id = mem[1][0].model_id, mem[0][0].model_id
    swapped = fuse.swap_subgraph(packed, out_id, (g2, w2))
    x2 = {**inputs, g2.model_id: Tensor(g2.input_spec, rng.standard_normal(g2.input_spec.element_count))}
    x2.pop(out_id)
    out = fuse.execute_fused(swapped, x2)
    ref = run_faithful(g2, w2, x2[g2.model_id].values)
    assert np.abs(out[g2.model_id].values - ref).max() <= 2e-2 * np.abs(ref).max()
    assert np.array_equal(out[keep_id].values, want[keep_id].values)
    fuse.unload(swapped)
