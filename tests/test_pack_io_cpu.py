"""Packed-arena files (paper_2410_21120_b200/pack_io.py), host side: the file
holds exactly the bytes device.WeightArena would upload, and the header and
program table round-trip."""

from pathlib import Path

import numpy as np

from paper_2410_21120_b200 import fuse, model_io, pack_io
from paper_2410_21120_b200.device import arena_layout, fill_arena, program_for

GOLD = Path(__file__).parent / "golden" / "models"


def members():
    out = []
    for mid in ("zoo_vgg16_bn", "zoo_mobilenet_v3_large", "zoo_densenet161"):
        out.append((model_io.load_graph(GOLD / f"{mid}.graph.json"),
                    model_io.load_weights(GOLD / f"{mid}.weights.fiwt")))
    return out


def test_packed_file_is_the_device_arena(tmp_path):
    mem = members()
    dag = fuse.fuse_models(mem)
    path = tmp_path / "dag.dfxpack"
    header = pack_io.save_packed(dag, path)
    hdr, table, off = pack_io.read_header(path)
    assert hdr == header and off % pack_io.PAGE == 0
    progs = [program_for(fuse._as_graph(sg), sg.weight_binding, "fp16") for sg in dag.subgraphs]
    layout, segments, total = arena_layout(progs)
    assert total == hdr["total"] and [m["blobs"] for m in hdr["members"]] == [dict(l) for l in layout]
    want = np.zeros(total, np.uint8)
    fill_arena(want, progs, layout)
    got = np.fromfile(path, np.uint8, offset=off)
    assert got.size == total and np.array_equal(got, want)
    for p, t, m in zip(progs, table, hdr["members"]):
        assert t.model_id == p.model_id and len(t.launches) == len(p.launches)
        assert t.blobs == {k: (str(v.dtype), tuple(v.shape)) for k, v in p.blobs.items()}
        g = model_io.graph_from_dict(m["graph"])
        assert model_io.graph_to_dict(g) == m["graph"]


def test_packed_weights_are_specs_only():
    spec = pack_io.TensorSpec((4, 3))
    w = pack_io.PackedWeights({"a": spec})
    assert "a" in w and w.byte_size == spec.byte_size and w.spec("a") == spec
    import pytest
    with pytest.raises(LookupError):
        w.values("a")
    with pytest.raises(TypeError):
        w.put("b", spec, np.zeros(12))


def test_rejects_foreign_files(tmp_path):
    p = tmp_path / "x.fiwt"
    p.write_bytes(b"FIWT" + b"\0" * 64)
    import pytest
    with pytest.raises(ValueError):
        pack_io.read_header(p)
