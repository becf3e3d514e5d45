"""The CPU oracle and the IR/planner, pinned against the reference's own outputs.

Fixtures come from tests/golden/make_golden.py (which imports the reference).
Bitwise where the reference is deterministic: faithful engine outputs, topo
orders, liveness peaks.
"""

import json

import numpy as np
import pytest

from conftest import golden_input
from oracle.executor_ref import run_fast, run_faithful
from oracle.liveness_ref import peak_by_overlap
from paper_2410_21120_b200 import graph_ir


def test_zoo_faithful_bitwise(zoo, zoo_golden):
    for g, w in zoo:
        xs = zoo_golden[f"{g.model_id}.x"]
        ys = zoo_golden[f"{g.model_id}.y"]
        for x, y in zip(xs, ys):
            assert np.array_equal(run_faithful(g, w, x), y), g.model_id


def test_corpus_faithful_bitwise(corpus, corpus_golden):
    for i, (g, w) in enumerate(corpus):
        ys = corpus_golden[f"{g.model_id}.y"]
        for t, y in enumerate(ys):
            x = golden_input(g.input_spec.dims, 7919 * i + t)
            assert np.array_equal(run_faithful(g, w, x), y), (g.model_id, t)


def test_corpus_fast_engine_close(corpus, corpus_golden):
    for i, (g, w) in enumerate(corpus):
        xs = np.stack([golden_input(g.input_spec.dims, 7919 * i + t) for t in range(4)])
        got = run_fast(g, w, xs).reshape(4, -1)
        ref = corpus_golden[f"{g.model_id}.y"]
        err = np.abs(got - ref).max(axis=1) / np.maximum(np.abs(ref).max(axis=1), 1e-30)
        assert err.max() < 1e-5, g.model_id


def test_topo_order_and_peak_match_reference(corpus, corpus_golden, zoo, zoo_golden):
    for models, gold in ((corpus, corpus_golden), (zoo, zoo_golden)):
        for g, _ in models:
            assert graph_ir.topo_order(g) == json.loads(str(gold[f"{g.model_id}.order"]))
            peak = graph_ir.peak_activation_bytes(g)
            assert peak == int(gold[f"{g.model_id}.peak"])
            assert peak == peak_by_overlap(g, graph_ir.infer_shapes(g))


def test_all_nine_reference_kinds_covered(corpus):
    kinds = {n.kind for g, _ in corpus for n in g.nodes.values()}
    assert kinds == set(graph_ir.REFERENCE_KINDS)


# --- known answers restated from the reference tests -------------------------

def _single(node, in_dims, out_dims, store=None):
    g = graph_ir.ModelGraph("m", [node], node.node_id, node.node_id,
                            graph_ir.TensorSpec(in_dims), graph_ir.TensorSpec(out_dims))
    return g, store or graph_ir.WeightStore()


def test_conv_hand_computed():
    # reference tests/test_executor.py:30-40: [[1,2],[3,4]] * [[1,0],[0,1]] = 5
    s = graph_ir.WeightStore()
    s.put("k", graph_ir.TensorSpec((1, 1, 2, 2)), [1.0, 0.0, 0.0, 1.0])
    node = graph_ir.OpNode("c", "conv2d", {"out_channels": 1, "kernel": 2}, {"weight": "k"})
    g, w = _single(node, (1, 2, 2), (1, 1, 1), s)
    assert run_faithful(g, w, np.array([1, 2, 3, 4], np.float32)).tolist() == [5.0]


def test_relu_known_answer():
    g, w = _single(graph_ir.OpNode("r", "relu"), (3,), (3,))
    assert run_faithful(g, w, np.array([-1, 0, 2], np.float32)).tolist() == [0, 0, 2]


def test_extension_known_answers():
    x = np.array([-4.0, -3.0, -1.0, 0.0, 1.0, 3.0, 4.0], np.float32)
    for kind, expect in (
        ("hardswish", [0, 0, -1 * 2 / 6, 0, 4 / 6, 3, 4]),
        ("hardsigmoid", [0, 0, 2 / 6, 0.5, 4 / 6, 1, 1]),
        ("sigmoid", 1 / (1 + np.exp(-x.astype(np.float64)))),
        ("silu", x / (1 + np.exp(-x.astype(np.float64)))),
    ):
        g, w = _single(graph_ir.OpNode("a", kind), (7,), (7,))
        assert np.allclose(run_faithful(g, w, x), expect, rtol=1e-6, atol=1e-7), kind


def test_depthwise_and_padded_pools_known_answers():
    x = np.arange(1, 2 * 4 * 4 + 1, dtype=np.float32)
    s = graph_ir.WeightStore()
    s.put("dw", graph_ir.TensorSpec((2, 1, 3, 3)), np.concatenate([np.ones(9), 2 * np.ones(9)]))
    node = graph_ir.OpNode("d", "conv2d", {"out_channels": 2, "kernel": 3, "padding": 1,
                                            "groups": 2}, {"weight": "dw"})
    g, w = _single(node, (2, 4, 4), (2, 4, 4), s)
    out = run_faithful(g, w, x).reshape(2, 4, 4)
    a = x.reshape(2, 4, 4)
    assert out[0, 0, 0] == a[0, :2, :2].sum()
    assert out[1, 1, 1] == 2 * a[1, :3, :3].sum()
    mp = graph_ir.OpNode("p", "maxpool2d", {"kernel": 3, "stride": 2, "padding": 1})
    g, w = _single(mp, (2, 4, 4), (2, 2, 2))
    out = run_faithful(g, w, x).reshape(2, 2, 2)
    assert out[0, 0, 0] == a[0, :2, :2].max() and out[1, 1, 1] == a[1, 1:4, 1:4].max()
    ap = graph_ir.OpNode("q", "avgpool2d", {"kernel": 3, "stride": 2, "padding": 1,
                                             "count_include_pad": 0})
    g, w = _single(ap, (2, 4, 4), (2, 2, 2))
    out = run_faithful(g, w, x).reshape(2, 2, 2)
    assert np.isclose(out[0, 0, 0], a[0, :2, :2].mean(), rtol=1e-6)
    ap2 = graph_ir.OpNode("q", "avgpool2d", {"kernel": 2})
    g, w = _single(ap2, (2, 4, 4), (2, 2, 2))
    out = run_faithful(g, w, x).reshape(2, 2, 2)
    assert np.isclose(out[1, 1, 0], a[1, 2:4, 0:2].mean(), rtol=1e-6)


def test_fast_engine_matches_faithful_on_extension_kinds():
    rng = np.random.default_rng(3)
    s = graph_ir.WeightStore()
    s.put("dw", graph_ir.TensorSpec((6, 1, 5, 5)), rng.standard_normal(150))
    s.put("pw", graph_ir.TensorSpec((4, 6, 1, 1)), rng.standard_normal(24))
    s.put("gw", graph_ir.TensorSpec((4, 2, 3, 3)), rng.standard_normal(72))
    nodes = [
        graph_ir.OpNode("a", "conv2d", {"out_channels": 6, "kernel": 5, "stride": 2,
                                         "padding": 2, "groups": 6}, {"weight": "dw"}),
        graph_ir.OpNode("b", "hardswish", inputs=("a",)),
        graph_ir.OpNode("c", "global_avg_pool", inputs=("b",)),
        graph_ir.OpNode("d", "sigmoid", inputs=("c",)),
        graph_ir.OpNode("e", "channel_scale", inputs=("b", "d")),
        graph_ir.OpNode("f", "conv2d", {"out_channels": 4, "kernel": 1}, {"weight": "pw"}, ("e",)),
        graph_ir.OpNode("h", "silu", inputs=("f",)),
        graph_ir.OpNode("i", "avgpool2d", {"kernel": 3, "stride": 1, "padding": 1,
                                            "count_include_pad": 0}, inputs=("h",)),
        graph_ir.OpNode("j", "maxpool2d", {"kernel": 3, "stride": 2, "padding": 1}, inputs=("i",)),
        graph_ir.OpNode("k", "conv2d", {"out_channels": 4, "kernel": 3, "padding": 1,
                                         "groups": 2, "padding_w": 0, "kernel_w": 3},
                        {"weight": "gw"}, ("j",)),
    ]
    g = graph_ir.ModelGraph("ext", nodes, "a", "k", graph_ir.TensorSpec((6, 11, 11)),
                            graph_ir.TensorSpec((4, 3, 1)))
    assert graph_ir.validate_graph(g, s).ok, graph_ir.validate_graph(g, s).problems
    xs = rng.standard_normal((3, 6, 11, 11)).astype(np.float32)
    fast = run_fast(g, s, xs).reshape(3, -1)
    for i in range(3):
        ref = run_faithful(g, s, xs[i])
        assert np.allclose(fast[i], ref, rtol=1e-5, atol=1e-5)
