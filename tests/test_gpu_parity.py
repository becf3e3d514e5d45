"""GPU parity: the sm_100a path (through libdfx) against the CPU oracle.

Tolerance (north star): per sample ||gpu - ref||inf / ||ref||inf <= 2e-2 for
every model at the default fp16 storage.  With bf16 storage a few random-init
toy models exceed it (the CPU emulation of the lowered program shows the same
margin, test_lowering_cpu.py), so the bf16 run is held to >= 97% of models at
2e-2 and every model at 6e-2.
"""

import threading

import numpy as np
import pytest

from conftest import golden_input
from oracle.executor_ref import run_faithful, run_fast
from paper_2410_21120_b200 import fuse, graph_ir
from paper_2410_21120_b200.executor import Tensor, run, run_batch

pytestmark = pytest.mark.gpu

TOL = 2e-2
TOY_MAX = 6e-2


def rel(got, ref):
    got = np.asarray(got, np.float64).reshape(len(got), -1)
    ref = np.asarray(ref, np.float64).reshape(len(ref), -1)
    return (np.abs(got - ref).max(axis=1) / np.maximum(np.abs(ref).max(axis=1), 1e-30)).max()


def single(node, in_dims, out_dims, store):
    return graph_ir.ModelGraph(node.node_id, [node], node.node_id, node.node_id,
                               graph_ir.TensorSpec(in_dims), graph_ir.TensorSpec(out_dims)), store


CONV_CASES = [
    # cin, h, w, cout, k, stride, pad, n
    (3, 8, 8, 4, 3, 1, 1, 2),
    (3, 32, 32, 64, 7, 2, 3, 2),
    (16, 17, 13, 24, 3, 1, 1, 3),
    (48, 14, 14, 192, 1, 1, 0, 2),
    (64, 28, 28, 128, 3, 2, 1, 1),
    (144, 7, 7, 48, 3, 1, 1, 4),
    (256, 14, 14, 512, 3, 1, 1, 1),
    (512, 7, 7, 1000, 1, 1, 0, 2),
    (40, 9, 11, 300, 5, 2, 2, 2),
]


@pytest.mark.parametrize("cin,h,w,cout,k,s,p,n", CONV_CASES)
def test_conv_layer(cin, h, w, cout, k, s, p, n):
    rng = np.random.default_rng(cin * 1000 + cout)
    st = graph_ir.WeightStore()
    st.put("w", graph_ir.TensorSpec((cout, cin, k, k)), rng.standard_normal(cout * cin * k * k) / np.sqrt(cin * k * k))
    st.put("b", graph_ir.TensorSpec((cout,)), rng.standard_normal(cout) * 0.1)
    node = graph_ir.OpNode("c", "conv2d", {"out_channels": cout, "kernel": k, "stride": s, "padding": p},
                           {"weight": "w", "bias": "b"})
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    g, st = single(node, (cin, h, w), (cout, oh, ow), st)
    xs = rng.standard_normal((n, cin, h, w)).astype(np.float32)
    got = [t.values for t in run_batch(g, st, [Tensor(g.input_spec, x) for x in xs])]
    ref = run_fast(g, st, xs)
    assert rel(got, ref) < TOL


# depthwise conv: 3x3 layers on the column-strip kernel (dfx_dw.cu: whole columns
# or row strips by grid size, stride 1 / 2, odd sizes), 5x5 on the tiled kernel
# (1, 2 or 4 outputs per thread by grid size, ragged last pixel group), and the
# generic kernel (C = 12)
DW_CASES = [
    # c, h, w, k, stride, n
    (16, 9, 11, 3, 1, 2), (32, 56, 56, 3, 1, 8), (24, 17, 23, 3, 2, 3), (72, 28, 28, 5, 2, 16),
    (40, 14, 13, 5, 1, 4), (96, 112, 112, 3, 2, 2), (12, 10, 10, 3, 1, 2),
    (1056, 14, 14, 3, 1, 32), (3840, 7, 7, 3, 1, 8), (48, 15, 15, 3, 2, 16), (64, 112, 112, 3, 1, 4),
]


@pytest.mark.parametrize("c,h,w,k,s,n", DW_CASES)
def test_depthwise_layer(c, h, w, k, s, n):
    rng = np.random.default_rng(c * 100 + h + k)
    st = graph_ir.WeightStore()
    st.put("w", graph_ir.TensorSpec((c, 1, k, k)), rng.standard_normal(c * k * k) / k)
    st.put("b", graph_ir.TensorSpec((c,)), rng.standard_normal(c) * 0.1)
    p = k // 2
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    nodes = [graph_ir.OpNode("d", "conv2d", {"out_channels": c, "kernel": k, "stride": s, "padding": p,
                                             "groups": c}, {"weight": "w", "bias": "b"}),
             graph_ir.OpNode("a", "silu", {}, {}, ("d",))]
    g = graph_ir.ModelGraph("dw", nodes, "d", "a", graph_ir.TensorSpec((c, h, w)),
                            graph_ir.TensorSpec((c, oh, ow)))
    xs = rng.standard_normal((n, c, h, w)).astype(np.float32)
    got = [t.values for t in run_batch(g, st, [Tensor(g.input_spec, x) for x in xs])]
    ref = run_fast(g, st, xs)
    assert rel(got, ref) < TOL


# large-M layers that take the 256-row CTA path (two M tiles per CTA sharing each
# weight stage, lower.gemm_tiling m2), including an odd M-tile count (last CTA
# holds one tile) and a stride-2 input; m2 needs >= 24 K stages (shorter K goes to
# the persistent kernel)
M2_CASES = [(192, 28, 28, 256, 3, 1, 1, 21), (192, 28, 28, 128, 3, 1, 1, 64),
            (1536, 14, 14, 256, 1, 1, 0, 148), (192, 56, 56, 256, 3, 2, 1, 21)]


@pytest.mark.parametrize("cin,h,w,cout,k,s,p,n", M2_CASES)
def test_conv_layer_m2_tiles(cin, h, w, cout, k, s, p, n):
    from paper_2410_21120_b200.lower import choose_cb, gemm_tiling
    cb = choose_cb(cin)
    oh = (h + 2 * p - k) // s + 1
    t = gemm_tiling(dict(cout=cout, cb=cb, ksteps=k * k * (-(-cin // cb)), sh=s, sw=s), n, oh, oh)
    assert t["m2"] == 1
    test_conv_layer(cin, h, w, cout, k, s, p, n)


# multi-wave layers that take the persistent kernel (dfx_gemm_persist.cu: one CTA
# per SM walks the tile list, a ring of TMEM accumulators): bn 64 / 128 / 256,
# ragged output width and channel tail
PERSIST_CASES = [(16, 112, 112, 64, 3, 1, 1, 4), (32, 56, 56, 128, 3, 1, 1, 13),
                 (24, 56, 56, 256, 1, 1, 0, 12), (40, 60, 57, 200, 3, 1, 1, 11)]


@pytest.mark.parametrize("cin,h,w,cout,k,s,p,n", PERSIST_CASES)
def test_conv_layer_persistent(cin, h, w, cout, k, s, p, n):
    from paper_2410_21120_b200.lower import choose_cb, gemm_tiling
    cb = choose_cb(cin)
    t = gemm_tiling(dict(cout=cout, cb=cb, ksteps=k * k * (-(-cin // cb)), sh=s, sw=s), n,
                    (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1)
    assert not t["m2"] and t["splits"] == 1 and t["tiles"] > 2 * 148
    test_conv_layer(cin, h, w, cout, k, s, p, n)


@pytest.mark.parametrize("units,fan_in,n", [(10, 7, 1), (4096, 25088 // 49, 2), (1000, 1280, 3), (240, 960, 1)])
def test_dense_layer(units, fan_in, n):
    rng = np.random.default_rng(units)
    st = graph_ir.WeightStore()
    st.put("w", graph_ir.TensorSpec((units, fan_in)), rng.standard_normal(units * fan_in) / np.sqrt(fan_in))
    st.put("b", graph_ir.TensorSpec((units,)), rng.standard_normal(units) * 0.1)
    node = graph_ir.OpNode("d", "dense", {"units": units, "fan_in": fan_in}, {"weight": "w", "bias": "b"})
    g, st = single(node, (fan_in,), (units,), st)
    xs = rng.standard_normal((n, fan_in)).astype(np.float32)
    got = [t.values for t in run_batch(g, st, [Tensor(g.input_spec, x) for x in xs])]
    assert rel(got, run_fast(g, st, xs)) < TOL


def test_extension_kinds_chain():
    rng = np.random.default_rng(5)
    st = graph_ir.WeightStore()
    st.put("dw", graph_ir.TensorSpec((24, 1, 5, 5)), rng.standard_normal(600) * 0.2)
    st.put("f1", graph_ir.TensorSpec((8, 24)), rng.standard_normal(192) * 0.2)
    st.put("f2", graph_ir.TensorSpec((24, 8)), rng.standard_normal(192) * 0.3)
    st.put("pw", graph_ir.TensorSpec((16, 24, 1, 1)), rng.standard_normal(384) * 0.2)
    for nm in ("g", "b", "m", "v"):
        st.put(nm, graph_ir.TensorSpec((24,)), rng.uniform(0.5, 1.5, 24) if nm in "gv" else rng.standard_normal(24) * 0.1)
    O = graph_ir.OpNode
    nodes = [
        O("a", "conv2d", {"out_channels": 24, "kernel": 5, "stride": 2, "padding": 2, "groups": 24}, {"weight": "dw"}),
        O("b", "batchnorm_inference", {}, {"gamma": "g", "beta": "b", "mean": "m", "var": "v"}, ("a",)),
        O("c", "hardswish", inputs=("b",)),
        O("d", "global_avg_pool", inputs=("c",)),
        O("e", "dense", {"units": 8, "fan_in": 24}, {"weight": "f1"}, ("d",)),
        O("f", "silu", inputs=("e",)),
        O("h", "dense", {"units": 24, "fan_in": 8}, {"weight": "f2"}, ("f",)),
        O("i", "hardsigmoid", inputs=("h",)),
        O("j", "channel_scale", inputs=("c", "i")),
        O("k", "conv2d", {"out_channels": 16, "kernel": 1}, {"weight": "pw"}, ("j",)),
        O("l", "avgpool2d", {"kernel": 3, "stride": 2, "padding": 1, "count_include_pad": 0}, inputs=("k",)),
        O("m", "maxpool2d", {"kernel": 3, "stride": 1, "padding": 1}, inputs=("l",)),
        O("n", "sigmoid", inputs=("m",)),
    ]
    g = graph_ir.ModelGraph("ext", nodes, "a", "n", graph_ir.TensorSpec((24, 20, 20)), graph_ir.TensorSpec((16, 5, 5)))
    assert graph_ir.validate_graph(g, st).ok
    xs = rng.standard_normal((3, 24, 20, 20)).astype(np.float32)
    got = [t.values for t in run_batch(g, st, [Tensor(g.input_spec, x) for x in xs])]
    assert rel(got, run_fast(g, st, xs)) < TOL


def test_toy_zoo(zoo, zoo_golden):
    for g, w in zoo:
        xs = zoo_golden[f"{g.model_id}.x"]
        got = [t.values for t in run_batch(g, w, [Tensor(g.input_spec, x) for x in xs])]
        assert rel(got, zoo_golden[f"{g.model_id}.y"]) < TOL, g.model_id


def test_corpus_fused_vs_reference_and_solo(corpus, corpus_golden):
    errs = []
    n_groups = int(corpus_golden["n_groups"])
    for gi in range(n_groups):
        members = [int(i) for i in corpus_golden[f"group{gi}.members"]]
        models = [corpus[i] for i in members]
        dag = fuse.fuse_models(models, validate=False)
        assert dag.total_mem_estimate_mib == float(corpus_golden[f"group{gi}.mem_mib"])
        for t in range(2):
            inputs = {corpus[i][0].model_id: Tensor(corpus[i][0].input_spec,
                                                    golden_input(corpus[i][0].input_spec.dims, 7919 * i + t))
                      for i in members}
            outs = fuse.execute_fused(dag, inputs)
            for i in members:
                g, w = corpus[i]
                ref = corpus_golden[f"{g.model_id}.y"][t]
                errs.append(rel([outs[g.model_id].values], [ref]))
                # fused and solo GPU runs use identical kernels in identical order: bitwise
                solo = run(g, w, inputs[g.model_id])
                assert np.array_equal(solo.values, outs[g.model_id].values), g.model_id
    errs = np.array(errs)
    assert errs.max() <= TOL, np.sort(errs)[-8:]


def test_corpus_bf16_storage(corpus, corpus_golden):
    errs = []
    n_groups = int(corpus_golden["n_groups"])
    for gi in range(n_groups):
        members = [int(i) for i in corpus_golden[f"group{gi}.members"]]
        dag = fuse.fuse_models([corpus[i] for i in members], validate=False)
        fuse.load_fused(dag, precision="bf16")
        inputs = {corpus[i][0].model_id: Tensor(corpus[i][0].input_spec,
                                                golden_input(corpus[i][0].input_spec.dims, 7919 * i))
                  for i in members}
        outs = fuse.execute_fused(dag, inputs)
        for i in members:
            mid = corpus[i][0].model_id
            errs.append(rel([outs[mid].values], [corpus_golden[f"{mid}.y"][0]]))
    errs = np.array(errs)
    assert (errs <= TOL).mean() >= 0.97, np.sort(errs)[-8:]
    assert errs.max() < TOY_MAX


def test_batched_members_and_empty(corpus):
    models = corpus[:3]
    dag = fuse.fuse_models(models)
    rng = np.random.default_rng(1)
    inputs = {g.model_id: [Tensor(g.input_spec, rng.standard_normal(g.input_spec.element_count))
                           for _ in range(k)] for k, (g, _) in zip((5, 0, 2), models)}
    outs = fuse.execute_fused(dag, inputs)
    assert [len(outs[g.model_id]) for g, _ in models] == [5, 0, 2]
    for k, (g, w) in zip((5, 0, 2), models):
        for x, y in zip(inputs[g.model_id], outs[g.model_id]):
            assert np.array_equal(run(g, w, x).values, y.values)


def test_swap_subgraph_on_device(corpus):
    models = corpus[10:14]
    dag = fuse.fuse_models(models)
    rng = np.random.default_rng(2)
    inputs = {g.model_id: Tensor(g.input_spec, rng.standard_normal(g.input_spec.element_count)) for g, _ in models}
    before = fuse.execute_fused(dag, inputs)
    incoming = corpus[20]
    new = fuse.swap_subgraph(dag, models[1][0].model_id, incoming)
    inputs2 = dict(inputs)
    del inputs2[models[1][0].model_id]
    inputs2[incoming[0].model_id] = Tensor(incoming[0].input_spec,
                                           rng.standard_normal(incoming[0].input_spec.element_count))
    after = fuse.execute_fused(new, inputs2)
    for g, w in (models[0], models[2], models[3]):
        assert np.array_equal(before[g.model_id].values, after[g.model_id].values)
    ref = run_faithful(incoming[0], incoming[1], inputs2[incoming[0].model_id].values)
    assert rel([after[incoming[0].model_id].values], [ref]) < TOL
    # the pre-swap DAG still answers correctly (re-loaded on demand)
    again = fuse.execute_fused(dag, inputs)
    for g, _ in models:
        assert np.array_equal(again[g.model_id].values, before[g.model_id].values)


def test_concurrent_execute_fused(corpus):
    models = corpus[30:33]
    dag = fuse.fuse_models(models)
    rng = np.random.default_rng(3)
    inputs = {g.model_id: Tensor(g.input_spec, rng.standard_normal(g.input_spec.element_count)) for g, _ in models}
    ref = fuse.execute_fused(dag, inputs)
    results, errors = [], []

    def worker():
        try:
            for _ in range(5):
                results.append(fuse.execute_fused(dag, inputs))
        except Exception as exc:  # noqa: BLE001
            errors.append(exc)

    ts = [threading.Thread(target=worker) for _ in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for out in results:
        for mid in ref:
            assert np.array_equal(out[mid].values, ref[mid].values)


# cluster split-K (DFX_SPLITK=cluster, dfx_gemm.cu): the splits of an output tile
# reduce over DSMEM in rank order; small-M layers with 2..8 splits
@pytest.mark.parametrize("cin,h,w,cout,k,s,p,n", [(192, 7, 7, 256, 3, 1, 1, 1), (1344, 14, 14, 224, 1, 1, 0, 1),
                                                  (1536, 7, 7, 384, 1, 1, 0, 2), (1024, 7, 7, 130, 1, 1, 0, 3)])
def test_conv_layer_cluster_splitk(cin, h, w, cout, k, s, p, n, monkeypatch):
    from paper_2410_21120_b200 import device, lower
    monkeypatch.setattr(lower, "SPLITK_MODE", "cluster")
    monkeypatch.setattr(device, "SPLITK_MODE", "cluster")
    cb = lower.choose_cb(cin)
    oh = (h + 2 * p - k) // s + 1
    t = lower.gemm_tiling(dict(cout=cout, cb=cb, ksteps=k * k * (-(-cin // cb)), sh=s, sw=s), n, oh, oh)
    assert t["csplit"] == 1 and 2 <= t["splits"] <= 8
    test_conv_layer(cin, h, w, cout, k, s, p, n)


# A-operand prologue transform (DFX_FOLD_PRE=1, lower.fold_pre_transforms): DenseNet's
# pre-activation BN + ReLU (mode 1) and the SE channel scale (mode 2) folded into the
# 1x1 conv that consumes them; freshly built models so the program cache misses
@pytest.mark.parametrize("name,mode", [("densenet161", 0), ("mobilenet_v3_large", 2)])
def test_fold_pre_transform(name, mode, monkeypatch):
    from paper_2410_21120_b200 import lower, zoo
    monkeypatch.setattr(lower, "FOLD_PRE", True)
    monkeypatch.setattr(lower, "SE_FUSE_SCALE", False)     # keep the scale as its own node
    g, w = zoo.build(name)
    prog = lower.lower_member(g, w)
    assert {L.pre.binop for L in prog.launches if L.pre is not None} == {mode}
    rng = np.random.default_rng(5)
    xs = rng.standard_normal((2,) + tuple(g.input_spec.dims)).astype(np.float32)
    got = [t.values for t in run_batch(g, w, [Tensor(g.input_spec, x) for x in xs])]
    ref = run_fast(g, w, xs)
    assert rel(got, ref) < TOL


# dw -> SE -> scale as one cluster launch (DFX_FUSE_DWSE=1, dfx_fused.cu dwse_kernel):
# MobileNetV3-L (3x3 / 5x5, stride 1 / 2, hardsigmoid gates) and EfficientNetV2-L's
# MBConv blocks at a small and a multi-image batch
@pytest.mark.parametrize("name,n", [("mobilenet_v3_large", 3), ("efficientnet_v2_l", 2)])
def test_fused_dw_se(name, n, monkeypatch):
    from paper_2410_21120_b200 import lower, zoo
    monkeypatch.setattr(lower, "FUSE_DWSE", True)
    monkeypatch.setattr(lower, "SE_FUSE_SCALE", False)
    g, w = zoo.build(name)
    prog = lower.lower_member(g, w)
    assert sum(L.kind == lower.DWSE for L in prog.launches) in (8, 61)
    rng = np.random.default_rng(11)
    xs = rng.standard_normal((n,) + tuple(g.input_spec.dims)).astype(np.float32)
    got = [t.values for t in run_batch(g, w, [Tensor(g.input_spec, x) for x in xs])]
    ref = run_fast(g, w, xs)
    assert rel(got, ref) < TOL


# squeeze-excitation with 4 images per cluster (batch >= 8, dfx_fused.cu se_kernel IPI = 4),
# including a last cluster with a partial image group (batch 10)
def test_se_multi_image_batch():
    import os
    from paper_2410_21120_b200 import zoo
    if os.environ.get("DFX_SE_IPI", "1") != "4":
        pytest.skip("4-image SE clusters are an A/B option (run with DFX_SE_IPI=4)")
    g, w = zoo.build("mobilenet_v3_large")
    rng = np.random.default_rng(17)
    xs = rng.standard_normal((10,) + tuple(g.input_spec.dims)).astype(np.float32)
    got = [t.values for t in run_batch(g, w, [Tensor(g.input_spec, x) for x in xs])]
    ref = run_fast(g, w, xs)
    assert rel(got, ref) < TOL
