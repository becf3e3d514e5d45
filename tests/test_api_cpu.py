"""Drop-in API surface on CPU: fuse/swap structure, errors before compute,
model I/O byte compatibility with reference-written files, repository,
validation codes, and the activation planner against the reference plan.
Restates the reference tests' contracts (tests/test_fuse.py, test_model_io.py,
test_graph_ir.py, test_repo.py under /root/reference/pkg)."""

import threading

import numpy as np
import pytest

from conftest import GOLDEN
from oracle.liveness_ref import peak_by_overlap
from paper_2410_21120_b200 import errors, fuse, graph_ir, model_io, planner
from paper_2410_21120_b200.executor import Tensor
from paper_2410_21120_b200.repo import Repository


# ------------------------------------------------------------------ fusion structure

def test_fuse_structure_and_preamble(corpus):
    models = corpus[:7]
    dag = fuse.fuse_models(models)
    assert dag.model_ids() == [g.model_id for g, _ in models]
    assert dag.cross_edge_count() == 0
    assert dag.node_count() == sum(g.node_count() for g, _ in models)
    assert all(c.multiplicity == 1 for c in dag.preamble.calls)
    assert set(c.function_name for c in dag.preamble.calls) == set(fuse.INIT_FUNCTIONS)
    assert all(c.multiplicity == 7 for c in fuse.build_preamble(7, fused=False).calls)
    sg = dag.subgraphs[0]
    g0, w0 = models[0]
    strip = len(g0.model_id) + 1
    assert {n[strip:] for n in sg.nodes} == set(g0.nodes)
    assert {(a[strip:], b[strip:]) for a, b in sg.edges} == set(g0.edges)
    assert sg.weight_binding is w0


def test_mem_estimate_equals_reference(corpus, corpus_golden):
    for gi in range(int(corpus_golden["n_groups"])):
        members = [corpus[int(i)] for i in corpus_golden[f"group{gi}.members"]]
        dag = fuse.fuse_models(members, validate=False)
        assert dag.total_mem_estimate_mib == float(corpus_golden[f"group{gi}.mem_mib"])


def test_errors_raised_before_any_device_work(corpus):
    models = corpus[:2]
    dag = fuse.fuse_models(models)
    g0, g1 = models[0][0], models[1][0]
    with pytest.raises(errors.MissingInput):
        fuse.execute_fused(dag, {g0.model_id: Tensor.zeros(g0.input_spec)})
    full = {g.model_id: Tensor.zeros(g.input_spec) for g, _ in models}
    with pytest.raises(errors.UnknownSubgraph):
        fuse.execute_fused(dag, {**full, "stranger": Tensor.zeros(g0.input_spec)})
    bad = dict(full)
    bad[g1.model_id] = Tensor.zeros(graph_ir.TensorSpec((1, 2, 3)))
    with pytest.raises(errors.ShapeMismatch):
        fuse.execute_fused(dag, bad)
    with pytest.raises(errors.DuplicateModelId):
        fuse.fuse_models([models[0], models[0]])
    with pytest.raises(ValueError):
        fuse.fuse_models([])


def test_swap_identity_and_errors(corpus):
    models = corpus[100:105]
    dag = fuse.fuse_models(models)
    incoming = corpus[150]
    out_id = models[2][0].model_id
    new = fuse.swap_subgraph(dag, out_id, incoming)
    assert new.compile_generation == dag.compile_generation + 1
    assert new.preamble is dag.preamble
    assert new.model_ids()[2] == incoming[0].model_id
    for a, b in zip(dag.subgraphs, new.subgraphs):
        if a.model_id != out_id:
            assert a is b
    back = fuse.swap_subgraph(new, incoming[0].model_id, models[2])
    assert back.model_ids() == dag.model_ids()
    assert back.subgraphs[2].weight_binding is models[2][1]
    with pytest.raises(errors.UnknownSubgraph):
        fuse.swap_subgraph(dag, "ghost", incoming)
    with pytest.raises(errors.DuplicateModelId):
        fuse.swap_subgraph(dag, models[0][0].model_id, models[1])


def test_validation_failures_surface(corpus):
    g, _ = corpus[0]
    with pytest.raises(errors.ValidationFailed):
        fuse.fuse_models([(g, graph_ir.WeightStore())])


def test_fuse_runtime_linear():
    import time

    def chain(mid, n):
        nodes = [graph_ir.OpNode("n0000", "relu")]
        nodes += [graph_ir.OpNode(f"n{i:04d}", "relu", inputs=(f"n{i - 1:04d}",)) for i in range(1, n)]
        return graph_ir.ModelGraph(mid, nodes, "n0000", f"n{n - 1:04d}", graph_ir.TensorSpec((4,)),
                                   graph_ir.TensorSpec((4,))), graph_ir.WeightStore()

    def best(models):
        t = float("inf")
        for _ in range(3):
            t0 = time.perf_counter()
            fuse.fuse_models(models)
            t = min(t, time.perf_counter() - t0)
        return t

    small = [chain(f"s{i}", 400) for i in range(4)]
    large = [chain(f"l{i}", 800) for i in range(4)]
    best(small)
    assert best(large) <= 2.5 * best(small) + 0.02


# ------------------------------------------------------------------ file formats

def test_model_io_byte_identical_to_reference_files():
    for name in ("zoo_vgg16", "zoo_densenet161", "rm000", "rm137"):
        gpath = GOLDEN / "models" / f"{name}.graph.json"
        wpath = GOLDEN / "models" / f"{name}.weights.fiwt"
        g = model_io.load_graph(gpath)
        w = model_io.load_weights(wpath)
        assert model_io.weights_to_bytes(w) == wpath.read_bytes()
        import json
        assert json.dumps(model_io.graph_to_dict(g), indent=1, sort_keys=True) + "\n" == gpath.read_text()


def test_weights_errors(tmp_path, corpus):
    _, w = corpus[3]
    p = tmp_path / "weights.fiwt"
    model_io.save_weights(w, p)
    blob = bytearray(p.read_bytes())
    bad = tmp_path / "bad.fiwt"
    bad.write_bytes(b"XXXX" + bytes(blob[4:]))
    with pytest.raises(errors.WeightsFormatError) as exc:
        model_io.load_weights(bad)
    assert "bad.fiwt" in str(exc.value) and "magic" in str(exc.value)
    bad.write_bytes(bytes(blob[:-7]))
    with pytest.raises(errors.WeightsFormatError):
        model_io.load_weights(bad)
    bad.write_bytes(bytes(blob) + b"\0")
    with pytest.raises(errors.WeightsFormatError):
        model_io.load_weights(bad)
    gp = tmp_path / "g.json"
    gp.write_text("{not json")
    with pytest.raises(errors.ModelFormatError):
        model_io.load_graph(gp)
    gp.write_text('{"model_id": "m"}')
    with pytest.raises(errors.ModelFormatError):
        model_io.load_graph(gp)


# ------------------------------------------------------------------ repository

def test_repository_round_trip_and_concurrency(tmp_path, corpus):
    repo = Repository(tmp_path / "r")
    for g, w in corpus[:4]:
        repo.register_model(g, w)
    with pytest.raises(errors.DuplicateModelId):
        repo.register_model(*corpus[0])
    with pytest.raises(errors.NotFound):
        repo.lookup("nope")
    again = Repository.open(tmp_path / "r")
    assert again.model_ids() == sorted(g.model_id for g, _ in corpus[:4])
    g2, w2 = again.load_pair(corpus[1][0].model_id)
    assert again.load_pair(corpus[1][0].model_id)[1] is w2          # cached per model id
    for name in corpus[1][1].names():
        assert np.array_equal(w2.values(name), corpus[1][1].values(name))
    errs = []

    def reader():
        try:
            for _ in range(100):
                again.get_many([g.model_id for g, _ in corpus[:3]])
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    def writer():
        try:
            for g, w in corpus[10:20]:
                again.register_model(g, w)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=reader) for _ in range(3)] + [threading.Thread(target=writer)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs and len(again.model_ids()) == 14


# ------------------------------------------------------------------ validation

def test_validation_problem_codes():
    O, S = graph_ir.OpNode, graph_ir.TensorSpec
    loop = graph_ir.ModelGraph("loop", [O("a", "relu", inputs=("b",)), O("b", "relu", inputs=("a",))],
                               "a", "b", S((2,)), S((2,)))
    assert any(p.code == "cycle" for p in graph_ir.validate_graph(loop, graph_ir.WeightStore()).problems)
    st = graph_ir.WeightStore()
    st.put("w", S((5,)), np.ones(5))
    g = graph_ir.ModelGraph("bad", [O("d", "dense", {"units": 1, "fan_in": 4}, {"weight": "w"})],
                            "d", "d", S((4,)), S((1,)))
    assert any(p.code == "weight-shape-mismatch" for p in graph_ir.validate_graph(g, st).problems)
    cat = graph_ir.ModelGraph("m", [O("c", "concat")], "c", "c", S((2,)), S((2,)))
    assert any(p.code in ("arity", "entry-arity") for p in graph_ir.validate_graph(cat, st).problems)
    cs = graph_ir.ModelGraph("m", [O("a", "relu"), O("s", "channel_scale", inputs=("a",))], "a", "s",
                             S((2, 3, 3)), S((2, 3, 3)))
    assert any(p.code == "arity" for p in graph_ir.validate_graph(cs, st).problems)
    with pytest.raises(errors.CycleDetected):
        graph_ir.topo_order(loop)


# ------------------------------------------------------------------ planner (P3)

def test_reference_plan_equals_reference_peak(corpus, corpus_golden, zoo, zoo_golden):
    for models, gold in ((corpus, corpus_golden), (zoo, zoo_golden)):
        for g, _ in models:
            plan = planner.member_plan(g)
            ref = int(gold[f"{g.model_id}.peak"])
            assert plan.peak == ref == peak_by_overlap(g, graph_ir.infer_shapes(g))
            planner.check_disjoint(plan.placements)
            assert plan.arena_bytes >= plan.peak
            assert len(plan.placements) == g.node_count() + 1


def test_fused_arena_sum_and_max(corpus):
    plans = [planner.member_plan(g) for g, _ in corpus[:5]]
    s = planner.fused_arena(plans, "sum", align=1)
    m = planner.fused_arena(plans, "max", align=1)
    assert s.total_bytes == sum(p.arena_bytes for p in plans)
    assert m.total_bytes == max(p.arena_bytes for p in plans)
    offs = [o for _, o, _ in s.segments]
    assert offs == sorted(offs) and all(b - a >= p.arena_bytes for a, b, p in zip(offs, offs[1:], plans))


@pytest.mark.slow
def test_vgg16_reference_plan():
    from paper_2410_21120_b200 import zoo
    g, _ = zoo.BUILDERS["vgg16"](calib={})
    plan = planner.member_plan(g)
    assert plan.peak == graph_ir.peak_activation_bytes(g) == 25_690_112
    planner.check_disjoint(plan.placements)
