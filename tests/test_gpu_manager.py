"""The manager on the GPU (paper_2410_21120_b200/manager.py): the reference
scheduler's control flow (cycle order, completions, rotation counts, swap
member sets -- tests/golden/manager_golden.json, recorded from the reference)
with a measured ledger and GPU outputs checked against the CPU oracle."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle.executor_ref import run_faithful
from paper_2410_21120_b200 import costmodel, manager, model_io
from paper_2410_21120_b200.repo import Repository

pytestmark = pytest.mark.gpu

GOLD = json.loads((Path(__file__).parent / "golden" / "manager_golden.json").read_text())
MODELS = Path(__file__).parent / "golden" / "models"
CT = costmodel.DEFAULT_COST_TABLE
TOL = 2e-2


def make_repo(tmp_path, ids):
    r = Repository(tmp_path / "repo", CT)
    prof = {f"m{i}": (50 + 10 * i, 2.0 + i) for i in range(6)} | {"fresh": (55, 3.0)}
    for mid in ids:
        r.register_model(model_io.load_graph(MODELS / f"mlp_{mid}.graph.json"),
                         model_io.load_weights(MODELS / f"mlp_{mid}.weights.fiwt"), profile=prof[mid])
    return r


def rotations(log):
    out, n = {}, 0
    for e in log.events:
        if e.kind == "rotate":
            n += 1
        if e.kind == "complete":
            out[e.payload["request_id"]] = n + 1
    return out


@pytest.mark.parametrize("k", range(len(GOLD["runs"])))
def test_run_plan_control_flow_matches_reference(k, tmp_path):
    g = GOLD["runs"][k]
    repo = make_repo(tmp_path, [f"m{i}" for i in range(6)])
    plan = manager.SchedulePlan(tuple(tuple(b) for b in g["plan"]), g["quantum"], g["budget"],
                                tuple(0.0 for _ in g["plan"]))
    reqs = [manager.InferenceRequest(rid, mid, "zeros", it) for rid, mid, it in g["requests"]]
    log = manager.run_plan(plan, reqs, repo, CT, g["mode"], timing_launches=2)
    assert [c.batch_index for c in log.cycles] == g["cycles"]
    assert sorted(log.completed) == g["completed"]
    assert rotations(log) == g["completion_rotation"]
    assert [e.kind for e in log.events] == g["event_kinds"]
    # measured ledger: real loads and iterations, a real device footprint
    for e in log.events_of("load"):
        if "error" not in e.payload:
            assert e.payload["duration_ms"] > 0 and e.payload["h2d_ms"] >= 0
    for c in log.cycles:
        assert c.iterate_ms > 0 and c.measured_peak_mib > 0
    # GPU outputs against the CPU oracle
    for rid, t in log.completed.items():
        mid = next(m for r, m, _ in g["requests"] if r == rid)
        gr, w = repo.load_pair(mid)
        ref = run_faithful(gr, w, np.zeros(gr.input_spec.element_count, np.float32))
        assert np.abs(t.values - ref).max() <= TOL * max(np.abs(ref).max(), 1e-6)


def test_run_plan_mode_equivalence_bitwise(tmp_path):
    repo = make_repo(tmp_path, [f"m{i}" for i in range(4)])
    plan = manager.plan_batches(repo.get_many([f"m{i}" for i in range(4)]), 24_000, CT)
    mk = lambda: [manager.InferenceRequest(f"e{i}", f"m{i}", f"rand:{40 + i}", 120) for i in range(4)]
    fused = manager.run_plan(plan, mk(), repo, CT, manager.FUSED, timing_launches=2)
    unfused = manager.run_plan(plan, mk(), repo, CT, manager.UNFUSED, timing_launches=2)
    assert set(fused.completed) == set(unfused.completed) == {f"e{i}" for i in range(4)}
    for rid in fused.completed:
        assert np.array_equal(fused.completed[rid].values, unfused.completed[rid].values)
    # one fused load vs four, one DAG iteration for all members vs four
    assert len(fused.events_of("load")) == len(unfused.events_of("load")) == 1


def test_run_swap_schedule_matches_reference(tmp_path):
    repo = make_repo(tmp_path, ["m0", "m1", "m2", "m3", "fresh"])
    swaps = [manager.SwapStep(25, "m1", "fresh"), manager.SwapStep(50, "m0", "m3")]
    for g in GOLD["swaps"]:
        log, records = manager.run_swap_schedule(["m0", "m1", "m2"], swaps, 25, repo, CT, g["mode"], 24_000.0,
                                                 timing_launches=2)
        assert [list(r.model_ids) for r in records] == g["segments"]
        assert [e.kind for e in log.events] == g["event_kinds"]
        ev = log.events_of("swap_subgraph")
        for got, want in zip(ev, g["swap_events"]):
            assert got.payload["out"] == want["out"] and got.payload["in"] == want["in"]
            if "untouched" in want:
                assert sorted(got.payload["untouched"]) == sorted(want["untouched"])
            assert got.payload["duration_ms"] > 0
        assert all(b.cumulative_ms > a.cumulative_ms for a, b in zip(records, records[1:]))


def test_request_swap_guards(tmp_path):
    repo = make_repo(tmp_path, ["m0", "m1", "m2", "fresh"])
    from paper_2410_21120_b200 import fuse
    dag = fuse.fuse_models([repo.load_pair(m) for m in ("m0", "m1", "m2")], cost_table=CT)
    mans = repo.get_many(["m0", "m1", "m2"])
    big = manager.ModelManifest("fresh", "g", "w", 30_000, 1.0, 1, "t")
    with pytest.raises(manager.BudgetExceeded):
        manager.request_swap(dag, "m1", repo.load_pair("fresh"), big, mans, 2_000.0, CT)
    with pytest.raises(manager.UnknownSubgraph):
        manager.request_swap(dag, "ghost", repo.load_pair("fresh"), repo.lookup("fresh"), mans, 50_000.0, CT)
