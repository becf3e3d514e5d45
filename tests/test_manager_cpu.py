"""Manager host logic (paper_2410_21120_b200/manager.py) against the reference
scheduler's own decisions (tests/golden/manager_golden.json, recorded by
tests/golden/make_manager_golden.py from /root/reference's scheduler.py)."""

import json
import threading
from pathlib import Path

import numpy as np
import pytest

from paper_2410_21120_b200 import costmodel, manager, model_io
from paper_2410_21120_b200.executor import Tensor
from paper_2410_21120_b200.repo import ModelManifest, Repository

GOLD = json.loads((Path(__file__).parent / "golden" / "manager_golden.json").read_text())
MODELS = Path(__file__).parent / "golden" / "models"


@pytest.mark.parametrize("case", range(len(GOLD["plans"])))
def test_plan_batches_matches_reference(case):
    c = GOLD["plans"][case]
    manifests = [ModelManifest(m["model_id"], "g", "w", m["mem"], 1.0, m["weight_bytes"], "t")
                 for m in c["models"]]
    plan = manager.plan_batches(manifests, c["budget"], costmodel.DEFAULT_COST_TABLE, quantum_iterations=50,
                                uptime_classes={m["model_id"]: m["cls"] for m in c["models"]}, mode=c["mode"])
    assert [list(b) for b in plan.batches] == c["batches"]
    assert list(plan.batch_estimates_mib) == c["estimates"]          # bit-equal arithmetic
    assert [u[0] for u in plan.unschedulable] == c["unschedulable"]
    if c["unschedulable"]:
        with pytest.raises(manager.Unschedulable):
            manager.require_schedulable(plan)


@pytest.fixture()
def repo(tmp_path):
    r = Repository(tmp_path / "repo", costmodel.DEFAULT_COST_TABLE)
    for i in range(6):
        g = model_io.load_graph(MODELS / f"mlp_m{i}.graph.json")
        w = model_io.load_weights(MODELS / f"mlp_m{i}.weights.fiwt")
        r.register_model(g, w, profile=(50 + 10 * i, 2.0 + i))
    return r


def test_ingest_accepts_and_rejects(repo):
    q = manager.RequestQueue()
    assert manager.ingest(q, manager.InferenceRequest("a", "m0", "zeros", 10), repo) == "accepted"
    assert manager.ingest(q, manager.InferenceRequest("b", "ghost", "zeros", 10), repo) == "rejected"
    assert q.rejected[-1].reason == "unknown model"
    assert manager.ingest(q, manager.InferenceRequest("c", "m0", "zeros", 0), repo) == "rejected"
    assert manager.ingest(q, manager.InferenceRequest("d", "m0", "zeros", 5, "weekly"), repo) == "rejected"
    bad = Tensor.zeros(model_io.load_graph(MODELS / "mlp_m1.graph.json").input_spec)
    spec = repo.input_spec("m0")
    if bad.spec.dims != spec.dims:
        assert manager.ingest(q, manager.InferenceRequest("e", "m0", bad, 5), repo) == "rejected"
    assert len(q) == 1 and [r.request_id for r in q.drain()] == ["a"] and len(q) == 0


def test_ingest_concurrent_fifo_by_arrival(repo):
    q = manager.RequestQueue()

    def producer(k):
        for j in range(50):
            manager.ingest(q, manager.InferenceRequest(f"t{k}_{j}", f"m{k % 6}", "zeros", 1), repo)

    ts = [threading.Thread(target=producer, args=(k,)) for k in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    snap = q.snapshot()
    assert len(snap) == 300
    arrivals = [r.arrival_time for r in snap]
    assert arrivals == sorted(arrivals) and len(set(arrivals)) == 300


def test_manager_needs_no_reference_at_run_time():
    src = (Path(manager.__file__)).read_text()
    assert "/root/reference" not in src.replace("(/root/reference/pkg/src/dagfuse/scheduler.py)", "")
