#!/usr/bin/env python3
"""Golden fixtures for the manager (paper_2410_21120_b200/manager.py).

Runs ONLY in the build container: imports the read-only reference at
/root/reference/pkg and records what ITS scheduler decides (nothing is
copied).  Output (committed): manager_golden.json with

  plans      ``scheduler.plan_batches`` on 40 seeded random manifest sets
             (memory, weight bytes, uptime classes, budget, mode): batches,
             estimates, unschedulable ids;
  runs       ``scheduler.run_plan`` control flow on toy MLP repositories
             (reference tests/test_scheduler.py:29-35 shapes): the batch index
             of every cycle, the completed request ids, and the rotation count
             at which each request completed -- the parts of the ledger that do
             not depend on simulated time, so the GPU manager must match them;
  swaps      ``scheduler.run_swap_schedule`` member sets per segment;
  models/mlp_*.graph.json / .weights.fiwt: the toy MLPs (``toygen.mlp``)
             those runs use, written by the reference's model_io.

Usage:  python tests/golden/make_manager_golden.py
"""

from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent / "manager_golden.json"
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF / "src"))

from dagfuse import costmodel, model_io, scheduler, toygen  # noqa: E402
from dagfuse.repo import ModelManifest, Repository  # noqa: E402


def plan_cases(ct):
    cases = []
    for seed in range(40):
        rng = np.random.default_rng(9000 + seed)
        n = int(rng.integers(1, 12))
        models = []
        for i in range(n):
            mem = int(rng.integers(20, 4000))
            wb = int(rng.integers(1, max(2, mem)) * (1 << 20) * rng.uniform(0.1, 0.9))
            models.append(dict(model_id=f"p{seed}_{i:02d}", mem=mem, weight_bytes=wb,
                               cls=["short", "long"][int(rng.integers(0, 2))]))
        budget = float(rng.integers(1000, 12000))
        mode = ["fused", "unfused"][seed % 2]
        manifests = [ModelManifest(m["model_id"], "g", "w", m["mem"], 1.0, m["weight_bytes"], "t")
                     for m in models]
        plan = scheduler.plan_batches(manifests, budget, ct, quantum_iterations=50,
                                      uptime_classes={m["model_id"]: m["cls"] for m in models}, mode=mode)
        cases.append(dict(models=models, budget=budget, mode=mode,
                          batches=[list(b) for b in plan.batches],
                          estimates=list(plan.batch_estimates_mib),
                          unschedulable=[u[0] for u in plan.unschedulable]))
    return cases


def _completion_rotations(log):
    out, rotations = {}, 0
    for e in log.events:
        if e.kind == "rotate":
            rotations += 1
        if e.kind == "complete":
            out[e.payload["request_id"]] = rotations + 1
    return out


def run_cases(ct):
    runs = []
    scenarios = [
        # (profiles per model, plan batches or None (= plan_batches), quantum, requests)
        dict(batches=[["m0"], ["m1"]], quantum=100, reqs=[("m0", 200), ("m1", 200)]),
        dict(batches=[["m0"], ["m1"], ["m2"]], quantum=100, reqs=[("m0", 300), ("m2", 100)]),
        dict(batches=None, budget=24000.0, quantum=100, reqs=[("m0", 50)]),
        dict(batches=[["m0", "m1"], ["m2"]], quantum=30, reqs=[("m0", 70), ("m1", 20), ("m2", 45),
                                                              ("m0", 10), ("m1", 61)]),
        dict(batches=None, budget=620.0, quantum=40, reqs=[("m0", 90), ("m1", 30), ("m2", 50),
                                                          ("m3", 120), ("m4", 10), ("m5", 41)]),
    ]
    for k, sc in enumerate(scenarios):
        with tempfile.TemporaryDirectory() as td:
            repo = Repository(Path(td) / "repo", ct)
            for i in range(6):
                g, w = toygen.mlp(f"m{i}", i)
                repo.register_model(g, w, profile=(50 + 10 * i, 2.0 + i))
            if sc["batches"] is None:
                ids = sorted({m for m, _ in sc["reqs"]})
                plan = scheduler.plan_batches(repo.get_many(ids), sc["budget"], ct,
                                              quantum_iterations=sc["quantum"])
            else:
                plan = scheduler.SchedulePlan(tuple(tuple(b) for b in sc["batches"]), sc["quantum"],
                                              24000.0, tuple(0.0 for _ in sc["batches"]))
            reqs = [scheduler.InferenceRequest(f"q{k}_{j}", m, "zeros", it) for j, (m, it) in enumerate(sc["reqs"])]
            for mode in ("fused", "unfused"):
                log = scheduler.run_plan(plan, [scheduler.InferenceRequest(r.request_id, r.model_id, "zeros",
                                                                           r.iterations_requested) for r in reqs],
                                         repo, ct, mode)
                runs.append(dict(scenario=k, mode=mode, plan=[list(b) for b in plan.batches],
                                 quantum=plan.quantum_iterations, budget=plan.device_budget_mib,
                                 requests=[[r.request_id, r.model_id, r.iterations_requested] for r in reqs],
                                 cycles=[c.batch_index for c in log.cycles],
                                 completed=sorted(log.completed),
                                 completion_rotation=_completion_rotations(log),
                                 event_kinds=[e.kind for e in log.events]))
    return runs


def swap_cases(ct):
    with tempfile.TemporaryDirectory() as td:
        repo = Repository(Path(td) / "repo", ct)
        for i in range(4):
            g, w = toygen.mlp(f"m{i}", i)
            repo.register_model(g, w, profile=(50 + 10 * i, 2.0 + i))
        g, w = toygen.mlp("fresh", 99)
        repo.register_model(g, w, profile=(55, 3.0))
        swaps = [scheduler.SwapStep(25, "m1", "fresh"), scheduler.SwapStep(50, "m0", "m3")]
        out = []
        for mode in ("fused", "unfused"):
            log, records = scheduler.run_swap_schedule(["m0", "m1", "m2"], swaps, 25, repo, ct, mode, 24000.0)
            out.append(dict(mode=mode, segments=[list(r.model_ids) for r in records],
                            swap_events=[{k: v for k, v in e.payload.items() if k in ("out", "in", "untouched")}
                                         for e in log.events_of("swap_subgraph")],
                            event_kinds=[e.kind for e in log.events]))
        return out


def save_models():
    d = OUT.parent / "models"
    d.mkdir(exist_ok=True)
    for mid, seed in [(f"m{i}", i) for i in range(6)] + [("fresh", 99)]:
        g, w = toygen.mlp(mid, seed)
        model_io.save_graph(g, d / f"mlp_{mid}.graph.json")
        model_io.save_weights(w, d / f"mlp_{mid}.weights.fiwt")


def main():
    ct = costmodel.DEFAULT_COST_TABLE
    save_models()
    payload = dict(plans=plan_cases(ct), runs=run_cases(ct), swaps=swap_cases(ct),
                   toy_mlp_seeds={f"m{i}": i for i in range(6)} | {"fresh": 99})
    OUT.write_text(json.dumps(payload, indent=1, sort_keys=True) + "\n")
    print("wrote", OUT, len(payload["plans"]), "plans", len(payload["runs"]), "runs")


if __name__ == "__main__":
    main()
