#!/usr/bin/env python3
"""Generate the golden fixtures that pin the oracle and the planner.

Runs ONLY in the build container, where the reference package is mounted
read-only at /root/reference.  It imports the reference itself and records
its outputs; nothing under /root/reference is copied.  Outputs (committed):

  toy_zoo.npz        the 34 toy-zoo models regenerated exactly as
                     tools/make_fixtures.py:213-222 does (seeds 101.. in
                     sorted model-id order), 3 inputs each, reference
                     ``executor.run`` outputs, ``peak_activation_bytes`` and
                     ``topo_order``
  corpus.npz         the C1 corpus of tests/test_acceptance.py:59-71
                     (200 ``toygen.random_model``s, groups from
                     default_rng(20_24)), 4 inputs per model, reference
                     outputs and ``execute_fused`` outputs per group
  models/            graph JSON + FIWT of every model above, written by the
                     REFERENCE ``save_graph`` / ``save_weights`` (so our
                     model_io is checked byte-for-byte against them)

Inputs are N(0,1) fp32 from ``np.random.default_rng(seed)`` with
seed = 7919 * model_index + trial (toy zoo: 104729 + ...), regenerable
without the reference.

Usage:  python tests/golden/make_golden.py
"""

from __future__ import annotations

import importlib.util
import json
import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF / "src"))

from dagfuse import executor, fuse, graph_ir, model_io, toygen  # noqa: E402


def _load_zoo_table():
    spec = importlib.util.spec_from_file_location("ref_make_fixtures", REF / "tools" / "make_fixtures.py")
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod
    spec.loader.exec_module(mod)
    return mod.ZOO


def input_for(spec_dims, seed):
    n = int(np.prod(spec_dims))
    return np.random.default_rng(seed).standard_normal(n).astype(np.float32)


def toy_zoo():
    zoo = _load_zoo_table()
    rows = {}
    models_dir = OUT / "models"
    models_dir.mkdir(exist_ok=True)
    for seed, (mid, (family, params)) in enumerate(sorted(zoo.items()), start=101):
        g, w = toygen.FAMILIES[family](mid, seed, **params)
        model_io.save_graph(g, models_dir / f"zoo_{mid}.graph.json")
        model_io.save_weights(w, models_dir / f"zoo_{mid}.weights.fiwt")
        xs, ys = [], []
        for t in range(3):
            x = input_for(g.input_spec.dims, 104729 + 13 * seed + t)
            y = executor.run(g, w, executor.Tensor(g.input_spec, x)).values
            xs.append(x)
            ys.append(np.array(y))
        rows[mid] = dict(seed=seed, x=np.stack(xs), y=np.stack(ys),
                         peak=graph_ir.peak_activation_bytes(g),
                         order=json.dumps(graph_ir.topo_order(g)))
    np.savez_compressed(
        OUT / "toy_zoo.npz",
        ids=np.array(sorted(rows)),
        **{f"{m}.x": r["x"] for m, r in rows.items()},
        **{f"{m}.y": r["y"] for m, r in rows.items()},
        **{f"{m}.peak": np.int64(r["peak"]) for m, r in rows.items()},
        **{f"{m}.order": np.array(r["order"]) for m, r in rows.items()},
    )
    print(f"toy zoo: {len(rows)} models")


def corpus():
    rng = np.random.default_rng(20_24)
    models = [toygen.random_model(f"rm{i:03d}", i) for i in range(200)]
    order = rng.permutation(200)
    groups, cur = [], 0
    while cur < 200:
        size = int(rng.integers(1, 8))
        groups.append([int(i) for i in order[cur:cur + size]])
        cur += size
    models_dir = OUT / "models"
    arrays = {}
    for i, (g, w) in enumerate(models):
        model_io.save_graph(g, models_dir / f"rm{i:03d}.graph.json")
        model_io.save_weights(w, models_dir / f"rm{i:03d}.weights.fiwt")
        xs, ys = [], []
        for t in range(4):
            x = input_for(g.input_spec.dims, 7919 * i + t)
            xs.append(x)
            ys.append(np.array(executor.run(g, w, executor.Tensor(g.input_spec, x)).values))
        arrays[f"rm{i:03d}.y"] = np.stack(ys)
        arrays[f"rm{i:03d}.peak"] = np.int64(graph_ir.peak_activation_bytes(g))
        arrays[f"rm{i:03d}.order"] = np.array(json.dumps(graph_ir.topo_order(g)))
    # fused outputs per group (trial 0 inputs), checked equal to solo by the reference
    for gi, grp in enumerate(groups):
        dag = fuse.fuse_models([models[i] for i in grp], validate=False)
        inputs = {models[i][0].model_id: executor.Tensor(models[i][0].input_spec,
                                                         input_for(models[i][0].input_spec.dims, 7919 * i))
                  for i in grp}
        outs = fuse.execute_fused(dag, inputs)
        for i in grp:
            mid = models[i][0].model_id
            assert np.array_equal(outs[mid].values, arrays[f"{mid}.y"][0])
        arrays[f"group{gi}.members"] = np.array(grp)
        arrays[f"group{gi}.mem_mib"] = np.float64(dag.total_mem_estimate_mib)
    arrays["n_groups"] = np.int64(len(groups))
    np.savez_compressed(OUT / "corpus.npz", **arrays)
    kinds = sorted({n.kind for g, _ in models for n in g.nodes.values()})
    print(f"corpus: 200 models, {len(groups)} groups, kinds={kinds}")


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    toy_zoo()
    corpus()
