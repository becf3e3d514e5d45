"""Device-image lifecycle of the drop-in API on the B200.

* ``swap_subgraph`` on a loaded DAG never writes bytes a query of the old DAG
  can read: six threads query the old DAG while the main thread swaps a member
  out (the reference's old DAG is immutable and stays valid,
  /root/reference/pkg/src/dagfuse/fuse.py:233-242; its concurrency contract is
  tests/test_fuse.py:180-205 there).
* ``unload`` returns the instances AND the weight arena; a dropped DAG's image
  is freed by its finalizer; a swap gives the new DAG its own re-packed arena
  (untouched members copied device-to-device), so the old DAG's block -- with
  the outgoing member's bytes -- returns whole when the old DAG is unloaded.
"""

import gc
import threading

import numpy as np
import pytest

from oracle.executor_ref import run_faithful
from paper_2410_21120_b200 import fuse, runtime as rt
from paper_2410_21120_b200.executor import Tensor

pytestmark = pytest.mark.gpu


def _inputs(models, seed):
    rng = np.random.default_rng(seed)
    return {g.model_id: Tensor(g.input_spec, rng.standard_normal(g.input_spec.element_count))
            for g, _ in models}


def test_queries_on_old_dag_during_swap(corpus):
    models = corpus[40:44]
    dag = fuse.fuse_models(models)
    inputs = _inputs(models, 11)
    ref = fuse.execute_fused(dag, inputs)
    stop = threading.Event()
    results, errors = [], []

    def worker():
        try:
            while not stop.is_set():
                results.append(fuse.execute_fused(dag, inputs))
        except Exception as exc:  # noqa: BLE001
            errors.append(exc)

    ts = [threading.Thread(target=worker) for _ in range(6)]
    for t in ts:
        t.start()
    news = []
    cur = dag
    for k, incoming in enumerate(corpus[50:53]):    # three swaps of the same slot
        cur = fuse.swap_subgraph(cur, cur.subgraphs[1].model_id, incoming)
        news.append(cur)
    stop.set()
    for t in ts:
        t.join()
    assert not errors, errors
    assert len(results) >= 6
    for out in results:                              # the old DAG never saw swapped weights
        for mid in ref:
            assert np.array_equal(out[mid].values, ref[mid].values), mid
    last = news[-1]
    inc_g, inc_w = corpus[52]
    inputs2 = {k: v for k, v in inputs.items() if k != models[1][0].model_id}
    inputs2[inc_g.model_id] = Tensor(inc_g.input_spec,
                                     np.random.default_rng(12).standard_normal(inc_g.input_spec.element_count))
    after = fuse.execute_fused(last, inputs2)
    for g, _ in (models[0], models[2], models[3]):
        assert np.array_equal(after[g.model_id].values, ref[g.model_id].values)
    want = run_faithful(inc_g, inc_w, inputs2[inc_g.model_id].values)
    got = after[inc_g.model_id].values
    assert np.abs(got - want).max() <= 2e-2 * np.abs(want).max()
    # the pre-swap DAG is still resident and still right, with no re-upload
    assert fuse.is_loaded(dag)
    again = fuse.execute_fused(dag, inputs)
    for mid in ref:
        assert np.array_equal(again[mid].values, ref[mid].values)
    for d in [dag] + news:
        fuse.unload(d)


def test_unload_returns_arena_and_instances(corpus):
    models = corpus[60:63]
    rt.pool_trim(0)
    gc.collect()
    _, used0 = rt.pool_stats()
    free0, _ = rt.mem_info()
    dag = fuse.fuse_models(models)
    fuse.execute_fused(dag, _inputs(models, 13))
    img = fuse.device_image(dag)
    _, used1 = rt.pool_stats()
    assert used1 - used0 >= img.arena.total
    new = fuse.swap_subgraph(dag, models[0][0].model_id, corpus[64])
    fuse.execute_fused(new, _inputs([(sg, None) for sg in new.subgraphs], 14))
    fuse.unload(dag)
    _, used2 = rt.pool_stats()
    assert used2 > used0                     # new holds its re-packed arena
    del img
    fuse.unload(new)
    gc.collect()
    _, used3 = rt.pool_stats()
    assert used3 == used0
    rt.pool_trim(0)
    free3, _ = rt.mem_info()
    assert free3 >= free0 - (8 << 20)         # instances, staging and arenas all returned


def test_dropped_dag_is_freed(corpus):
    models = corpus[70:72]
    rt.pool_trim(0)
    gc.collect()
    _, used0 = rt.pool_stats()
    dag = fuse.fuse_models(models)
    fuse.execute_fused(dag, _inputs(models, 16))
    _, used1 = rt.pool_stats()
    assert used1 > used0
    del dag
    gc.collect()
    _, used2 = rt.pool_stats()
    assert used2 == used0


def test_swap_repacks_arena_and_cycles(corpus):
    """After a swap and the old DAG's unload, the device holds exactly the post-swap
    arena (the outgoing member's bytes went back with the old block: no dead
    segments pile up over a swap sequence, Table V); the swapped arena
    still cycles through swap-out / swap-in (its host copy read back once)."""
    models = corpus[80:84]
    rt.pool_trim(0)
    gc.collect()
    _, used0 = rt.pool_stats()
    dag = fuse.fuse_models(models)
    fuse.execute_fused(dag, _inputs(models, 21))
    cur = dag
    for k, inc in enumerate(corpus[85:88]):           # three swaps, each old DAG unloaded
        nxt = fuse.swap_subgraph(cur, cur.subgraphs[k].model_id, inc)
        fuse.unload(cur)
        cur = nxt
    ins = _inputs([(sg, None) for sg in cur.subgraphs], 22)
    out1 = fuse.execute_fused(cur, ins)
    img = fuse.device_image(cur)
    gc.collect()
    _, used1 = rt.pool_stats()
    assert img.arena.total <= used1 - used0 <= img.arena.total + (4 << 20)
    img.free_instances()
    img.arena.unload()                                 # swap-out (D2H of the repacked layout)
    img.arena.upload()                                 # swap-in: one allocation + one H2D
    out2 = fuse.execute_fused(cur, ins)
    for mid in out1:
        assert np.array_equal(out1[mid].values, out2[mid].values), mid
    for (g, w) in [(sg, sg.weight_binding) for sg in cur.subgraphs]:
        want = run_faithful(g, w, ins[g.model_id].values)
        assert np.abs(out2[g.model_id].values - want).max() <= 2e-2 * np.abs(want).max()
    fuse.unload(cur)
