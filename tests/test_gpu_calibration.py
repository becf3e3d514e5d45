"""Cost-model recalibration on the GPU: the reference's
calibration episode (/root/reference/pkg/src/dagfuse/costmodel.py:391-474 format,
calibrate.py's measured phases) re-measured on this B200 with two members, and the
committed calibration/b200.cfg checked against the fresh measurement."""

from pathlib import Path

import pytest

from paper_2410_21120_b200 import calibration, costmodel, zoo

pytestmark = pytest.mark.gpu

CFG = Path(__file__).resolve().parents[1] / "calibration" / "b200.cfg"


class _Manifest:
    def __init__(self, w):
        self.weight_bytes = w.byte_size


@pytest.fixture(scope="module")
def episode(tmp_path_factory):
    models = [zoo.build("resnet50"), zoo.build("mobilenet_v3_large")]
    ct, rep = calibration.measure(models, tmp_path_factory.mktemp("cal"))
    return models, ct, rep


def test_episode_table_round_trips(episode, tmp_path):
    _, ct, _ = episode
    p = tmp_path / "b200.cfg"
    calibration.dump_cost_table(ct, p, header="test episode")
    back = calibration.load_cost_table(p)
    assert back.calibration_models == 2
    assert back.function_names == ct.function_names
    for name in ct.function_names:
        a, b = ct.init_call_costs[name], back.init_call_costs[name]
        assert b.unfused_total_ms == pytest.approx(a.unfused_total_ms, rel=1e-3, abs=1e-6)
        assert b.fused_total_ms == pytest.approx(a.fused_total_ms, rel=1e-3, abs=1e-6)


def test_episode_measures_fusion_savings(episode):
    """One arena beats per-tensor allocation and copies; the packed header beats
    parse + lower; the per-kind op latencies exist for the kinds that ran."""
    _, ct, rep = episode
    c = ct.init_call_costs
    assert c[calibration.MALLOC_FUNCTION].fused_total_ms < c[calibration.MALLOC_FUNCTION].unfused_total_ms
    assert c[calibration.MEMCPY_FUNCTION].fused_total_ms < c[calibration.MEMCPY_FUNCTION].unfused_total_ms
    assert c[calibration.SCHEMA_FUNCTION].fused_total_ms < c[calibration.SCHEMA_FUNCTION].unfused_total_ms
    assert ct.context_base_mib > 0 and ct.per_model_overhead_mib >= 0
    assert "conv2d" in ct.op_latency_ms_per_mflop and ct.op_latency_ms_per_mflop["conv2d"] > 0
    # the fused H2D of the packed arena runs at a pinned-copy rate (> 10 GB/s)
    fused_ms = sorted(t[1] for t in rep["fused_malloc_memcpy_ms"])[1]
    arena_bytes = rep["weight_bytes"] / 2          # fp16 device storage of fp32 weights
    assert arena_bytes / (fused_ms * 1e-3) > 10e9


def test_committed_table_predicts_this_box(episode):
    """calibration/b200.cfg (8-model episode, committed) predicts this 2-model
    episode's fused copy time within 2x, and the fresh table reproduces its own
    episode through simulate_load exactly."""
    models, ct, rep = episode
    committed = calibration.load_cost_table(CFG)
    manifests = [_Manifest(w) for _, w in models]
    wb = sum(m.weight_bytes for m in manifests)
    measured = ct.init_call_costs[calibration.MEMCPY_FUNCTION].fused_total_ms
    predicted = committed.memcpy_ms(wb, costmodel.FUSED)
    assert measured / 2 <= predicted <= measured * 2, (predicted, measured)
    sim = calibration.simulate_load(manifests, costmodel.FUSED, ct)
    assert sim["memcpy"] == pytest.approx(measured, rel=1e-9)
    assert sim["malloc"] == pytest.approx(ct.init_call_costs[calibration.MALLOC_FUNCTION].fused_total_ms, rel=1e-9)
