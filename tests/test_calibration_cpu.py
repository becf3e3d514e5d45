"""Calibration file format (paper_2410_21120_b200/calibration.py): round trip in the
reference's cost-table format, the reference's scaling rules, and (when the
reference is mounted, i.e. in the build container) the reference's own parser
loading our B200 table."""

import importlib.util
import sys
from pathlib import Path

import pytest

from paper_2410_21120_b200 import calibration as cal
from paper_2410_21120_b200.costmodel import FUSED, UNFUSED, estimate_memory


def table():
    costs = {n: cal.FunctionCost(0.7 * (i + 1), 0.1 * (i + 1)) for i, n in enumerate(cal.INIT_FUNCTIONS)}
    costs[cal.MEMCPY_FUNCTION] = cal.FunctionCost(80.0, 11.0)
    return cal.CostTable(context_base_mib=515.0, per_model_overhead_mib=30.5, dedup_saving_mib_per_extra_model=30.5,
                         op_latency_ms_per_mflop={"conv2d": 2.5e-5, "dense": 4e-4}, init_call_costs=costs,
                         calibration_models=8, calibration_weight_bytes=1_000_000_000)


def test_round_trip(tmp_path):
    ct = table()
    cal.dump_cost_table(ct, tmp_path / "b.cfg", header="test")
    back = cal.load_cost_table(tmp_path / "b.cfg")
    assert back.init_call_costs.keys() == ct.init_call_costs.keys()
    for k in ct.init_call_costs:
        assert back.init_call_costs[k].unfused_total_ms == pytest.approx(ct.init_call_costs[k].unfused_total_ms)
        assert back.init_call_costs[k].fused_total_ms == pytest.approx(ct.init_call_costs[k].fused_total_ms)
    assert back.op_latency_ms_per_mflop == ct.op_latency_ms_per_mflop
    assert (back.context_base_mib, back.calibration_models) == (515.0, 8)


def test_scaling_rules():
    ct = table()

    class M:
        weight_bytes = 250_000_000
    one, four = cal.simulate_load([M()], FUSED, ct), cal.simulate_load([M()] * 4, FUSED, ct)
    assert one["memcpy"] == pytest.approx(11.0 / 4) and four["memcpy"] == pytest.approx(11.0)
    assert cal.simulate_load([M()] * 8, UNFUSED, ct)["malloc"] == pytest.approx(ct.init_call_costs["cudaMalloc"].unfused_total_ms)
    assert cal.simulate_swap(M(), FUSED, ct)["total"] < cal.simulate_swap(M(), UNFUSED, ct)["total"]
    assert estimate_memory([], FUSED, ct).peak_mib == 0.0


REF = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted")
def test_reference_parser_loads_our_table(tmp_path):
    sys.path.insert(0, str(REF))
    try:
        from dagfuse import costmodel as refcm
        ct = table()
        cal.dump_cost_table(ct, tmp_path / "b.cfg")
        ref = refcm.load_cost_table(tmp_path / "b.cfg")
        assert ref.calibration_models == 8 and ref.context_base_mib == 515.0
        assert ref.init_call_costs["cudaMemcpyAsync"].fused_total_ms == pytest.approx(11.0)
    finally:
        sys.path.remove(str(REF))
