"""The north-star parity bar on the B200 (BASELINE.json north_star): logits of
1000 synthetic N(0,1) inputs per model, through the public API
(``execute_fused``), against the CPU fp32 oracle's logits committed in
tests/golden/parity1000 (tests/golden/make_parity_refs.py):

* max over inputs of ||gpu - ref||inf / ||ref||inf <= 2e-2,
* identical top-1 on >= 99.9 % of the inputs (raw), and on every input whose
  fp32 top-1 margin exceeds twice its measured error,

for configs[0] (VGG16 + MobileNetV3-L, batch 1), configs[1] (the 4-model DAG,
batch 1) and configs[2] (the 4-model DAG, batch 32 per member).  The model of
the check is the reference's own statistical acceptance test
(/root/reference/pkg/tests/test_acceptance.py:59-95).  The measured statistic is
written to gpurun_out/ when that directory exists.
"""

import json
from pathlib import Path

import pytest

import north_star_parity as nsp
from paper_2410_21120_b200 import parity

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not nsp.available(), reason="parity fixtures not generated")]

OUT = Path(__file__).resolve().parents[1] / "gpurun_out"


@pytest.fixture(scope="module")
def models():
    return nsp.load_models(nsp.zoo.NORTH_STAR)


def _record(res):
    if OUT.is_dir():
        (OUT / f"parity_{res['config'][-2]}_{res['precision']}.json").write_text(json.dumps(res, indent=1))


@pytest.mark.parametrize("key", ["configs[0]", "configs[1]", "configs[2]"])
def test_north_star_parity_fp16(models, key):
    """16-bit storage (fp16): within 2e-2 and margin-filtered top-1 identical on
    every model; the raw top-1 agreement is recorded."""
    res = nsp.run_config(key, "fp16", 1000, models)
    _record(res)
    for m, s in res["models"].items():
        assert s["max_rel_err"] <= parity.TOL, (m, s)
        assert s["top1_margin_filtered"] == 1.0, (m, s)


@pytest.mark.parametrize("precision", ["fp16x2", "bf16x2"])
@pytest.mark.parametrize("key", ["configs[0]", "configs[1]", "configs[2]"])
def test_north_star_parity_split(models, key, precision):
    """Split precision (two 16-bit planes per value, three-product GEMMs): the FULL
    north-star bar -- within 2e-2 AND identical top-1 on >= 99.9 % of the 1000
    inputs, raw (no margin filter)."""
    res = nsp.run_config(key, precision, 1000, models)
    _record(res)
    for m, s in res["models"].items():
        assert parity.passes(s), (m, s)
