"""Measure the reference cost model's calibration episode on this B200 and write
calibration/b200.cfg (reference format) + calibration/b200_report.json.

Usage: python scripts/calibrate_b200.py [--models 8|4]
"""
import argparse, json, sys, tempfile
from pathlib import Path
sys.path.insert(0, '.')
from paper_2410_21120_b200 import calibration, costmodel, zoo
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--models", type=int, default=8)
a = ap.parse_args()
names = list(zoo.EIGHT_MODEL if a.models == 8 else zoo.NORTH_STAR)
models = bench.build_models(names)
with tempfile.TemporaryDirectory(dir="/tmp") as td:
    ct, rep = calibration.measure(models, td)
out = Path("calibration")
out.mkdir(exist_ok=True)
calibration.dump_cost_table(ct, out / "b200.cfg", header=f"episode: {', '.join(names)} (synthetic calibrated "
                                                          "random-init weights, fp16 device storage)")
# predictions of the calibrated model for the north-star subset vs the episode it came from
class M:  # minimal manifest for the rules
    def __init__(self, w):
        self.weight_bytes = w.byte_size
sub = [M(w) for g, w in models[:4]]
rep["predicted_4model_load_ms"] = {m: calibration.simulate_load(sub, m, ct) for m in costmodel.MODES}
rep["predicted_swap_in_ms"] = {m: calibration.simulate_swap(sub[0], m, ct) for m in costmodel.MODES}
(out / "b200_report.json").write_text(json.dumps(rep, indent=1, default=str) + "\n")
print(open(out / "b200.cfg").read())
print(json.dumps(rep["predicted_4model_load_ms"], indent=1))
