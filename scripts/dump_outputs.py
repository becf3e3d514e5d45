"""Outputs of the fused 4-model DAG for seeded inputs -> .npz (development A/B helper:
run under different DFX_* knobs, then compare the files)."""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_21120_b200 import zoo  # noqa: E402
from paper_2410_21120_b200.device import DeviceDag  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--precision", default="fp16x2")
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--out", required=True)
a = ap.parse_args()
members = [zoo.build(n) for n in zoo.NORTH_STAR]
dd = DeviceDag(members, 0, "concurrent", precision=a.precision)
inst = dd.acquire(tuple([a.batch] * len(members)))
rng = np.random.default_rng(11)
inst.upload_inputs([rng.standard_normal((a.batch,) + tuple(g.input_spec.dims)).astype(np.float32) for g, _ in members])
inst.launch_graph()
inst.sync()
np.savez(a.out, *inst.download_outputs())
