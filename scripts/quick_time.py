"""Device-timed step of the fused 4-model DAG (development A/B helper; knobs via DFX_* env).
Usage: python scripts/quick_time.py --precision fp16x2 --batch 1 [--member efficientnet_v2_l]"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_21120_b200 import runtime as rt, zoo  # noqa: E402
from paper_2410_21120_b200.device import DeviceDag  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--precision", default="fp16x2")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--steps", type=int, default=60)
ap.add_argument("--models", nargs="+", default=list(zoo.NORTH_STAR))
ap.add_argument("--tag", default="")
a = ap.parse_args()
rt.init_device(0)
members = [zoo.build(n) for n in a.models]
dd = DeviceDag(members, 0, "concurrent", precision=a.precision)
batch = tuple([a.batch] * len(members))
inst = dd.acquire(batch)
rng = np.random.default_rng(0)
inst.upload_inputs([rng.standard_normal((a.batch,) + tuple(g.input_spec.dims)).astype(np.float32) for g, _ in members])
flush = rt.malloc(256 << 20)
for _ in range(5):
    inst.launch_graph()
inst.sync()
ms = []
for _ in range(a.steps):
    rt.memset(flush, 0, 256 << 20, inst.stream)
    e0, e1 = rt.Event(), rt.Event()
    e0.record(inst.stream)
    inst.launch_graph()
    e1.record(inst.stream)
    ms.append(e0.elapsed_ms(e1))
inst.sync()
print(f"{a.tag:30s} {a.precision} b{a.batch} {'+'.join(m[:6] for m in a.models)}: median {np.median(ms):.3f} ms "
      f"min {np.min(ms):.3f} nodes {inst.kernel_nodes}", flush=True)
