"""Per-member graph time at batch B (each member alone) vs the fused DAG (development script)."""
import sys, argparse
sys.path.insert(0, '.')
import numpy as np
from paper_2410_21120_b200 import zoo, runtime as rt
from paper_2410_21120_b200.device import DeviceDag
ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--set", choices=("north", "eight"), default="north")
ap.add_argument("--precision", default="fp16x2")
a = ap.parse_args()
names = zoo.NORTH_STAR if a.set == "north" else zoo.EIGHT_MODEL
models = [zoo.build(n) for n in names]


def timeit(dag, batch, K=30):
    inst = dag.acquire(batch)
    inst.upload_inputs([np.random.default_rng(0).standard_normal((b,) + tuple(g.input_spec.dims)).astype(np.float32)
                        for b, (g, _) in zip(batch, dag.members)])
    for _ in range(3): inst.launch_graph()
    inst.sync(); e0, e1 = rt.Event(), rt.Event(); e0.record(inst.stream)
    for _ in range(K): inst.launch_graph()
    e1.record(inst.stream); return e0.elapsed_ms(e1) / K, inst.kernel_nodes


for (g, w), name in zip(models, names):
    d = DeviceDag([(g, w)], precision=a.precision)
    ms, nodes = timeit(d, (a.batch,))
    print(f"{name:22s} alone: {ms:7.3f} ms  nodes {nodes:5d}  {ms / nodes * 1e3:6.2f} us/node", flush=True)
d = DeviceDag(models, precision=a.precision)
ms, nodes = timeit(d, tuple([a.batch] * len(models)))
print(f"{'fused (concurrent)':22s}      {ms:7.3f} ms  nodes {nodes:5d}")
d = DeviceDag(models, mode="sequential", precision=a.precision)
ms, nodes = timeit(d, tuple([a.batch] * len(models)))
print(f"{'fused (sequential)':22s}      {ms:7.3f} ms  nodes {nodes:5d}")
