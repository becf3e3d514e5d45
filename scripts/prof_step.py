"""Load the fused DAG and run its CUDA graph once (for ncu launch lists).

--algo prints the mean algorithmic bytes / FLOPs per GEMM launch of the step
(the per-launch figure the bench's roofline uses), for summarize_profiles.py traffic.
"""
import argparse, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2410_21120_b200 import fuse, zoo, runtime as rt
ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--runs", type=int, default=1)
ap.add_argument("--models", nargs="+", default=list(zoo.NORTH_STAR))
ap.add_argument("--algo", action="store_true")
ap.add_argument("--precision", default="fp16x2")
a = ap.parse_args()
models = [zoo.build(n) for n in a.models]
dag = fuse.fuse_models(models)
img = fuse.load_fused(dag, precision=a.precision)
inst = img.acquire(tuple([a.batch] * len(models)))
inst.upload_inputs([np.random.default_rng(i).standard_normal((a.batch,) + tuple(g.input_spec.dims))
                    .astype(np.float32) for i, (g, _) in enumerate(models)])
if a.algo:
    gem = [info for op, _, info in inst.nodes if op == rt.OP_GEMM]
    print(sum(i["bytes"] for i in gem) / len(gem))
    sys.exit(0)
for _ in range(a.runs):
    inst.launch_graph()
inst.sync()
print("nodes", inst.kernel_nodes)
