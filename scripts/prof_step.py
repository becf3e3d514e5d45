"""Load the 4-model fused DAG and run its CUDA graph once (for ncu launch lists)."""
import argparse, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2410_21120_b200 import fuse, zoo
ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--runs", type=int, default=1)
ap.add_argument("--models", nargs="+", default=list(zoo.NORTH_STAR))
a = ap.parse_args()
models = [zoo.build(n) for n in a.models]
dag = fuse.fuse_models(models)
img = fuse.load_fused(dag)
inst = img.acquire(tuple([a.batch] * len(models)))
inst.upload_inputs([np.random.default_rng(i).standard_normal((a.batch, 3, 224, 224)).astype(np.float32)
                    for i in range(len(models))])
for _ in range(a.runs):
    inst.launch_graph()
inst.sync()
print("nodes", inst.kernel_nodes)
