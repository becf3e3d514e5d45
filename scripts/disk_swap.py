"""Swap-in from disk: FIWT path vs packed-arena file (development script)."""
import json, sys, argparse
sys.path.insert(0, '.')
import bench
from paper_2410_21120_b200 import fuse, zoo, runtime as rt
rt.init_device(0)
models = bench.build_models(list(zoo.NORTH_STAR))
dag = fuse.fuse_models(models)
members = [(sg, sg.weight_binding) for sg in dag.subgraphs]
args = argparse.Namespace(precision="fp16")
for _ in range(2):
    print(json.dumps(bench.swap_from_disk(args, members)))
