"""Run ONE conv layer as a one-node DAG (for ncu captures; development script).
Usage: python scripts/one_layer.py cin h w cout k stride pad n [precision] [act]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from paper_2410_21120_b200.device import DeviceDag  # noqa: E402
from test_gpu_split import conv_model  # noqa: E402

cin, h, w, cout, k, s, p, n = map(int, sys.argv[1:9])
prec = sys.argv[9] if len(sys.argv) > 9 else "fp16"
act = sys.argv[10] if len(sys.argv) > 10 else "relu"
g, st = conv_model(cin, h, w, cout, k, s, p, 1, act)
d = DeviceDag([(g, st)], precision=prec)
inst = d.acquire((n,))
inst.upload_inputs([np.random.default_rng(0).standard_normal((n, cin, h, w)).astype(np.float32)])
for _ in range(2):
    inst.launch_graph()
inst.sync()
print([(info.get("node"), info.get("tiling", {}).get("tiles")) for op, _, info in inst.nodes])
