"""Single-conv micro benchmark through the device path (development script)."""
import sys, argparse
sys.path.insert(0, '.')
import numpy as np
from paper_2410_21120_b200 import graph_ir
from paper_2410_21120_b200.device import DeviceDag
ap = argparse.ArgumentParser()
ap.add_argument("--cases", default="96:48:28:1,96:96:28:1,96:128:28:1,96:144:28:1,96:192:28:1,96:256:28:1,160:960:7:1,96:384:28:32")
a = ap.parse_args()
for case in a.cases.split(","):
    cin, cout, hw, n = map(int, case.split(":"))
    st = graph_ir.WeightStore()
    rng = np.random.default_rng(0)
    st.put("w", graph_ir.TensorSpec((cout, cin, 1, 1)), rng.standard_normal(cout * cin) * 0.1)
    node = graph_ir.OpNode("c", "conv2d", {"out_channels": cout, "kernel": 1}, {"weight": "w"})
    g = graph_ir.ModelGraph("m", [node], "c", "c", graph_ir.TensorSpec((cin, hw, hw)), graph_ir.TensorSpec((cout, hw, hw)))
    d = DeviceDag([(g, st)])
    inst = d.acquire((n,))
    inst.upload_inputs([rng.standard_normal((n, cin, hw, hw)).astype(np.float32)])
    prof = inst.profile_nodes(reps=8)
    t = [r for r in prof if r["kind"] == "gemm"][0]
    print(f"cin={cin} cout={cout} hw={hw} n={n} tiling={ {k: t['tiling'][k] for k in ('tiles','splits','stages','bn','tn','tp','tq')} } {t['ms']*1e3:.1f} us", flush=True)
