"""Single depthwise-conv micro benchmark through the device path (development script)."""
import sys, argparse
sys.path.insert(0, '.')
import numpy as np
from paper_2410_21120_b200 import graph_ir
from paper_2410_21120_b200.device import DeviceDag
ap = argparse.ArgumentParser()
ap.add_argument("--cases", default="1344:14:32:3:1,768:28:32:3:2,384:56:32:3:1,960:7:32:5:1")
a = ap.parse_args()
for case in a.cases.split(","):
    c, hw, n, k, s = map(int, case.split(":"))
    st = graph_ir.WeightStore()
    rng = np.random.default_rng(0)
    st.put("w", graph_ir.TensorSpec((c, 1, k, k)), rng.standard_normal(c * k * k) * 0.1)
    nodes = [graph_ir.OpNode("d", "conv2d", {"out_channels": c, "kernel": k, "stride": s, "padding": k // 2, "groups": c}, {"weight": "w"}),
             graph_ir.OpNode("a", "silu", {}, {}, ("d",))]
    oh = (hw + 2 * (k // 2) - k) // s + 1
    g = graph_ir.ModelGraph("m", nodes, "d", "a", graph_ir.TensorSpec((c, hw, hw)), graph_ir.TensorSpec((c, oh, oh)))
    d = DeviceDag([(g, st)])
    inst = d.acquire((n,))
    inst.upload_inputs([rng.standard_normal((n, c, hw, hw)).astype(np.float32)])
    prof = inst.profile_nodes(reps=8)
    t = [r for r in prof if r["kind"] == "dwconv"][0]
    print(f"c={c} hw={hw} n={n} k={k} s={s}: {t['ms']*1e3:.1f} us {t['bytes']/t['ms']/1e6:.0f} GB/s", flush=True)
