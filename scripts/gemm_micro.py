"""Single-conv micro benchmark through the device path (development script)."""
import sys, argparse
sys.path.insert(0, '.')
import numpy as np
from paper_2410_21120_b200 import graph_ir
from paper_2410_21120_b200.device import DeviceDag
ap = argparse.ArgumentParser()
ap.add_argument("--cases", default="96:48:28:1,96:96:28:1,96:128:28:1,96:144:28:1,96:192:28:1,96:256:28:1,160:960:7:1,96:384:28:32")
ap.add_argument("--act", default="")
a = ap.parse_args()
for case in a.cases.split(","):
    f = list(map(int, case.split(":")))
    cin, cout, hw, n = f[:4]
    k = f[4] if len(f) > 4 else 1
    act = a.act
    st = graph_ir.WeightStore()
    rng = np.random.default_rng(0)
    st.put("w", graph_ir.TensorSpec((cout, cin, k, k)), rng.standard_normal(cout * cin * k * k) * 0.1)
    node = graph_ir.OpNode("c", "conv2d", {"out_channels": cout, "kernel": k, "padding": k // 2}, {"weight": "w"})
    nodes, exit_id = [node], "c"
    if act:
        nodes.append(graph_ir.OpNode("a", act, {}, {}, ("c",)))
        exit_id = "a"
    g = graph_ir.ModelGraph("m", nodes, "c", exit_id, graph_ir.TensorSpec((cin, hw, hw)), graph_ir.TensorSpec((cout, hw, hw)))
    d = DeviceDag([(g, st)])
    inst = d.acquire((n,))
    inst.upload_inputs([rng.standard_normal((n, cin, hw, hw)).astype(np.float32)])
    prof = inst.profile_nodes(reps=8)
    t = [r for r in prof if r["kind"] == "gemm"][0]
    print(f"cin={cin} cout={cout} hw={hw} n={n} tiling={ {k: t['tiling'][k] for k in ('tiles','splits','stages','bn','tn','tp','tq')} } {t['ms']*1e3:.1f} us {t['flops']/t['ms']/1e9:.1f} TF/s", flush=True)
