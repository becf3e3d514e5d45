"""Timeline of one squeeze-excitation cluster kernel (CTA 0 of image 0); development script.
Usage: DFX_LIBRARY=/tmp/libdfx_tl.so python scripts/se_timeline.py --cases C:Cr:hw:n,...
"""
import argparse
import ctypes as C
import sys

sys.path.insert(0, '.')
import numpy as np

from paper_2410_21120_b200 import graph_ir, runtime as rt
from paper_2410_21120_b200.device import DeviceDag

ap = argparse.ArgumentParser()
ap.add_argument("--cases", default="1344:56:14:1,2304:96:7:1,3840:160:7:1,960:240:7:1,1344:56:14:32")
ap.add_argument("--precision", default="fp16")
a = ap.parse_args()
names = {0: "start", 1: "griddep", 2: "pooled", 3: "weights", 4: "fc1", 5: "cluster.sync",
         6: "hidden", 7: "gate+scale", 8: "final sync"}
O, S = graph_ir.OpNode, graph_ir.TensorSpec
for case in a.cases.split(","):
    c, cr, hw, n = map(int, case.split(":"))
    rng = np.random.default_rng(0)
    st = graph_ir.WeightStore()
    st.put("f1", S((cr, c)), rng.standard_normal(cr * c) * 0.05)
    st.put("f2", S((c, cr)), rng.standard_normal(cr * c) * 0.05)
    nodes = [O("a", "relu"), O("b", "global_avg_pool", inputs=("a",)),
             O("c", "dense", {"units": cr, "fan_in": c}, {"weight": "f1"}, ("b",)),
             O("d", "silu", inputs=("c",)),
             O("e", "dense", {"units": c, "fan_in": cr}, {"weight": "f2"}, ("d",)),
             O("f", "sigmoid", inputs=("e",)), O("g", "channel_scale", inputs=("a", "f"))]
    g = graph_ir.ModelGraph("m", nodes, "a", "g", S((c, hw, hw)), S((c, hw, hw)))
    d = DeviceDag([(g, st)], precision=a.precision)
    inst = d.acquire((n,))
    inst.upload_inputs([rng.standard_normal((n, c, hw, hw)).astype(np.float32)])
    se = [(op, p) for op, p, info in inst.nodes if op == rt.OP_SE][0]
    graph = rt.Graph()
    graph.add(se[0], se[1])
    graph.instantiate()
    for _ in range(3):
        graph.launch(inst.stream)
    e0, e1 = rt.Event(), rt.Event()
    e0.record(inst.stream)
    graph.launch(inst.stream)
    e1.record(inst.stream)
    ms = e0.elapsed_ms(e1)
    buf = (C.c_ulonglong * 64)()
    rt.lib().dfx_debug_timeline_se(buf, 64)
    base = buf[0]
    print(f"{a.precision} C={c} Cr={cr} hw={hw} n={n}: graph {ms * 1e3:.1f} us; CTA0: " +
          ", ".join(f"{nm} +{(buf[i] - base) / 1e3:.2f}" for i, nm in names.items()), flush=True)
