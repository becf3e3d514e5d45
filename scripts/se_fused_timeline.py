"""Phase timeline of a GEMM with the fused depthwise + SE epilogue (block 0, %globaltimer
probes 5 and 48-57; development script).  One MBConv middle at 7x7 / 14x14, batch 1.
Build the probe library first (DFX_TIMELINE) and point DFX_LIBRARY at it."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_21120_b200 import graph_ir, runtime as rt  # noqa: E402
from paper_2410_21120_b200.device import DeviceDag  # noqa: E402

NAMES = {0: "start", 2: "griddep", 3: "stage0", 4: "lastMMA", 5: "accum", 48: "dw-drain", 50: "dw-done", 51: "means", 52: "fc1-part", 53: "barrier",
         54: "gather", 55: "hidden", 56: "gates", 57: "stored"}


def mbconv(cin, cexp, hw, cr, prec):
    rng = np.random.default_rng(0)
    st = graph_ir.WeightStore()
    for k, shp in {"e": (cexp, cin, 1, 1), "d": (cexp, 1, 3, 3), "f1": (cr, cexp), "f2": (cexp, cr),
                   "p": (cin, cexp, 1, 1)}.items():
        st.put(k, graph_ir.TensorSpec(shp), rng.standard_normal(int(np.prod(shp))) * 0.1)
    O = graph_ir.OpNode
    nodes = [O("e", "conv2d", {"out_channels": cexp, "kernel": 1}, {"weight": "e"}),
             O("ea", "silu", inputs=("e",)),
             O("d", "conv2d", {"out_channels": cexp, "kernel": 3, "stride": 1, "padding": 1, "groups": cexp},
               {"weight": "d"}, ("ea",)),
             O("da", "silu", inputs=("d",)),
             O("g", "global_avg_pool", inputs=("da",)),
             O("f1", "dense", {"units": cr, "fan_in": cexp}, {"weight": "f1"}, ("g",)),
             O("f1a", "silu", inputs=("f1",)),
             O("f2", "dense", {"units": cexp, "fan_in": cr}, {"weight": "f2"}, ("f1a",)),
             O("f2a", "sigmoid", inputs=("f2",)),
             O("s", "channel_scale", inputs=("da", "f2a"))]
    return graph_ir.ModelGraph("mb", nodes, "e", "s", graph_ir.TensorSpec((cin, hw, hw)),
                               graph_ir.TensorSpec((cexp, hw, hw))), st


for prec in ("fp16", "fp16x2"):
    for cin, cexp, hw, cr in ((384, 2304, 7, 96), (640, 3840, 7, 160), (224, 1344, 14, 56)):
        g, w = mbconv(cin, cexp, hw, cr, prec)
        d = DeviceDag([(g, w)], precision=prec)
        inst = d.acquire((1,))
        inst.upload_inputs([np.random.default_rng(1).standard_normal((1, cin, hw, hw)).astype(np.float32)])
        nodes = [(op, info.get("tiling", {})) for op, _, info in inst.nodes]
        fused = [t for op, t in nodes if op == rt.OP_GEMM and t.get("se") is not None]
        for _ in range(3):
            inst.launch_graph()
        inst.sync()
        buf = (C.c_ulonglong * 64)()
        rt.lib().dfx_debug_timeline(buf, 64)
        t0 = buf[0]
        line = "  ".join(f"{NAMES[i]} {(buf[i] - t0) / 1e3:+.2f}" for i in (2, 3, 4, 5, 48, 50, 51, 52, 53, 54, 55, 56, 57))
        prof = inst.profile_nodes(reps=8)
        line += "  | node us: " + " ".join(f"{r['kind']}={r['ms'] * 1e3:.1f}" for r in prof)
        tl = fused[0] if fused else {}
        print(f"{prec:7s} {cin}->{cexp} {hw}x{hw} cr {cr}: tiles {tl.get('tiles')} bn {tl.get('bn')} "
              f"nslots {tl.get('nslots')} | {line}", flush=True)
        d.free()
