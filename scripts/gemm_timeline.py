"""Timeline of one GEMM CTA (block 0) from %globaltimer probes (development script).

Build the debug library first:
  nvcc ... -DDFX_TIMELINE -o /tmp/libdfx_tl.so ...   (see scripts/gpu_timeline.sh)
Usage: DFX_LIBRARY=/tmp/libdfx_tl.so python scripts/gemm_timeline.py --cases cin:cout:hw:n
"""
import argparse
import ctypes as C
import sys

sys.path.insert(0, '.')
import numpy as np

from paper_2410_21120_b200 import graph_ir, runtime as rt
from paper_2410_21120_b200.device import DeviceDag

ap = argparse.ArgumentParser()
ap.add_argument("--cases", default="384:2304:7:1,576:256:56:1,192:768:14:1,2304:384:7:1")
ap.add_argument("--chain", type=int, default=1, help="copies of the node chained in one graph")
ap.add_argument("--global-desc", action="store_true")
a = ap.parse_args()
names = {0: "start", 7: "desc", 8: "mbar", 9: "tmem", 10: "sync", 1: "w-pref", 2: "griddep",
         3: "stage0", 4: "lastMMA", 5: "accum", 11: "epi", 12: "tmem-ld", 6: "stored"}
for case in a.cases.split(","):
    cin, cout, hw, n = map(int, case.split(":"))
    st = graph_ir.WeightStore()
    rng = np.random.default_rng(0)
    st.put("w", graph_ir.TensorSpec((cout, cin, 1, 1)), rng.standard_normal(cout * cin) * 0.05)
    node = graph_ir.OpNode("c", "conv2d", {"out_channels": cout, "kernel": 1}, {"weight": "w"})
    g = graph_ir.ModelGraph("m", [node], "c", "c", graph_ir.TensorSpec((cin, hw, hw)),
                            graph_ir.TensorSpec((cout, hw, hw)))
    d = DeviceDag([(g, st)])
    inst = d.acquire((n,))
    inst.upload_inputs([rng.standard_normal((n, cin, hw, hw)).astype(np.float32)])
    gemm = [(op, p, info) for op, p, info in inst.nodes if op == rt.OP_GEMM][0]
    if a.global_desc:
        gemm[1].flags = 1          # debug: read descriptor + tensor maps from global memory
    graph = rt.Graph()
    last = None
    for _ in range(a.chain):
        last = graph.add(gemm[0], gemm[1], [] if last is None else [last])
    graph.instantiate()
    for _ in range(3):
        graph.launch(inst.stream)
    e0, e1 = rt.Event(), rt.Event()
    e0.record(inst.stream)
    graph.launch(inst.stream)
    e1.record(inst.stream)
    ms = e0.elapsed_ms(e1)
    buf = (C.c_ulonglong * 64)()
    rt.lib().dfx_debug_timeline(buf, 64)
    base = buf[0]
    tl = ", ".join(f"{nm} +{(buf[i] - base) / 1e3:.2f}" for i, nm in names.items())
    stages = gemm[2]['tiling']['sps']
    tl += "\n   stages landed: " + " ".join(f"{(buf[12 + i] - base) / 1e3:.2f}"
                                          for i in range(1, min(stages, 9)))
    tl += "\n   MMAs issued:   " + " ".join(f"{(buf[21 + i] - base) / 1e3:.2f}"
                                          for i in range(0, min(stages, 8)))
    tl += f"\n   A loads issued: {(buf[29] - base) / 1e3:.2f}"
    tl += "\n   B prefetch issued: " + " ".join(f"{(buf[30 + i] - base) / 1e3:.2f}"
                                              for i in range(0, min(stages, 8)))
    tl += "\n   MMA loop cycles (landed->fenced->issued, from stage-0 landing): " + "  ".join(
        f"{buf[42 + 3 * i] - buf[42]}/{buf[43 + 3 * i] - buf[42]}/{buf[44 + 3 * i] - buf[42]}"
        for i in range(0, min(stages, 7)))
    tl += f"\n   SM clock over the CTA: {(buf[41] - buf[40]) / max(buf[6] - buf[0], 1) * 1e3:.0f} MHz"
    print(f"cin={cin} cout={cout} hw={hw} n={n} tiling={gemm[2]['tiling']['tiles']}t/"
          f"{gemm[2]['tiling']['splits']}s/{gemm[2]['tiling']['stages']}st  graph {ms * 1e3 / a.chain:.1f} us/node"
          f"\n   CTA0 (us): {tl}", flush=True)
