"""EfficientNetV2-L batch 1: isolated node times of expand GEMM (+ depthwise) with and
without the depthwise epilogue (development script)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2410_21120_b200 import zoo, device
from paper_2410_21120_b200.device import DeviceDag

g, w = zoo.build("efficientnet_v2_l")
x = np.random.default_rng(0).standard_normal((1, 3, 224, 224)).astype(np.float32)
res = {}
for on in (False, True):
    device.GEMM_DW = on
    d = DeviceDag([(g, w)])
    inst = d.acquire((1,))
    inst.upload_inputs([x])
    prof = inst.profile_nodes(reps=8)
    res[on] = prof
    d.free_instances()
off = res[False]
on = res[True]
# pair: unfused gemm followed by dwconv  vs fused gemm with the same node id
by_node_on = {r["node"]: r for r in on if r["kind"] == "gemm"}
tot_a = tot_b = 0.0
for i, r in enumerate(off[:-1]):
    if r["kind"] == "gemm" and off[i + 1]["kind"] == "dwconv" and r["node"] in by_node_on:
        f = by_node_on[r["node"]]
        if f["tiling"].get("dw") is None:
            continue
        a = (r["ms"] + off[i + 1]["ms"]) * 1e3
        b = f["ms"] * 1e3
        tot_a += a; tot_b += b
        t0, t1 = r["tiling"], f["tiling"]
        print(f"{r['node'][:28]:28s} gemm {r['ms']*1e3:6.2f} + dw {off[i+1]['ms']*1e3:6.2f} = {a:6.2f} us"
              f" | fused {b:6.2f} us  (tiles {t0['tiles']} bn {t0['bn']} spl {t0['splits']} -> tiles {t1['tiles']} bn {t1['bn']} m2 {t1['m2']})")
print(f"total two-launch {tot_a:.1f} us, fused {tot_b:.1f} us")
