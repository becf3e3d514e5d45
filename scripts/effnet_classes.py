"""EfficientNetV2-L batch 1 alone: per-class node time sums (profile_nodes) for one
precision (development script; knobs via DFX_* env)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_21120_b200 import zoo  # noqa: E402
from paper_2410_21120_b200.device import DeviceDag  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp16x2"
tag = sys.argv[2] if len(sys.argv) > 2 else ""
g, w = zoo.build("efficientnet_v2_l")
d = DeviceDag([(g, w)], precision=prec)
inst = d.acquire((1,))
inst.upload_inputs([np.random.default_rng(0).standard_normal((1, 3, 224, 224)).astype(np.float32)])
prof = inst.profile_nodes(reps=8)
cls = {}
for r in prof:
    k = r["kind"]
    if k == "gemm":
        k = "gemm+dw" if r["tiling"].get("dw") is not None else ("gemm-splitk" if r["split"] or r["tiling"]["splits"] > 1 else "gemm")
    c = cls.setdefault(k, [0, 0.0])
    c[0] += 1
    c[1] += r["ms"] * 1e3
print(f"{tag:20s} {prec:7s} total {sum(v[1] for v in cls.values()):8.1f} us  " +
      "  ".join(f"{k} {n}x{us / n:.1f}={us:.0f}" for k, (n, us) in sorted(cls.items())), flush=True)
