"""Per-kind node-time breakdown of the 8-model mixed-batch DAG (development script)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import bench
from paper_2410_21120_b200 import zoo
from paper_2410_21120_b200.device import DeviceDag
names = list(zoo.EIGHT_MODEL)
batches = (1, 2, 4, 8, 1, 2, 4, 8)
m8 = bench.build_models(names)
d = DeviceDag(m8)
inst = d.acquire(batches)
inst.upload_inputs([np.random.default_rng(7 + i).standard_normal((b,) + tuple(g.input_spec.dims)).astype(np.float32)
                    for i, (b, (g, _)) in enumerate(zip(batches, m8))])
prof = inst.profile_nodes(reps=4)
by = {}
for r in prof:
    k = (names[r["member"]] if isinstance(r["member"], int) else r["member"], r["kind"])
    a = by.setdefault(k, [0, 0.0, 0])
    a[0] += 1; a[1] += r["ms"]; a[2] += r["flops"]
for k, (n, ms, fl) in sorted(by.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{k[0]:22s} {k[1]:8s} n={n:4d} {ms:7.3f} ms  {fl / max(ms, 1e-9) / 1e9:7.1f} TF/s")
