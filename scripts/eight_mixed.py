"""8-model mixed-batch step time (configs[4]) for A/B runs (development script)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import bench
from paper_2410_21120_b200 import zoo, runtime as rt
from paper_2410_21120_b200.device import DeviceDag
names = list(zoo.EIGHT_MODEL)
batches = (1, 2, 4, 8, 1, 2, 4, 8)
m8 = bench.build_models(names)
d = DeviceDag(m8)
inst = d.acquire(batches)
inst.upload_inputs([np.random.default_rng(7 + i).standard_normal((b,) + tuple(g.input_spec.dims)).astype(np.float32)
                    for i, (b, (g, _)) in enumerate(zip(batches, m8))])
flush = rt.malloc(256 << 20)
med, _ = bench.time_device_steps(rt, inst, flush, steps=20)
print(f"eight mixed: {med:.3f} ms  nodes {inst.kernel_nodes}")
