"""Where the e2e overhead over the device time goes (development script)."""
import sys, time, ctypes as C
sys.path.insert(0, '.')
import numpy as np
import bench
from paper_2410_21120_b200 import fuse, zoo, runtime as rt
from paper_2410_21120_b200.executor import Tensor

models = bench.build_models(list(zoo.NORTH_STAR))
dag = fuse.fuse_models(models)
img = fuse.load_fused(dag, precision=sys.argv[1] if len(sys.argv) > 1 else "fp16x2")
xs = {g.model_id: Tensor(g.input_spec, np.random.default_rng(i).standard_normal((3, 224, 224)).astype(np.float32))
      for i, (g, _) in enumerate(models)}
for _ in range(20):
    fuse.execute_fused(dag, xs)
inst = img.acquire((1, 1, 1, 1))
arrs = [xs[g.model_id].values for g, _ in models]
srcs = (C.c_void_p * 4)(*[a.ctypes.data for a in arrs])
sizes = (C.c_size_t * 4)(*[a.nbytes for a in arrs])
K = 300


def t(fn):
    for _ in range(10):
        fn()
    t0 = time.perf_counter()
    for _ in range(K):
        fn()
    return (time.perf_counter() - t0) / K * 1e6


print("execute_fused        %.1f us" % t(lambda: fuse.execute_fused(dag, xs)))
print("inst.run             %.1f us" % t(lambda: inst.run([[a] for a in arrs])))
print("execute_gather (C)   %.1f us" % t(lambda: inst.graph.execute_gather(srcs, sizes, inst.host_in, inst.dev_in, inst.host_out, inst.dev_out, inst.out_bytes, inst.stream)))
print("execute (C, staged)  %.1f us" % t(lambda: inst.graph.execute(inst.host_in, inst.dev_in, inst.in_bytes, inst.host_out, inst.dev_out, inst.out_bytes, inst.stream)))
print("launch+sync          %.1f us" % t(lambda: (inst.launch_graph(), inst.sync())))
print("read_outputs         %.1f us" % t(lambda: inst.read_outputs()))
