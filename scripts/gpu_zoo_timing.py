"""Quick timing of the 4-model fused DAG (batch 1 and 32) — development script."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2410_21120_b200 import fuse, zoo, runtime as rt
t0 = time.time()
models = [zoo.build(n) for n in zoo.NORTH_STAR]
print(f"build {time.time()-t0:.1f}s", flush=True)
dag = fuse.fuse_models(models)
t0 = time.time()
img = fuse.load_fused(dag)
print(f"lower+pack+upload {time.time()-t0:.1f}s; upload {img.swap_in_ms:.1f} ms for {img.arena.total/1e6:.1f} MB "
      f"= {img.arena.total/img.swap_in_ms/1e6:.1f} GB/s", flush=True)
for B in (1, 32):
    inst = img.acquire(tuple([B]*4))
    xs = [np.random.default_rng(i).standard_normal((B, 3, 224, 224)).astype(np.float32) for i in range(4)]
    inst.upload_inputs(xs)
    print(f"B={B}: graph nodes {inst.kernel_nodes}, act arena {inst.act_bytes/1e6:.1f} MB, ws {inst.ws_bytes/1e6:.1f} MB", flush=True)
    for _ in range(3):
        inst.launch_graph()
    inst.sync()
    e0, e1 = rt.Event(), rt.Event()
    e0.record(inst.stream)
    K = 20
    for _ in range(K):
        inst.launch_graph()
    e1.record(inst.stream)
    ms = e0.elapsed_ms(e1) / K
    print(f"B={B}: {ms:.3f} ms/query, {4*B/ms*1e3:.0f} img/s, {71.3e9*B/(ms*1e-3)/1e12:.1f} TFLOP/s", flush=True)
    img.release(inst)
