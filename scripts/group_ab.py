"""A/B of the grouped cross-member GEMM (device.GROUP_GEMM) on the B200:
configs[4] (8-model DAG, mixed batches), the 4-model DAG at batch 1, and
ResNet-50 + ResNet-152 alone (the pair with the most shared layer shapes).
Device-timed steps (CUDA events, L2 flushed between steps), median of 50."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2410_21120_b200 import device, runtime as rt, zoo  # noqa: E402
from paper_2410_21120_b200.device import DeviceDag  # noqa: E402


def timed(members, batch, group, steps=50):
    device.GROUP_GEMM = group
    dd = DeviceDag(members, 0, "concurrent")
    inst = dd.acquire(batch)
    rng = np.random.default_rng(1)
    inst.upload_inputs([rng.standard_normal((b,) + tuple(g.input_spec.dims)).astype(np.float32)
                        for b, (g, _) in zip(batch, members)])
    flush = rt.malloc(256 << 20)
    for _ in range(5):
        inst.launch_graph()
    inst.sync()
    ms = []
    for _ in range(steps):
        rt.memset(flush, 0, 256 << 20, inst.stream)
        e0, e1 = rt.Event(), rt.Event()
        e0.record(inst.stream)
        inst.launch_graph()
        e1.record(inst.stream)
        ms.append(e0.elapsed_ms(e1))
    inst.sync()
    out = dict(ms=float(np.median(ms)), nodes=inst.kernel_nodes, grouped=inst.grouped_launches)
    rt.free(flush)
    dd.release(inst)
    dd.free()
    return out


def main():
    rt.init_device(0)
    built = {n: zoo.build(n) for n in zoo.EIGHT_MODEL}
    cases = [("configs[4] 8-model mixed batch", list(zoo.EIGHT_MODEL), (1, 2, 4, 8, 1, 2, 4, 8)),
             ("4-model batch 1", list(zoo.NORTH_STAR), (1, 1, 1, 1)),
             ("resnet50 + resnet152 batch 1", ["resnet50", "resnet152"], (1, 1)),
             ("resnet50 + resnet152 batch 8", ["resnet50", "resnet152"], (8, 8))]
    res = {}
    for name, names, batch in cases:
        members = [built[n] for n in names]
        res[name] = {"off": timed(members, batch, False), "on": timed(members, batch, True)}
        print(name, res[name], flush=True)
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "group_ab.json").write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
