"""North-star parity runs on the GPU against the committed CPU fp32 fixtures
(tests/golden/parity1000, written by tests/golden/make_parity_refs.py).

configs[0]: VGG16 + MobileNetV3-L fused, batch 1, 1000 queries.
configs[1]: the 4-model fused DAG, batch 1, 1000 queries.
configs[2]: the 4-model fused DAG, batch 32 per member (1000 inputs = 31 x 32 + 8).
Every query goes through the public API (``fuse.execute_fused`` with host
Tensors).  Shared by tests/test_gpu_north_star.py and bench.py's ``parity``
block; test infrastructure only.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))

from make_parity_refs import OUT as FIXTURES, parity_input, weights_digest  # noqa: E402
from paper_2410_21120_b200 import fuse, parity, zoo  # noqa: E402
from paper_2410_21120_b200.executor import Tensor  # noqa: E402

CONFIGS = {
    "configs[0]": (("vgg16", "mobilenet_v3_large"), 1),
    "configs[1]": (zoo.NORTH_STAR, 1),
    "configs[2]": (zoo.NORTH_STAR, 32),
}


def available() -> bool:
    return (FIXTURES / "meta.json").exists() and all((FIXTURES / f"{m}.npy").exists() for m in zoo.NORTH_STAR)


def load_models(names):
    meta = json.loads((FIXTURES / "meta.json").read_text())
    out = {}
    for name in names:
        g, w = zoo.build(name)
        if weights_digest(w) != meta[name]["weights_sha256_32"]:
            raise AssertionError(f"{name}: weights differ from the ones the fixtures were made with")
        out[name] = (g, w)
    return out


def run_config(key: str, precision: str = "fp16", n: int = 1000, models=None) -> dict:
    names, batch = CONFIGS[key]
    models = models or load_models(names)
    members = [models[m] for m in names]
    dag = fuse.fuse_models(members)
    fuse.load_fused(dag, precision=precision)
    got = {m: [] for m in names}
    t0 = time.perf_counter()
    for q0 in range(0, n, batch):
        rows = range(q0, min(n, q0 + batch))
        inputs = {}
        for m in names:
            g = models[m][0]
            mi = zoo.NORTH_STAR.index(m)
            ts = [Tensor(g.input_spec, parity_input(mi, i, tuple(g.input_spec.dims)).reshape(-1)) for i in rows]
            inputs[g.model_id] = ts if batch > 1 else ts[0]
        outs = fuse.execute_fused(dag, inputs)
        for m in names:
            o = outs[models[m][0].model_id]
            got[m].extend([t.values for t in o] if batch > 1 else [o.values])
    wall = time.perf_counter() - t0
    fuse.unload(dag)
    res = {"config": key, "precision": precision, "batch_per_member": batch, "inputs_per_model": n,
           "wall_s": round(wall, 2), "models": {}}
    for m in names:
        ref = np.load(FIXTURES / f"{m}.npy", mmap_mode="r")[:n]
        res["models"][m] = parity.stats(np.stack(got[m]), ref)
    res["pass"] = all(parity.passes(s) for s in res["models"].values())
    return res


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", nargs="+", default=["fp16", "bf16"])
    ap.add_argument("--configs", nargs="+", default=list(CONFIGS))
    ap.add_argument("--n", type=int, default=1000)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    allm = load_models(zoo.NORTH_STAR)
    results = [run_config(k, p, a.n, allm) for p in a.precision for k in a.configs]
    txt = json.dumps(results, indent=1)
    print(txt)
    if a.out:
        Path(a.out).write_text(txt + "\n")
