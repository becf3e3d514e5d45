"""Generate the north-star parity fixtures: CPU fp32 oracle logits of the four
north-star models on 1000 seeded N(0,1) inputs each (SURVEY.md §7 hard part 2:
">= 1000 inputs are needed for a 99.9 % claim to mean anything").

Test infrastructure (run here, in the build container; the GPU box only reads
the committed .npy files):

    python tests/golden/make_parity_refs.py [--n 1000] [--models ...]

Input i of member m (index in zoo.NORTH_STAR) is
``default_rng(1000*m + i).standard_normal((3, 224, 224), float32)``, the seed
rule of SURVEY.md §8(d).  The oracle is ``oracle.executor_ref.run_fast`` (the
BLAS engine, pinned to the reference executor bitwise on its kinds and to
torchvision fp64 on the extension kinds).  ``meta.json`` records a digest of
every model's weights so a test can prove the GPU box rebuilt identical ones.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
OUT = ROOT / "tests" / "golden" / "parity1000"


def parity_input(member_index: int, i: int, dims=(3, 224, 224)) -> np.ndarray:
    return np.random.default_rng(1000 * member_index + i).standard_normal(dims, dtype=np.float32)


def weights_digest(w) -> str:
    h = hashlib.sha256()
    for name in sorted(w.names()):
        h.update(name.encode())
        h.update(np.ascontiguousarray(w.values(name)).tobytes())
    return h.hexdigest()[:32]


def main():
    from oracle.executor_ref import run_fast
    from paper_2410_21120_b200 import zoo
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1000)
    ap.add_argument("--chunk", type=int, default=25)
    ap.add_argument("--models", nargs="+", default=list(zoo.NORTH_STAR))
    args = ap.parse_args()
    OUT.mkdir(parents=True, exist_ok=True)
    meta_path = OUT / "meta.json"
    meta = json.loads(meta_path.read_text()) if meta_path.exists() else {}
    for name in args.models:
        m = zoo.NORTH_STAR.index(name)
        g, w = zoo.build(name)
        t0 = time.time()
        refs = []
        for c0 in range(0, args.n, args.chunk):
            xs = np.stack([parity_input(m, i, tuple(g.input_spec.dims))
                           for i in range(c0, min(args.n, c0 + args.chunk))])
            refs.append(run_fast(g, w, xs).astype(np.float32))
            print(f"{name}: {c0 + len(xs)}/{args.n} ({time.time() - t0:.0f} s)", flush=True)
        np.save(OUT / f"{name}.npy", np.concatenate(refs))
        meta[name] = {"member_index": m, "n": args.n, "weights_sha256_32": weights_digest(w),
                      "input_rule": "default_rng(1000*member_index + i).standard_normal((3,224,224), float32)",
                      "oracle": "oracle.executor_ref.run_fast (numpy fp32, BLAS)"}
        meta_path.write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
