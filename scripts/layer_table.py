"""Per-GEMM-launch timing table of the fused DAG (development script).

Usage: python scripts/layer_table.py --batch 1 [--top 40]
"""
import argparse
import json
import sys

sys.path.insert(0, '.')
import numpy as np

from paper_2410_21120_b200 import fuse, zoo

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--models", nargs="+", default=list(zoo.NORTH_STAR))
ap.add_argument("--json", default=None)
ap.add_argument("--precision", default="fp16")
a = ap.parse_args()
models = [zoo.build(n) for n in a.models]
dag = fuse.fuse_models(models)
img = fuse.load_fused(dag, precision=a.precision)
inst = img.acquire(tuple([a.batch] * len(models)))
inst.upload_inputs([np.random.default_rng(i).standard_normal((a.batch, 3, 224, 224)).astype(np.float32)
                    for i in range(len(models))])
prof = inst.profile_nodes(reps=8)
tot = sum(r["ms"] for r in prof)
by = {}
for r in prof:
    by.setdefault(r["kind"], [0, 0.0])
    by[r["kind"]][0] += 1
    by[r["kind"]][1] += r["ms"]
print(f"batch {a.batch}: sum of node times {tot:.3f} ms")
for k, (n, ms) in sorted(by.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:8s} n={n:4d} {ms:8.3f} ms  avg {ms / n * 1e3:7.2f} us")
g = [r for r in prof if r["kind"] == "gemm"]
g.sort(key=lambda r: -r["ms"])
print(f"{'member':20s} {'node':24s} {'M':>7s} {'N':>5s} {'K':>6s} {'cb':>3s} {'tiles':>6s} {'spl':>4s} "
      f"{'stg':>4s} {'us':>8s} {'GB/s':>7s} {'TF/s':>7s}")
for r in g[:a.top]:
    t, ge = r["tiling"], r["geom"]
    M = r["flops"] // 2 // (ge["cout"] * ge["cin"] * ge["kh"] * ge["kw"])
    print(f"{r['member']:20s} {r['node'][:24]:24s} {M:7d} {ge['cout']:5d} {ge['cin'] * ge['kh'] * ge['kw']:6d} "
          f"{ge['cb']:3d} {t['tiles']:6d} {t['splits']:4d} {t['stages']:4d} {r['ms'] * 1e3:8.1f} "
          f"{r['bytes'] / r['ms'] / 1e6:7.0f} {r['flops'] / r['ms'] / 1e9:7.1f}")
if a.json:
    json.dump(prof, open(a.json, "w"), default=str)
