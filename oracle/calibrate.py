#!/usr/bin/env python3
"""Data-calibrated init statistics for the zoo models — test infrastructure.

One forward pass of the fast oracle engine over a synthetic N(0,1) batch with
a hook that, in topological order,
  * at every batchnorm node records the per-channel mean/variance of its
    input (variance clamped from below at the layer's median, SURVEY.md §7
    hard part 2) and normalises with those statistics;
  * at every conv2d/dense node NOT followed by a batchnorm applies LSUV:
    rescales weights+bias so the output has unit standard deviation.
The resulting dict is saved to paper_2410_21120_b200/zoo/calib/<model>.npz and
applied by ``zoo.build`` when generating weights (no forward pass needed
there, so every machine regenerates bit-identical weights).

Usage:  python oracle/calibrate.py [model ...]     (default: all zoo models)
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.executor_ref import bn_coeffs, eval_node_fast, run_fast  # noqa: E402
from paper_2410_21120_b200 import zoo  # noqa: E402


LSUV_MODELS = ("vgg16",)     # BN-free: layer-sequential unit-variance scaling


def calibrate(name: str, batch: int = 6, seed: int = 4242) -> dict:
    g, w = zoo.BUILDERS[name](calib={})
    lsuv = name in LSUV_MODELS
    users = {nid: [] for nid in g.nodes}
    for nid, node in g.nodes.items():
        for s in node.inputs:
            users[s].append(nid)
    calib: dict[str, np.ndarray] = {}

    def hook(nid, node, ins):
        if node.kind == "batchnorm_inference":
            x = ins[0]
            axes = (0, 2, 3) if x.ndim == 4 else (0,)
            mean = x.mean(axis=axes, dtype=np.float64)
            var = x.var(axis=axes, dtype=np.float64)
            var = np.maximum(var, np.median(var))
            calib[f"{nid}:mean"] = mean.astype(np.float32)
            calib[f"{nid}:var"] = var.astype(np.float32)
            gamma, beta, _, _ = bn_coeffs(w, node)
            eps = float(node.attrs.get("epsilon", 1e-5))
            sh = (1, -1) + (1,) * (x.ndim - 2)
            inv = 1.0 / np.sqrt(var + eps)
            return ((x - mean.reshape(sh)) * (gamma * inv).reshape(sh) + beta.reshape(sh)).astype(np.float32)
        if node.kind in ("conv2d", "dense"):
            out = eval_node_fast(node, ins, w)
            nxt = users[nid]
            if lsuv and not (len(nxt) == 1 and g.nodes[nxt[0]].kind == "batchnorm_inference"):
                f = 1.0 / max(float(out.std()), 1e-6)
                calib[f"{nid}:lsuv"] = np.float32(f)
                out = (out * np.float32(f)).astype(np.float32)
            return out
        return None

    xs = np.random.default_rng(seed).standard_normal((batch,) + tuple(g.input_spec.dims)).astype(np.float32)
    run_fast(g, w, xs, hook=hook)
    return calib


def main(names):
    zoo.CALIB_DIR.mkdir(exist_ok=True)
    for name in names:
        t0 = time.time()
        calib = calibrate(name)
        np.savez_compressed(zoo.CALIB_DIR / f"{name}.npz", **calib)
        print(f"{name}: {len(calib)} entries in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main(sys.argv[1:] or list(zoo.BUILDERS))
