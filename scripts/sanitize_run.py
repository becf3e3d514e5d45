"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): every kernel
family of libdfx once, on small inputs, each checked against the CPU oracle so a
sanitizer run also proves the kernels still compute the right thing.

  compute-sanitizer --tool memcheck python scripts/sanitize_run.py

Families: gemm_kernel (plain, split-K + splitk_kernel, cluster split-K, m2,
depthwise epilogue incl. its 2-CTA cluster form), gemm_persist_kernel,
dwconv (tiled + generic), pool, gap, ew (vector + generic), SE cluster kernel,
in / in_im2col / out, LN / tokens / attention (tiny ViT), and the split-precision
(fp16x2) instantiations of the GEMM and bandwidth kernels.
"""

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle.executor_ref import run_fast  # noqa: E402
from paper_2410_21120_b200 import graph_ir, zoo  # noqa: E402
from paper_2410_21120_b200.device import DeviceDag  # noqa: E402
from test_gpu_split import conv_model  # noqa: E402


def rel(got, ref):
    got = np.asarray(got, np.float64).reshape(len(got), -1)
    ref = np.asarray(ref, np.float64).reshape(len(ref), -1)
    return float((np.abs(got - ref).max(axis=1) / np.maximum(np.abs(ref).max(axis=1), 1e-30)).max())


def check(name, g, w, xs, precision="fp16", tol=2e-2):
    t0 = time.perf_counter()
    dd = DeviceDag([(g, w)], 0, "concurrent", precision=precision)
    try:
        (got,) = dd.execute([xs])
    finally:
        dd.free()
    err = rel(got, run_fast(g, w, xs))
    ok = err <= tol
    print(f"{'ok  ' if ok else 'FAIL'} {name:42s} {precision:7s} rel {err:.2e}  {time.perf_counter() - t0:.1f}s",
          flush=True)
    return ok


def kinds_chain():
    """depthwise 3x3 + 5x5/2, SE (GAP -> FC -> act -> FC -> sigmoid -> scale), pools,
    residual add, dense: the bandwidth kernels."""
    rng = np.random.default_rng(3)
    st = graph_ir.WeightStore()
    shapes = {"pw0": ((32, 16, 1, 1), .25), "dw": ((32, 1, 3, 3), .3), "f1": ((8, 32), .2), "f2": ((32, 8), .3),
              "dw5": ((32, 1, 5, 5), .2), "pw1": ((16, 32, 1, 1), .2), "fc": ((10, 16), .3), "fcb": ((10,), .1)}
    for k, (shp, sc) in shapes.items():
        st.put(k, graph_ir.TensorSpec(shp), rng.standard_normal(int(np.prod(shp))) * sc)
    O = graph_ir.OpNode
    nodes = [
        O("a", "conv2d", {"out_channels": 32, "kernel": 1}, {"weight": "pw0"}),
        O("b", "hardswish", inputs=("a",)),
        O("c", "conv2d", {"out_channels": 32, "kernel": 3, "stride": 1, "padding": 1, "groups": 32},
          {"weight": "dw"}, ("b",)),
        O("d", "silu", inputs=("c",)),
        O("e", "global_avg_pool", inputs=("d",)),
        O("f", "dense", {"units": 8, "fan_in": 32}, {"weight": "f1"}, ("e",)),
        O("h", "relu", inputs=("f",)),
        O("i", "dense", {"units": 32, "fan_in": 8}, {"weight": "f2"}, ("h",)),
        O("j", "sigmoid", inputs=("i",)),
        O("k", "channel_scale", inputs=("d", "j")),
        O("l", "conv2d", {"out_channels": 32, "kernel": 5, "stride": 2, "padding": 2, "groups": 32},
          {"weight": "dw5"}, ("k",)),
        O("m", "maxpool2d", {"kernel": 3, "stride": 1, "padding": 1}, inputs=("l",)),
        O("n", "avgpool2d", {"kernel": 3, "stride": 1, "padding": 1, "count_include_pad": 0}, inputs=("m",)),
        O("o", "residual_add", inputs=("n", "l")),
        O("p", "conv2d", {"out_channels": 16, "kernel": 1}, {"weight": "pw1"}, ("o",)),
        O("q", "global_avg_pool", inputs=("p",)),
        O("r", "dense", {"units": 10, "fan_in": 16}, {"weight": "fc", "bias": "fcb"}, ("q",)),
    ]
    g = graph_ir.ModelGraph("kinds", nodes, "a", "r", graph_ir.TensorSpec((16, 20, 20)), graph_ir.TensorSpec((10,)))
    return g, st, rng.standard_normal((3, 16, 20, 20)).astype(np.float32)


def main():
    quick = "--quick" in sys.argv
    ok = True
    rng = np.random.default_rng(0)
    convs = [  # cin, h, w, cout, k, s, p, n: stem/im2col, plain, split-K, persistent, m2
        ("stem im2col 7x7/2", (3, 32, 32, 64, 7, 2, 3, 2)),
        ("3x3 split-K (cluster at batch 1)", (256, 14, 14, 512, 3, 1, 1, 1)),
        ("3x3 split-K workspace + splitk_kernel", (512, 7, 7, 512, 3, 1, 1, 3)),
        ("persistent multi-wave 3x3", (32, 56, 56, 128, 3, 1, 1, 13)),
        ("m2 256-row CTAs", (192, 28, 28, 256, 3, 1, 1, 21)),
        ("ragged 5x5/2 channel tail", (40, 9, 11, 300, 5, 2, 2, 2)),
    ]
    for name, c in convs:
        g, w = conv_model(*c[:7], seed=c[0] * 7 + c[3], act="relu")
        xs = rng.standard_normal((c[7],) + c[:3]).astype(np.float32)
        ok &= check(name, g, w, xs)
        if name.startswith(("stem", "3x3 split-K (", "persistent")):
            ok &= check(name, g, w, xs, "fp16x2", 2e-4)
    g, w, xs = kinds_chain()
    ok &= check("dw / SE / pools / residual / dense chain", g, w, xs)
    ok &= check("dw / SE / pools / residual / dense chain", g, w, xs, "fp16x2", 2e-4)
    vt, vw = zoo.vit_b_16(model_id="vit_tiny", res=32, patch=8, hidden=128, layers=1, heads=2, mlp=256, classes=10)
    ok &= check("tiny ViT (LN / tokens / attention)", vt, vw, rng.standard_normal((2, 3, 32, 32)).astype(np.float32))
    if not quick:
        # EfficientNetV2-L at batch 1: depthwise epilogue (one-tile and 2-CTA cluster),
        # SE clusters with the x tile, cluster split-K; DenseNet-161: concat copies,
        # pre-activation BN ew kernels
        for name in ("efficientnet_v2_l", "densenet161"):
            g, w = zoo.build(name)
            xs = np.random.default_rng(5).standard_normal((1,) + tuple(g.input_spec.dims)).astype(np.float32)
            ok &= check(name + " batch 1", g, w, xs)
    print("SANITIZE-RUN", "PASS" if ok else "FAIL")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
