"""Real-size CNNs written in the graph IR (reference JSON/FIWT compatible).

The north-star fused DAG is VGG16 + MobileNetV3-Large + DenseNet161 +
EfficientNetV2-L at 3x224x224 (BASELINE.json configs).  The reference only
ships 3x8x8 toy stand-ins for them (/root/reference/pkg/scenario/models/), so
these builders reproduce the torchvision architectures layer for layer
(checked against torchvision CPU fp32 in tests/test_zoo_torchvision.py):
VGG16 needs only the nine reference kinds and runs unchanged through the
reference executor; the others use the extension kinds of graph_ir.

Weights are synthetic (no checkpoints offline), seeded, with torchvision's
own init per model (kaiming-normal convs, the models' Linear inits, zero
biases), BN gamma ~ U(0.5, 1.5), beta ~ N(0, 0.1); VGG16 (no BN) uses
N(0, 1/fan_in) + LSUV.  The
"calibrated init" of SURVEY.md §7 hard part 2 makes logits input-sensitive:
BN running statistics are measured on synthetic N(0,1) batches (variance
clamped at its per-layer median) and BN-free layers are LSUV-scaled to unit
output variance.  Those statistics are data files
(zoo/calib/<model>.npz, produced by oracle/calibrate.py) so every machine
regenerates bit-identical weights from (seed, calib) without running a
forward pass.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from ..graph_ir import ModelGraph, OpNode, TensorSpec, WeightStore, infer_shapes

CALIB_DIR = Path(__file__).resolve().parent / "calib"
F32 = np.float32


def make_divisible(v: float, divisor: int = 8) -> int:
    new = max(divisor, int(v + divisor / 2) // divisor * divisor)
    if new < 0.9 * v:
        new += divisor
    return new


class Net:
    """Incremental builder: nodes in creation order, weights from one seeded RNG."""

    def __init__(self, model_id: str, input_dims, seed: int, calib: dict | None = None,
                 init: str = "kaiming_fan_out"):
        self.model_id = model_id
        self.init = init
        self.input_dims = tuple(input_dims)
        self.rng = np.random.default_rng(seed)
        self.calib = calib or {}
        self.nodes: list[OpNode] = []
        self.w = WeightStore()
        self.dims: dict[str, tuple] = {}
        self.entry = None

    # ---- plumbing
    def _in_dims(self, src):
        return self.input_dims if src is None else self.dims[src]

    def _add(self, nid, kind, src, attrs=None, refs=None, extra=(), out_dims=None):
        ins = () if src is None else (src,)
        node = OpNode(nid, kind, attrs or {}, refs or {}, ins + tuple(extra))
        self.nodes.append(node)
        if self.entry is None:
            self.entry = nid
        self.dims[nid] = out_dims
        return nid

    def _put(self, name, dims, values):
        self.w.put(name, TensorSpec(dims), np.asarray(values, dtype=F32))
        return name

    def _scale(self, nid) -> float:
        return float(self.calib.get(f"{nid}:lsuv", 1.0))

    # ---- layers
    def conv(self, nid, src, cout, k, stride=1, pad=None, groups=1, bias=False):
        cin, h, w = self._in_dims(src)
        kh, kw = (k, k) if isinstance(k, int) else k
        if pad is None:
            pad = ((kh - 1) // 2, (kw - 1) // 2)
        ph, pw = (pad, pad) if isinstance(pad, int) else pad
        sh, sw = (stride, stride) if isinstance(stride, int) else stride
        fan_in = (cin // groups) * kh * kw
        s = self._scale(nid)
        if self.init == "lsuv":          # N(0, 1/fan_in), rescaled by calibration
            std = s / np.sqrt(fan_in)
        elif self.init == "kaiming_fan_in":
            std = np.sqrt(2.0 / fan_in)
        else:                            # torchvision kaiming_normal_(mode="fan_out")
            std = np.sqrt(2.0 / (cout * kh * kw))
        wt = self.rng.standard_normal(cout * fan_in, dtype=F32) * F32(std)
        refs = {"weight": self._put(f"{nid}.weight", (cout, cin // groups, kh, kw), wt)}
        if bias:
            b = self.rng.standard_normal(cout, dtype=F32) * F32(0.01 * s) if self.init == "lsuv" \
                else np.zeros(cout, F32)
            refs["bias"] = self._put(f"{nid}.bias", (cout,), b)
        attrs = {"out_channels": cout, "stride": sh, "padding": ph}
        if kh == kw:
            attrs["kernel"] = kh
        else:
            attrs.update(kernel_h=kh, kernel_w=kw)
        if pw != ph:
            attrs.update(padding_h=ph, padding_w=pw)
        if sw != sh:
            attrs.update(stride_h=sh, stride_w=sw)
        if groups != 1:
            attrs["groups"] = groups
        oh, ow = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
        return self._add(nid, "conv2d", src, attrs, refs, out_dims=(cout, oh, ow))

    def dense(self, nid, src, units, bias=True, init=None):
        """init: "lsuv" | "se" (1x1-conv kaiming fan_out) | "torch_linear"
        (U(+-1/sqrt(fan_in)) weight and bias) | "uniform_fanout" | "normal001"."""
        (fan_in,) = self._in_dims(src)
        s = self._scale(nid)
        init = init or self.init
        b = np.zeros(units, F32)
        if init == "lsuv":
            wt = self.rng.standard_normal(units * fan_in, dtype=F32) * F32(s / np.sqrt(fan_in))
            b = self.rng.standard_normal(units, dtype=F32) * F32(0.01 * s)
        elif init == "se":
            wt = self.rng.standard_normal(units * fan_in, dtype=F32) * F32(np.sqrt(2.0 / units))
        elif init == "torch_linear":
            r = 1.0 / np.sqrt(fan_in)
            wt = self.rng.uniform(-r, r, units * fan_in).astype(F32)
            b = self.rng.uniform(-r, r, units).astype(F32)
        elif init == "uniform_fanout":
            r = 1.0 / np.sqrt(units)
            wt = self.rng.uniform(-r, r, units * fan_in).astype(F32)
        elif init == "normal001":
            wt = self.rng.standard_normal(units * fan_in, dtype=F32) * F32(0.01)
        else:
            raise ValueError(init)
        refs = {"weight": self._put(f"{nid}.weight", (units, fan_in), wt)}
        if bias:
            refs["bias"] = self._put(f"{nid}.bias", (units,), b)
        return self._add(nid, "dense", src, {"units": units, "fan_in": fan_in}, refs,
                         out_dims=(units,))

    def bn(self, nid, src, eps=1e-5):
        c = self._in_dims(src)[0]
        gamma = self.rng.uniform(0.5, 1.5, c).astype(F32)
        beta = (self.rng.standard_normal(c) * 0.1).astype(F32)
        mean = np.asarray(self.calib.get(f"{nid}:mean", np.zeros(c)), F32)
        var = np.asarray(self.calib.get(f"{nid}:var", np.ones(c)), F32)
        refs = {r: self._put(f"{nid}.{r}", (c,), v)
                for r, v in (("gamma", gamma), ("beta", beta), ("mean", mean), ("var", var))}
        return self._add(nid, "batchnorm_inference", src, {"epsilon": eps}, refs,
                         out_dims=self._in_dims(src))

    def act(self, nid, src, kind):
        return self._add(nid, kind, src, out_dims=self._in_dims(src))

    def pool(self, nid, src, kind, k, stride=None, pad=0, count_include_pad=1):
        c, h, w = self._in_dims(src)
        stride = k if stride is None else stride
        attrs = {"kernel": k, "stride": stride}
        if pad:
            attrs["padding"] = pad
        if kind == "avgpool2d" and not count_include_pad:
            attrs["count_include_pad"] = 0
        oh, ow = (h + 2 * pad - k) // stride + 1, (w + 2 * pad - k) // stride + 1
        return self._add(nid, kind, src, attrs, out_dims=(c, oh, ow))

    def gap(self, nid, src):
        return self._add(nid, "global_avg_pool", src, out_dims=(self._in_dims(src)[0],))

    def flatten(self, nid, src):
        return self._add(nid, "flatten", src, out_dims=(int(np.prod(self._in_dims(src))),))

    def add(self, nid, a, b):
        return self._add(nid, "residual_add", a, extra=(b,), out_dims=self.dims[a])

    def scale(self, nid, x, s):
        return self._add(nid, "channel_scale", x, extra=(s,), out_dims=self.dims[x])

    def concat(self, nid, parts):
        d0 = self.dims[parts[0]]
        out = (sum(self.dims[p][0] for p in parts),) + tuple(d0[1:])
        return self._add(nid, "concat", parts[0], extra=tuple(parts[1:]), out_dims=out)

    def build(self, exit_id) -> tuple[ModelGraph, WeightStore]:
        g = ModelGraph(self.model_id, self.nodes, self.entry, exit_id, TensorSpec(self.input_dims),
                       TensorSpec(self.dims[exit_id]))
        shapes = infer_shapes(g)
        for nid, d in self.dims.items():
            assert shapes[nid].dims == tuple(d), (nid, shapes[nid].dims, d)
        return g, self.w


# ----------------------------------------------------------------------------- VGG16

VGG16_CFG = (64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M")


def vgg16(model_id="vgg16", seed=1601, calib=None, res=224, classes=1000):
    """torchvision vgg16 (config D, no BN); only reference-IR kinds.  LSUV init."""
    n = Net(model_id, (3, res, res), seed, calib, init="lsuv")
    x, i, blk = None, 0, 1
    for v in VGG16_CFG:
        if v == "M":
            x = n.pool(f"b{blk}_pool", x, "maxpool2d", 2)
            blk, i = blk + 1, 0
        else:
            i += 1
            x = n.conv(f"b{blk}_conv{i}", x, v, 3, pad=1, bias=True)
            x = n.act(f"b{blk}_relu{i}", x, "relu")
    x = n.flatten("flatten", x)
    x = n.act("fc6_relu", n.dense("fc6", x, 4096), "relu")
    x = n.act("fc7_relu", n.dense("fc7", x, 4096), "relu")
    x = n.dense("fc8", x, classes)
    return n.build(x)


# ----------------------------------------------------------------------------- MobileNetV3-L

MBV3L_CFG = (  # in, kernel, expanded, out, se, act, stride
    (16, 3, 16, 16, False, "relu", 1), (16, 3, 64, 24, False, "relu", 2),
    (24, 3, 72, 24, False, "relu", 1), (24, 5, 72, 40, True, "relu", 2),
    (40, 5, 120, 40, True, "relu", 1), (40, 5, 120, 40, True, "relu", 1),
    (40, 3, 240, 80, False, "hardswish", 2), (80, 3, 200, 80, False, "hardswish", 1),
    (80, 3, 184, 80, False, "hardswish", 1), (80, 3, 184, 80, False, "hardswish", 1),
    (80, 3, 480, 112, True, "hardswish", 1), (112, 3, 672, 112, True, "hardswish", 1),
    (112, 5, 672, 160, True, "hardswish", 2), (160, 5, 960, 160, True, "hardswish", 1),
    (160, 5, 960, 160, True, "hardswish", 1),
)


def mobilenet_v3_large(model_id="mobilenet_v3_large", seed=1602, calib=None, res=224, classes=1000):
    n = Net(model_id, (3, res, res), seed, calib)
    eps = 1e-3
    x = n.conv("stem_conv", None, 16, 3, stride=2, pad=1)
    x = n.act("stem_act", n.bn("stem_bn", x, eps), "hardswish")
    for bi, (cin, k, exp, cout, se, act, s) in enumerate(MBV3L_CFG, start=1):
        p = f"blk{bi:02d}"
        inp = x
        if exp != cin:
            x = n.act(f"{p}_exp_act", n.bn(f"{p}_exp_bn", n.conv(f"{p}_exp", x, exp, 1, pad=0), eps), act)
        x = n.conv(f"{p}_dw", x, exp, k, stride=s, pad=(k - 1) // 2, groups=exp)
        x = n.act(f"{p}_dw_act", n.bn(f"{p}_dw_bn", x, eps), act)
        if se:
            sq = make_divisible(exp // 4, 8)
            t = n.gap(f"{p}_se_pool", x)
            t = n.act(f"{p}_se_relu", n.dense(f"{p}_se_fc1", t, sq, init="se"), "relu")
            t = n.act(f"{p}_se_gate", n.dense(f"{p}_se_fc2", t, exp, init="se"), "hardsigmoid")
            x = n.scale(f"{p}_se_scale", x, t)
        x = n.bn(f"{p}_proj_bn", n.conv(f"{p}_proj", x, cout, 1, pad=0), eps)
        if s == 1 and cin == cout:
            x = n.add(f"{p}_add", x, inp)
    x = n.conv("last_conv", x, 960, 1, pad=0)
    x = n.act("last_act", n.bn("last_bn", x, eps), "hardswish")
    x = n.gap("pool", x)
    x = n.act("fc1_act", n.dense("fc1", x, 1280, init="normal001"), "hardswish")
    x = n.dense("fc2", x, classes, init="normal001")
    return n.build(x)


# ----------------------------------------------------------------------------- DenseNet161

def densenet161(model_id="densenet161", seed=1603, calib=None, res=224, classes=1000,
                growth=48, blocks=(6, 12, 36, 24), init=96, bn_size=4):
    n = Net(model_id, (3, res, res), seed, calib, init="kaiming_fan_in")
    x = n.conv("stem_conv", None, init, 7, stride=2, pad=3)
    x = n.act("stem_relu", n.bn("stem_bn", x), "relu")
    x = n.pool("stem_pool", x, "maxpool2d", 3, stride=2, pad=1)
    c = init
    for bi, layers in enumerate(blocks, start=1):
        feats = x
        for li in range(1, layers + 1):
            p = f"d{bi}_l{li:02d}"
            t = n.act(f"{p}_relu1", n.bn(f"{p}_bn1", feats), "relu")
            t = n.conv(f"{p}_conv1", t, bn_size * growth, 1, pad=0)
            t = n.act(f"{p}_relu2", n.bn(f"{p}_bn2", t), "relu")
            t = n.conv(f"{p}_conv2", t, growth, 3, pad=1)
            feats = n.concat(f"{p}_cat", [feats, t])
            c += growth
        x = feats
        if bi != len(blocks):
            p = f"t{bi}"
            x = n.act(f"{p}_relu", n.bn(f"{p}_bn", x), "relu")
            c //= 2
            x = n.conv(f"{p}_conv", x, c, 1, pad=0)
            x = n.pool(f"{p}_pool", x, "avgpool2d", 2)
    x = n.act("final_relu", n.bn("final_bn", x), "relu")
    x = n.gap("pool", x)
    x = n.dense("classifier", x, classes, init="torch_linear")
    return n.build(x)


# ----------------------------------------------------------------------------- EfficientNetV2-L

EFFV2L_CFG = (  # block, expand, kernel, stride, in, out, layers
    ("fused", 1, 3, 1, 32, 32, 4), ("fused", 4, 3, 2, 32, 64, 7),
    ("fused", 4, 3, 2, 64, 96, 7), ("mb", 4, 3, 2, 96, 192, 10),
    ("mb", 6, 3, 1, 192, 224, 19), ("mb", 6, 3, 2, 224, 384, 25),
    ("mb", 6, 3, 1, 384, 640, 7),
)


def efficientnet_v2_l(model_id="efficientnet_v2_l", seed=1604, calib=None, res=224, classes=1000):
    n = Net(model_id, (3, res, res), seed, calib)
    eps = 1e-3
    x = n.conv("stem_conv", None, 32, 3, stride=2, pad=1)
    x = n.act("stem_act", n.bn("stem_bn", x, eps), "silu")
    for si, (kind, e, k, s0, cin0, cout, layers) in enumerate(EFFV2L_CFG, start=1):
        for li in range(1, layers + 1):
            cin, s = (cin0, s0) if li == 1 else (cout, 1)
            p = f"s{si}_b{li:02d}"
            inp = x
            if kind == "fused":
                if e == 1:
                    x = n.act(f"{p}_act", n.bn(f"{p}_bn", n.conv(f"{p}_conv", x, cout, k, stride=s), eps), "silu")
                else:
                    x = n.conv(f"{p}_exp", x, make_divisible(cin * e), k, stride=s)
                    x = n.act(f"{p}_exp_act", n.bn(f"{p}_exp_bn", x, eps), "silu")
                    x = n.bn(f"{p}_proj_bn", n.conv(f"{p}_proj", x, cout, 1, pad=0), eps)
            else:
                exp = make_divisible(cin * e)
                x = n.act(f"{p}_exp_act", n.bn(f"{p}_exp_bn", n.conv(f"{p}_exp", x, exp, 1, pad=0), eps), "silu")
                x = n.conv(f"{p}_dw", x, exp, k, stride=s, groups=exp)
                x = n.act(f"{p}_dw_act", n.bn(f"{p}_dw_bn", x, eps), "silu")
                sq = max(1, cin // 4)
                t = n.gap(f"{p}_se_pool", x)
                t = n.act(f"{p}_se_act", n.dense(f"{p}_se_fc1", t, sq, init="se"), "silu")
                t = n.act(f"{p}_se_gate", n.dense(f"{p}_se_fc2", t, exp, init="se"), "sigmoid")
                x = n.scale(f"{p}_se_scale", x, t)
                x = n.bn(f"{p}_proj_bn", n.conv(f"{p}_proj", x, cout, 1, pad=0), eps)
            if s == 1 and cin == cout:
                x = n.add(f"{p}_add", x, inp)
    x = n.conv("head_conv", x, 1280, 1, pad=0)
    x = n.act("head_act", n.bn("head_bn", x, eps), "silu")
    x = n.gap("pool", x)
    x = n.dense("classifier", x, classes, init="uniform_fanout")
    return n.build(x)


BUILDERS = {
    "vgg16": vgg16,
    "mobilenet_v3_large": mobilenet_v3_large,
    "densenet161": densenet161,
    "efficientnet_v2_l": efficientnet_v2_l,
}
NORTH_STAR = ("vgg16", "mobilenet_v3_large", "densenet161", "efficientnet_v2_l")
PAIR = ("vgg16", "mobilenet_v3_large")


def load_calib(name: str) -> dict | None:
    path = CALIB_DIR / f"{name}.npz"
    if not path.exists():
        return None
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def build(name: str, calibrated: bool = True, **kw):
    """Graph + weights of a zoo model; calibrated statistics when available."""
    calib = load_calib(name) if calibrated else None
    return BUILDERS[name](calib=calib, **kw)
