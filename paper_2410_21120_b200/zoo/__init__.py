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
        self.beta_shift = 0.0           # mean of BN beta (see inception_v3)
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
    def conv(self, nid, src, cout, k, stride=1, pad=None, groups=1, bias=False, std=None):
        cin, h, w = self._in_dims(src)
        kh, kw = (k, k) if isinstance(k, int) else k
        if pad is None:
            pad = ((kh - 1) // 2, (kw - 1) // 2)
        ph, pw = (pad, pad) if isinstance(pad, int) else pad
        sh, sw = (stride, stride) if isinstance(stride, int) else stride
        fan_in = (cin // groups) * kh * kw
        s = self._scale(nid)
        if std is not None:              # explicit (ViT conv_proj)
            pass
        elif self.init == "lsuv":        # N(0, 1/fan_in), rescaled by calibration
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

    def dense(self, nid, src, units, bias=True, init=None, bias_std=0.0):
        """init: "lsuv" | "se" (1x1-conv kaiming fan_out) | "torch_linear"
        (U(+-1/sqrt(fan_in)) weight and bias) | "uniform_fanout" | "normal001" |
        "xavier_uniform" | "normal002".  A rank-2 (L, fan_in) input is row-wise."""
        idims = self._in_dims(src)
        fan_in = idims[-1]
        s = self._scale(nid)
        init = init or self.init
        b = (self.rng.standard_normal(units) * bias_std).astype(F32) if bias_std else np.zeros(units, F32)
        if init == "xavier_uniform":
            r = np.sqrt(6.0 / (fan_in + units))
            wt = self.rng.uniform(-r, r, units * fan_in).astype(F32)
        elif init == "normal002":
            wt = self.rng.standard_normal(units * fan_in, dtype=F32) * F32(0.02)
        elif init == "lsuv":
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
                         out_dims=tuple(idims[:-1]) + (units,))

    def layernorm(self, nid, src, eps=1e-6):
        """gamma ~ U(0.5, 1.5), beta ~ N(0, 0.1) (synthetic, like bn)."""
        c = self._in_dims(src)[-1]
        gamma = self.rng.uniform(0.5, 1.5, c).astype(F32)
        beta = (self.rng.standard_normal(c) * 0.1).astype(F32)
        refs = {"gamma": self._put(f"{nid}.gamma", (c,), gamma),
                "beta": self._put(f"{nid}.beta", (c,), beta)}
        return self._add(nid, "layernorm", src, {"epsilon": eps}, refs, out_dims=self._in_dims(src))

    def tokens(self, nid, src):
        """class token N(0, 0.02) (torchvision: zeros), pos_embedding N(0, 0.02)."""
        c, h, w = self._in_dims(src)
        cls = self.rng.standard_normal(c) * 0.02
        pos = self.rng.standard_normal((1 + h * w) * c) * 0.02
        refs = {"class_token": self._put(f"{nid}.class_token", (c,), cls),
                "pos_embedding": self._put(f"{nid}.pos_embedding", (1 + h * w, c), pos)}
        return self._add(nid, "tokens", src, {}, refs, out_dims=(1 + h * w, c))

    def attention(self, nid, src, heads):
        seq, c3 = self._in_dims(src)
        return self._add(nid, "attention", src, {"heads": heads}, out_dims=(seq, c3 // 3))

    def select_token(self, nid, src, index=0):
        return self._add(nid, "select_token", src, {"index": index},
                         out_dims=(self._in_dims(src)[-1],))

    def bn(self, nid, src, eps=1e-5, gamma_scale=1.0):
        """gamma ~ U(0.5, 1.5) * gamma_scale (gamma_scale < 1 on the last BN of a
        residual branch: the small residual-branch gain of trained ResNets, cf.
        torchvision's zero_init_residual), beta ~ N(0, 0.1)."""
        c = self._in_dims(src)[0]
        gamma = (self.rng.uniform(0.5, 1.5, c) * gamma_scale).astype(F32)
        beta = (self.rng.standard_normal(c) * 0.1 + self.beta_shift).astype(F32)
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


# Residual-branch gain of EfficientNetV2's MBConv / FusedMBConv blocks (gamma of the
# projection BN of every block with a skip connection), as for ResNet: at random init
# the 56 residual blocks otherwise compound into logits so input-chaotic that fp16
# storage noise reads as a 2-3% logit error on some inputs.
EFFNET_BRANCH_GAIN = 0.2


def efficientnet_v2_l(model_id="efficientnet_v2_l", seed=1604, calib=None, res=224, classes=1000,
                      branch_gain=None):
    n = Net(model_id, (3, res, res), seed, calib)
    gain = EFFNET_BRANCH_GAIN if branch_gain is None else branch_gain
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
                    x = n.bn(f"{p}_proj_bn", n.conv(f"{p}_proj", x, cout, 1, pad=0), eps,
                             gamma_scale=gain if (s == 1 and cin == cout) else 1.0)
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
                x = n.bn(f"{p}_proj_bn", n.conv(f"{p}_proj", x, cout, 1, pad=0), eps,
                         gamma_scale=gain if (s == 1 and cin == cout) else 1.0)
            if s == 1 and cin == cout:
                x = n.add(f"{p}_add", x, inp)
    x = n.conv("head_conv", x, 1280, 1, pad=0)
    x = n.act("head_act", n.bn("head_bn", x, eps), "silu")
    x = n.gap("pool", x)
    x = n.dense("classifier", x, classes, init="uniform_fanout")
    return n.build(x)


# ----------------------------------------------------------------------------- ResNet-50 / 152

RESNET_BRANCH_GAIN = 0.2

def _resnet(model_id, seed, calib, res, classes, layers, branch_gain=RESNET_BRANCH_GAIN):
    n = Net(model_id, (3, res, res), seed, calib)
    x = n.conv("stem_conv", None, 64, 7, stride=2, pad=3)
    x = n.act("stem_relu", n.bn("stem_bn", x), "relu")
    x = n.pool("stem_pool", x, "maxpool2d", 3, stride=2, pad=1)
    cin = 64
    for li, (blocks, planes) in enumerate(zip(layers, (64, 128, 256, 512)), start=1):
        for bi in range(1, blocks + 1):
            p = f"l{li}_b{bi:02d}"
            stride = 2 if (bi == 1 and li > 1) else 1
            inp = x
            t = n.act(f"{p}_relu1", n.bn(f"{p}_bn1", n.conv(f"{p}_conv1", x, planes, 1, pad=0)), "relu")
            t = n.act(f"{p}_relu2", n.bn(f"{p}_bn2", n.conv(f"{p}_conv2", t, planes, 3, stride=stride)), "relu")
            t = n.bn(f"{p}_bn3", n.conv(f"{p}_conv3", t, planes * 4, 1, pad=0), gamma_scale=branch_gain)
            if bi == 1:
                inp = n.bn(f"{p}_dsbn", n.conv(f"{p}_dsconv", x, planes * 4, 1, stride=stride, pad=0))
            x = n.act(f"{p}_relu3", n.add(f"{p}_add", t, inp), "relu")
            cin = planes * 4
    x = n.gap("pool", x)
    x = n.dense("fc", x, classes, init="torch_linear")
    return n.build(x)


def resnet50(model_id="resnet50", seed=1605, calib=None, res=224, classes=1000):
    return _resnet(model_id, seed, calib, res, classes, (3, 4, 6, 3))


def resnet152(model_id="resnet152", seed=1606, calib=None, res=224, classes=1000):
    return _resnet(model_id, seed, calib, res, classes, (3, 8, 36, 3))


# ----------------------------------------------------------------------------- Inception-v3

# Mean of the synthetic BN betas in Inception-v3.  With zero-mean betas the
# random-init net (no residual path) flips about half of its ReLU signs per
# layer and the logits become chaotic in the input: fp16 storage noise then
# reads as a 4% logit error.  A positive shift keeps it smooth (fp16 error
# 0.8%) while the logits still vary by ~19% across inputs.
INCEPTION_BETA_SHIFT = 0.5


def inception_v3(model_id="inception_v3", seed=1607, calib=None, res=299, classes=1000,
                 beta_shift=None):
    """torchvision inception_v3 (eval, no aux head): BasicConv2d = conv + BN(1e-3) + ReLU."""
    n = Net(model_id, (3, res, res), seed, calib)
    n.beta_shift = INCEPTION_BETA_SHIFT if beta_shift is None else beta_shift

    def basic(nid, src, cout, k, stride=1, pad=0):
        x = n.conv(f"{nid}_conv", src, cout, k, stride=stride, pad=pad)
        return n.act(f"{nid}_relu", n.bn(f"{nid}_bn", x, 1e-3), "relu")

    def block_a(p, x, pool_features):
        b1 = basic(f"{p}_b1x1", x, 64, 1)
        b5 = basic(f"{p}_b5x5_2", basic(f"{p}_b5x5_1", x, 48, 1), 64, 5, pad=2)
        bd = basic(f"{p}_b3x3dbl_1", x, 64, 1)
        bd = basic(f"{p}_b3x3dbl_3", basic(f"{p}_b3x3dbl_2", bd, 96, 3, pad=1), 96, 3, pad=1)
        bp = basic(f"{p}_bpool", n.pool(f"{p}_avg", x, "avgpool2d", 3, stride=1, pad=1), pool_features, 1)
        return n.concat(f"{p}_cat", [b1, b5, bd, bp])

    def block_b(p, x):
        b3 = basic(f"{p}_b3x3", x, 384, 3, stride=2)
        bd = basic(f"{p}_b3x3dbl_1", x, 64, 1)
        bd = basic(f"{p}_b3x3dbl_3", basic(f"{p}_b3x3dbl_2", bd, 96, 3, pad=1), 96, 3, stride=2)
        bp = n.pool(f"{p}_max", x, "maxpool2d", 3, stride=2)
        return n.concat(f"{p}_cat", [b3, bd, bp])

    def block_c(p, x, c7):
        b1 = basic(f"{p}_b1x1", x, 192, 1)
        b7 = basic(f"{p}_b7x7_1", x, c7, 1)
        b7 = basic(f"{p}_b7x7_2", b7, c7, (1, 7), pad=(0, 3))
        b7 = basic(f"{p}_b7x7_3", b7, 192, (7, 1), pad=(3, 0))
        bd = basic(f"{p}_b7x7dbl_1", x, c7, 1)
        bd = basic(f"{p}_b7x7dbl_2", bd, c7, (7, 1), pad=(3, 0))
        bd = basic(f"{p}_b7x7dbl_3", bd, c7, (1, 7), pad=(0, 3))
        bd = basic(f"{p}_b7x7dbl_4", bd, c7, (7, 1), pad=(3, 0))
        bd = basic(f"{p}_b7x7dbl_5", bd, 192, (1, 7), pad=(0, 3))
        bp = basic(f"{p}_bpool", n.pool(f"{p}_avg", x, "avgpool2d", 3, stride=1, pad=1), 192, 1)
        return n.concat(f"{p}_cat", [b1, b7, bd, bp])

    def block_d(p, x):
        b3 = basic(f"{p}_b3x3_2", basic(f"{p}_b3x3_1", x, 192, 1), 320, 3, stride=2)
        b7 = basic(f"{p}_b7x7x3_1", x, 192, 1)
        b7 = basic(f"{p}_b7x7x3_2", b7, 192, (1, 7), pad=(0, 3))
        b7 = basic(f"{p}_b7x7x3_3", b7, 192, (7, 1), pad=(3, 0))
        b7 = basic(f"{p}_b7x7x3_4", b7, 192, 3, stride=2)
        bp = n.pool(f"{p}_max", x, "maxpool2d", 3, stride=2)
        return n.concat(f"{p}_cat", [b3, b7, bp])

    def block_e(p, x):
        b1 = basic(f"{p}_b1x1", x, 320, 1)
        b3 = basic(f"{p}_b3x3_1", x, 384, 1)
        b3 = n.concat(f"{p}_b3x3_cat", [basic(f"{p}_b3x3_2a", b3, 384, (1, 3), pad=(0, 1)),
                                        basic(f"{p}_b3x3_2b", b3, 384, (3, 1), pad=(1, 0))])
        bd = basic(f"{p}_b3x3dbl_2", basic(f"{p}_b3x3dbl_1", x, 448, 1), 384, 3, pad=1)
        bd = n.concat(f"{p}_b3x3dbl_cat", [basic(f"{p}_b3x3dbl_3a", bd, 384, (1, 3), pad=(0, 1)),
                                           basic(f"{p}_b3x3dbl_3b", bd, 384, (3, 1), pad=(1, 0))])
        bp = basic(f"{p}_bpool", n.pool(f"{p}_avg", x, "avgpool2d", 3, stride=1, pad=1), 192, 1)
        return n.concat(f"{p}_cat", [b1, b3, bd, bp])

    x = basic("c1a", None, 32, 3, stride=2)
    x = basic("c2a", x, 32, 3)
    x = basic("c2b", x, 64, 3, pad=1)
    x = n.pool("pool1", x, "maxpool2d", 3, stride=2)
    x = basic("c3b", x, 80, 1)
    x = basic("c4a", x, 192, 3)
    x = n.pool("pool2", x, "maxpool2d", 3, stride=2)
    x = block_a("m5b", x, 32)
    x = block_a("m5c", x, 64)
    x = block_a("m5d", x, 64)
    x = block_b("m6a", x)
    for p, c7 in (("m6b", 128), ("m6c", 160), ("m6d", 160), ("m6e", 192)):
        x = block_c(p, x, c7)
    x = block_d("m7a", x)
    x = block_e("m7b", x)
    x = block_e("m7c", x)
    x = n.gap("pool", x)
    x = n.dense("fc", x, classes, init="torch_linear")
    return n.build(x)


# ----------------------------------------------------------------------------- ViT-B/16

def vit_b_16(model_id="vit_b_16", seed=1608, calib=None, res=224, classes=1000,
             patch=16, hidden=768, layers=12, heads=12, mlp=3072):
    """torchvision vit_b_16 (eval): conv_proj 16x16/16 -> [class token; patches] +
    pos_embedding -> 12 pre-LN encoder blocks (LN 1e-6, MHA with packed in_proj,
    out_proj, residual; LN, Linear-GELU-Linear, residual) -> LN -> token 0 -> head.
    Inits follow torchvision (trunc-normal conv_proj ~ N(0, 1/fan_in), xavier
    in_proj / MLP, N(0, 1e-6) MLP biases) except the zero-initialised pieces,
    which are synthetic here so every path carries signal: class token and LN
    affine (see Net.tokens / Net.layernorm) and the head, N(0, 0.02)."""
    n = Net(model_id, (3, res, res), seed, calib)
    x = n.conv("conv_proj", None, hidden, patch, stride=patch, pad=0, bias=True,
               std=np.sqrt(1.0 / (3 * patch * patch)))
    x = n.tokens("tokens", x)
    for i in range(layers):
        p = f"enc{i:02d}"
        y = n.layernorm(f"{p}_ln1", x)
        y = n.dense(f"{p}_qkv", y, 3 * hidden, init="xavier_uniform")
        y = n.attention(f"{p}_attn", y, heads)
        y = n.dense(f"{p}_out", y, hidden, init="torch_linear")
        x = n.add(f"{p}_add1", x, y)
        y = n.layernorm(f"{p}_ln2", x)
        y = n.dense(f"{p}_fc1", y, mlp, init="xavier_uniform", bias_std=1e-6)
        y = n.act(f"{p}_gelu", y, "gelu")
        y = n.dense(f"{p}_fc2", y, hidden, init="xavier_uniform", bias_std=1e-6)
        x = n.add(f"{p}_add2", x, y)
    x = n.layernorm("ln", x)
    x = n.select_token("cls", x, 0)
    x = n.dense("head", x, classes, init="normal002")
    return n.build(x)


BUILDERS = {
    "vit_b_16": vit_b_16,
    "vgg16": vgg16,
    "mobilenet_v3_large": mobilenet_v3_large,
    "densenet161": densenet161,
    "efficientnet_v2_l": efficientnet_v2_l,
    "resnet50": resnet50,
    "resnet152": resnet152,
    "inception_v3": inception_v3,
}
NORTH_STAR = ("vgg16", "mobilenet_v3_large", "densenet161", "efficientnet_v2_l")
EIGHT_MODEL_CNNS = NORTH_STAR + ("resnet50", "resnet152", "inception_v3")
EIGHT_MODEL = EIGHT_MODEL_CNNS + ("vit_b_16",)
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
