"""Zoo builders + oracle extension kinds vs torchvision (same weights), incl. ViT-B/16.

Pins the parts of the oracle that have no reference code (depthwise/grouped
conv, padded pools, avgpool, hardswish/hardsigmoid/SiLU/sigmoid, channel
scale) and checks that the IR builders reproduce the torchvision
architectures layer for layer: parameters are copied in module registration
order and the two forwards must agree to 1e-5 (per sample, norm-relative).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
tv = pytest.importorskip("torchvision")

from oracle.executor_ref import run_fast  # noqa: E402
from paper_2410_21120_b200 import zoo  # noqa: E402

TV = {
    "vgg16": lambda: tv.models.vgg16(),
    "mobilenet_v3_large": lambda: tv.models.mobilenet_v3_large(),
    "densenet161": lambda: tv.models.densenet161(),
    "efficientnet_v2_l": lambda: tv.models.efficientnet_v2_l(),
    "resnet50": lambda: tv.models.resnet50(),
    "resnet152": lambda: tv.models.resnet152(),
    "inception_v3": lambda: tv.models.inception_v3(aux_logits=False, init_weights=False),
    "vit_b_16": lambda: tv.models.vit_b_16(),
}


def _load_vit(g, w):
    """ViT-B/16: parameters by name (MHA's packed in_proj is not a Linear module)."""
    model = TV["vit_b_16"]().eval()

    def a(name):
        return torch.from_numpy(w.array(name).copy())

    sd = {"conv_proj.weight": a("conv_proj.weight"), "conv_proj.bias": a("conv_proj.bias"),
          "class_token": a("tokens.class_token").reshape(1, 1, -1),
          "encoder.pos_embedding": a("tokens.pos_embedding")[None],
          "encoder.ln.weight": a("ln.gamma"), "encoder.ln.bias": a("ln.beta"),
          "heads.head.weight": a("head.weight"), "heads.head.bias": a("head.bias")}
    layers = sum(1 for n in g.nodes if n.endswith("_attn"))
    for i in range(layers):
        p, q = f"enc{i:02d}", f"encoder.layers.encoder_layer_{i}"
        for ours, theirs in (("ln1", "ln_1"), ("ln2", "ln_2")):
            sd[f"{q}.{theirs}.weight"], sd[f"{q}.{theirs}.bias"] = a(f"{p}_{ours}.gamma"), a(f"{p}_{ours}.beta")
        for ours, theirs in (("out", "self_attention.out_proj"), ("fc1", "mlp.0"), ("fc2", "mlp.3")):
            sd[f"{q}.{theirs}.weight"], sd[f"{q}.{theirs}.bias"] = a(f"{p}_{ours}.weight"), a(f"{p}_{ours}.bias")
        sd[f"{q}.self_attention.in_proj_weight"] = a(f"{p}_qkv.weight")
        sd[f"{q}.self_attention.in_proj_bias"] = a(f"{p}_qkv.bias")
    model.load_state_dict(sd, strict=True)
    return model


def _input(g, seed, n):
    return np.random.default_rng(seed).standard_normal((n,) + tuple(g.input_spec.dims)).astype(np.float32)


def _load_into_torchvision(name, g, w):
    if name == "vit_b_16":
        return _load_vit(g, w)
    model = TV[name]().eval()
    mods = [m for m in model.modules()
            if isinstance(m, (torch.nn.Conv2d, torch.nn.Linear, torch.nn.BatchNorm2d))]
    ours = [n for n in g.nodes.values() if n.kind in ("conv2d", "dense", "batchnorm_inference")]
    order = list(g.nodes)              # builder creation order == module registration order
    ours.sort(key=lambda n: order.index(n.node_id))
    assert len(mods) == len(ours), (len(mods), len(ours))
    with torch.no_grad():
        for m, n in zip(mods, ours):
            if isinstance(m, torch.nn.BatchNorm2d):
                assert n.kind == "batchnorm_inference"
                m.weight.copy_(torch.from_numpy(w.array(n.weight_refs["gamma"]).copy()))
                m.bias.copy_(torch.from_numpy(w.array(n.weight_refs["beta"]).copy()))
                m.running_mean.copy_(torch.from_numpy(w.array(n.weight_refs["mean"]).copy()))
                m.running_var.copy_(torch.from_numpy(w.array(n.weight_refs["var"]).copy()))
                assert abs(m.eps - n.attrs["epsilon"]) < 1e-12
            else:
                wt = w.array(n.weight_refs["weight"])
                shape = tuple(m.weight.shape)
                # torchvision's squeeze-excitation FCs are 1x1 convs on (C,1,1)
                assert shape == wt.shape or shape == wt.shape + (1, 1), (n.node_id, shape, wt.shape)
                m.weight.copy_(torch.from_numpy(wt.copy()).reshape(shape))
                if m.bias is not None:
                    m.bias.copy_(torch.from_numpy(w.array(n.weight_refs["bias"]).copy()))
                else:
                    assert "bias" not in n.weight_refs
    return model


@pytest.mark.slow
@pytest.mark.parametrize("name", zoo.EIGHT_MODEL)
def test_builder_and_oracle_match_torchvision(name):
    torch.set_num_threads(8)
    g, w = zoo.build(name)
    model = _load_into_torchvision(name, g, w)
    xs = _input(g, 11, 2)
    with torch.no_grad():
        t32 = model(torch.from_numpy(xs)).numpy()
        t64 = model.double()(torch.from_numpy(xs).double()).numpy()
    got = run_fast(g, w, xs)

    def rel(a):
        return (np.abs(a - t64).max(axis=1) / np.abs(t64).max(axis=1)).max()

    # Reference = torchvision in fp64.  The oracle (fp32) must be as close to it as
    # torchvision's own fp32 forward is (deep residual nets reach ~3e-4 of pure
    # fp32 noise, ResNet-152); a semantic mismatch shows up at >= 1e-2.
    assert rel(got) <= max(2e-5, 2.0 * rel(t32)), (rel(got), rel(t32))


@pytest.mark.slow
@pytest.mark.parametrize("name", zoo.EIGHT_MODEL)
def test_calibrated_logits_are_input_sensitive(name):
    g, w = zoo.build(name)
    xs = _input(g, 12, 4)
    out = run_fast(g, w, xs)
    spread = np.abs(out - out.mean(axis=0)).max() / np.abs(out).max()
    assert spread > 0.05, spread
    assert np.all(np.isfinite(out))
