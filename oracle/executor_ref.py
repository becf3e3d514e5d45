"""numpy restatement of the reference executor — test infrastructure only.

Faithful engine (``run_faithful``): one sample, fp32, the fold orders of
/root/reference/pkg/src/dagfuse/executor.py:
  dense        acc += W[:, j] * x[j], j ascending; bias added last   (:56-65)
  conv2d       zero pad; acc += W[:, c, ki, kj] (x) window over
               (c, ki, kj) ascending; bias last                      (:68-92)
  maxpool2d    running max over (ki, kj) ascending, floor mode       (:95-109)
  batchnorm    gamma*(x-mean)*fp32(1/sqrt(var+eps)) + beta           (:112-123)
  gap          acc += x[:, i], i ascending; acc * fp32(1/HW)          (:126-133)
  relu         max(x, 0)                                              (:142-143)
  residual_add left fold in declared input order                     (:148-156)
  flatten      reshape(-1) (CHW order)                                (:159-160)
  concat       channel concatenation in input order                  (:161-166)
Extension kinds follow the same conventions (ascending folds, multiply by an
fp32 reciprocal for means, no implicit broadcasting):
  conv2d groups=g   per group, the (c, ki, kj) fold over that group's inputs
  maxpool2d pad     windows padded with -inf
  avgpool2d         zero-padded window sum over (ki, kj) ascending, times
                    fp32(1/count), count = kh*kw (count_include_pad) or the
                    in-bounds element count
  hardswish         x * clip(x + 3, 0, 6) / 6
  hardsigmoid       clip(x + 3, 0, 6) / 6
  silu              x / (1 + exp(-x))
  sigmoid           1 / (1 + exp(-x))
  channel_scale     x * s[:, None, None]
ViT extension kinds (torchvision VisionTransformer semantics, fp32 with
fp64 reductions — there is no reference code to follow):
  gelu              0.5 x (1 + erf(x / sqrt 2))
  dense rank-2      row-wise dense over the last axis
  tokens            [class_token; x.reshape(C, H*W).T] + pos_embedding
  layernorm         (x - mean) / sqrt(var + eps) * gamma + beta, biased var
                    over the last axis
  attention         q|k|v = split(x, 3, axis=-1); per head h (columns
                    h*d:(h+1)*d, d = C/heads): softmax(q k^T / sqrt d) v,
                    heads concatenated in order
  select_token      x[index]

Fast engine (``run_fast``): the same functions over a batch (N, ...) with
conv/dense as BLAS matmuls (im2col), for real-size models; equal to the
faithful engine up to fp32 reassociation.
"""

from __future__ import annotations

import numpy as np

from paper_2410_21120_b200.graph_ir import conv_geometry, pool_geometry, topo_order

F32 = np.float32


def _w(ws, node, role):
    return ws.array(node.weight_refs[role])


# ----------------------------------------------------------------------------
# shared elementwise definitions (batch-agnostic)

def act(kind: str, x: np.ndarray) -> np.ndarray:
    if kind == "relu":
        return np.maximum(x, F32(0.0))
    if kind == "hardswish":
        return (x * np.clip(x + F32(3.0), F32(0.0), F32(6.0)) / F32(6.0)).astype(F32)
    if kind == "hardsigmoid":
        return (np.clip(x + F32(3.0), F32(0.0), F32(6.0)) / F32(6.0)).astype(F32)
    if kind == "silu":
        with np.errstate(over="ignore"):
            return (x / (F32(1.0) + np.exp(-x))).astype(F32)
    if kind == "sigmoid":
        with np.errstate(over="ignore"):
            return (F32(1.0) / (F32(1.0) + np.exp(-x))).astype(F32)
    if kind == "gelu":
        from scipy.special import erf
        x64 = x.astype(np.float64)
        return (0.5 * x64 * (1.0 + erf(x64 / np.sqrt(2.0)))).astype(F32)
    raise KeyError(kind)


# ----------------------------------------------------------------------------
# token (ViT) kinds, batch-agnostic over leading axes

def tokens(ws, node, x):
    """x (..., C, H, W) -> (..., 1 + H*W, C)."""
    cls = _w(ws, node, "class_token")
    pos = _w(ws, node, "pos_embedding")
    c = x.shape[-3]
    t = np.swapaxes(x.reshape(x.shape[:-3] + (c, -1)), -1, -2)
    cls_b = np.broadcast_to(cls, x.shape[:-3] + (1, c))
    return (np.concatenate([cls_b, t], axis=-2) + pos).astype(F32)


def layernorm(ws, node, x):
    eps = float(node.attrs.get("epsilon", 1e-5))
    x64 = x.astype(np.float64)
    mu = x64.mean(axis=-1, keepdims=True)
    var = ((x64 - mu) ** 2).mean(axis=-1, keepdims=True)
    y = (x64 - mu) / np.sqrt(var + eps)
    return (y * _w(ws, node, "gamma") + _w(ws, node, "beta")).astype(F32)


def attention(node, x):
    """x (..., L, 3C) -> (..., L, C)."""
    heads = int(node.attrs["heads"])
    c = x.shape[-1] // 3
    d = c // heads
    x64 = x.astype(np.float64)
    outs = []
    for h in range(heads):
        q = x64[..., h * d:(h + 1) * d]
        k = x64[..., c + h * d:c + (h + 1) * d]
        v = x64[..., 2 * c + h * d:2 * c + (h + 1) * d]
        s = (q @ np.swapaxes(k, -1, -2)) / np.sqrt(d)
        s = np.exp(s - s.max(axis=-1, keepdims=True))
        outs.append((s / s.sum(axis=-1, keepdims=True)) @ v)
    return np.concatenate(outs, axis=-1).astype(F32)


def bn_coeffs(ws, node):
    eps = F32(node.attrs.get("epsilon", 1e-5))
    var = _w(ws, node, "var")
    inv = (F32(1.0) / np.sqrt(var + eps)).astype(F32)
    return _w(ws, node, "gamma"), _w(ws, node, "beta"), _w(ws, node, "mean"), inv


# ----------------------------------------------------------------------------
# faithful single-sample engine

def _pad_hw(x, ph, pw, value=0.0):
    if ph == 0 and pw == 0:
        return x
    return np.pad(x, ((0, 0), (ph, ph), (pw, pw)), mode="constant",
                  constant_values=value).astype(F32)


def _conv_faithful(node, x, ws):
    wt = _w(ws, node, "weight")
    cout, cin_g, kh, kw = wt.shape
    _, _, sh, sw, ph, pw = conv_geometry(node.attrs)
    groups = int(node.attrs.get("groups", 1))
    xp = _pad_hw(x, ph, pw)
    oh = (xp.shape[1] - kh) // sh + 1
    ow = (xp.shape[2] - kw) // sw + 1
    acc = np.zeros((cout, oh, ow), dtype=F32)
    cout_g = cout // groups
    for g in range(groups):
        o0, o1 = g * cout_g, (g + 1) * cout_g
        for c in range(cin_g):
            plane = xp[g * cin_g + c]
            for ki in range(kh):
                for kj in range(kw):
                    win = plane[ki:ki + oh * sh:sh, kj:kj + ow * sw:sw]
                    acc[o0:o1] += wt[o0:o1, c, ki, kj][:, None, None] * win[None, :, :]
    if "bias" in node.weight_refs:
        acc = acc + _w(ws, node, "bias")[:, None, None]
    return acc


def _dense_faithful(node, x, ws):
    wt = _w(ws, node, "weight")
    acc = np.zeros(x.shape[:-1] + (wt.shape[0],), dtype=F32)
    for j in range(wt.shape[1]):
        acc += wt[:, j] * x[..., j, None]
    if "bias" in node.weight_refs:
        acc = acc + _w(ws, node, "bias")
    return acc


def _pool_faithful(node, x):
    kh, kw, sh, sw, ph, pw = pool_geometry(node.attrs)
    is_max = node.kind == "maxpool2d"
    xp = _pad_hw(x, ph, pw, -np.inf if is_max else 0.0)
    oh = (xp.shape[1] - kh) // sh + 1
    ow = (xp.shape[2] - kw) // sw + 1
    acc = None
    for ki in range(kh):
        for kj in range(kw):
            win = xp[:, ki:ki + oh * sh:sh, kj:kj + ow * sw:sw]
            if acc is None:
                acc = win.copy()
            else:
                acc = np.maximum(acc, win) if is_max else acc + win
    if is_max:
        return acc
    return acc * _avg_scale(node, x.shape[1], x.shape[2], oh, ow)


def _avg_scale(node, h, w, oh, ow):
    """fp32 reciprocal of each output position's divisor, shape (oh, ow)."""
    kh, kw, sh, sw, ph, pw = pool_geometry(node.attrs)
    if int(node.attrs.get("count_include_pad", 1)):
        return np.full((oh, ow), F32(1.0 / (kh * kw)), dtype=F32)
    rows = np.array([min(i * sh - ph + kh, h) - max(i * sh - ph, 0) for i in range(oh)])
    cols = np.array([min(j * sw - pw + kw, w) - max(j * sw - pw, 0) for j in range(ow)])
    return (1.0 / (rows[:, None] * cols[None, :]).astype(np.float64)).astype(F32)


def _gap_faithful(x):
    flat = x.reshape(x.shape[0], -1)
    acc = np.zeros(x.shape[0], dtype=F32)
    for i in range(flat.shape[1]):
        acc += flat[:, i]
    return acc * F32(1.0 / flat.shape[1])


def eval_node_faithful(node, ins, ws):
    k = node.kind
    if k == "dense":
        return _dense_faithful(node, ins[0], ws)
    if k == "conv2d":
        return _conv_faithful(node, ins[0], ws)
    if k in ("maxpool2d", "avgpool2d"):
        return _pool_faithful(node, ins[0])
    if k == "batchnorm_inference":
        gamma, beta, mean, inv = bn_coeffs(ws, node)
        sh = (-1,) + (1,) * (ins[0].ndim - 1)
        return (gamma.reshape(sh) * (ins[0] - mean.reshape(sh)) * inv.reshape(sh)
                + beta.reshape(sh)).astype(F32)
    if k == "residual_add":
        acc = ins[0]
        for a in ins[1:]:
            acc = acc + a
        return acc
    if k == "global_avg_pool":
        return _gap_faithful(ins[0])
    if k == "flatten":
        return ins[0].reshape(-1)
    if k == "concat":
        return np.concatenate(ins, axis=0)
    if k == "channel_scale":
        return (ins[0] * ins[1][:, None, None]).astype(F32)
    if k == "tokens":
        return tokens(ws, node, ins[0])
    if k == "layernorm":
        return layernorm(ws, node, ins[0])
    if k == "attention":
        return attention(node, ins[0])
    if k == "select_token":
        return ins[0][int(node.attrs.get("index", 0))].copy()
    return act(k, ins[0])


def run_faithful(g, ws, x: np.ndarray) -> np.ndarray:
    """One sample (input dims, fp32) -> exit value, reference fold order."""
    vals: dict[str, np.ndarray] = {}
    x = np.asarray(x, dtype=F32).reshape(g.input_spec.dims)
    for nid in topo_order(g):
        node = g.nodes[nid]
        ins = [x] if nid == g.entry else [vals[s] for s in node.inputs]
        vals[nid] = eval_node_faithful(node, ins, ws)
    return vals[g.exit].reshape(-1)


# ----------------------------------------------------------------------------
# fast batched engine (BLAS)

def _im2col(xp, kh, kw, sh, sw, oh, ow):
    n, c = xp.shape[:2]
    cols = np.empty((n, oh, ow, c, kh, kw), dtype=F32)
    for ki in range(kh):
        for kj in range(kw):
            cols[:, :, :, :, ki, kj] = xp[:, :, ki:ki + oh * sh:sh, kj:kj + ow * sw:sw] \
                .transpose(0, 2, 3, 1)
    return cols.reshape(n * oh * ow, c * kh * kw)


def _conv_fast(node, x, ws):
    wt = _w(ws, node, "weight")
    cout, cin_g, kh, kw = wt.shape
    _, _, sh, sw, ph, pw = conv_geometry(node.attrs)
    groups = int(node.attrs.get("groups", 1))
    n, cin, h, w = x.shape
    xp = np.pad(x, ((0, 0), (0, 0), (ph, ph), (pw, pw))) if (ph or pw) else x
    oh = (h + 2 * ph - kh) // sh + 1
    ow = (w + 2 * pw - kw) // sw + 1
    if groups == cin and cin_g == 1 and cout == cin:          # depthwise: per-tap FMA
        acc = np.zeros((n, cout, oh, ow), dtype=F32)
        for ki in range(kh):
            for kj in range(kw):
                acc += wt[:, 0, ki, kj][None, :, None, None] * \
                    xp[:, :, ki:ki + oh * sh:sh, kj:kj + ow * sw:sw]
        out = acc
    else:
        cout_g = cout // groups
        outs = []
        for gi in range(groups):
            xs = xp[:, gi * cin_g:(gi + 1) * cin_g]
            cols = _im2col(xs, kh, kw, sh, sw, oh, ow)
            wm = wt[gi * cout_g:(gi + 1) * cout_g].reshape(cout_g, -1)
            outs.append((cols @ wm.T).reshape(n, oh, ow, cout_g).transpose(0, 3, 1, 2))
        out = outs[0] if groups == 1 else np.concatenate(outs, axis=1)
    if "bias" in node.weight_refs:
        out = out + _w(ws, node, "bias")[None, :, None, None]
    return np.ascontiguousarray(out, dtype=F32)


def _pool_fast(node, x):
    kh, kw, sh, sw, ph, pw = pool_geometry(node.attrs)
    is_max = node.kind == "maxpool2d"
    xp = np.pad(x, ((0, 0), (0, 0), (ph, ph), (pw, pw)),
                constant_values=-np.inf if is_max else 0.0) if (ph or pw) else x
    oh = (x.shape[2] + 2 * ph - kh) // sh + 1
    ow = (x.shape[3] + 2 * pw - kw) // sw + 1
    acc = None
    for ki in range(kh):
        for kj in range(kw):
            win = xp[:, :, ki:ki + oh * sh:sh, kj:kj + ow * sw:sw]
            acc = win.copy() if acc is None else (np.maximum(acc, win) if is_max else acc + win)
    if is_max:
        return acc.astype(F32)
    return (acc * _avg_scale(node, x.shape[2], x.shape[3], oh, ow)).astype(F32)


def eval_node_fast(node, ins, ws):
    k = node.kind
    x = ins[0]
    if k == "dense":
        out = x @ _w(ws, node, "weight").T
        if "bias" in node.weight_refs:
            out = out + _w(ws, node, "bias")
        return out.astype(F32)
    if k == "conv2d":
        return _conv_fast(node, x, ws)
    if k in ("maxpool2d", "avgpool2d"):
        return _pool_fast(node, x)
    if k == "batchnorm_inference":
        gamma, beta, mean, inv = bn_coeffs(ws, node)
        sh = (1, -1) + (1,) * (x.ndim - 2)
        return (gamma.reshape(sh) * (x - mean.reshape(sh)) * inv.reshape(sh)
                + beta.reshape(sh)).astype(F32)
    if k == "residual_add":
        acc = ins[0]
        for a in ins[1:]:
            acc = acc + a
        return acc
    if k == "global_avg_pool":
        n, c = x.shape[:2]
        return (x.reshape(n, c, -1).sum(axis=2, dtype=F32) * F32(1.0 / (x[0, 0].size))).astype(F32)
    if k == "flatten":
        return x.reshape(x.shape[0], -1)
    if k == "concat":
        return np.concatenate(ins, axis=1)
    if k == "channel_scale":
        return (x * ins[1][:, :, None, None]).astype(F32)
    if k == "tokens":
        return tokens(ws, node, x)
    if k == "layernorm":
        return layernorm(ws, node, x)
    if k == "attention":
        return attention(node, x)
    if k == "select_token":
        return np.ascontiguousarray(x[:, int(node.attrs.get("index", 0))])
    return act(k, x)


def run_fast(g, ws, xs: np.ndarray, hook=None) -> np.ndarray:
    """Batch (N, *input_dims) -> (N, *output_dims).  ``hook(nid, node, ins)`` may
    return a replacement output (used by calibration)."""
    xs = np.asarray(xs, dtype=F32).reshape((-1,) + tuple(g.input_spec.dims))
    vals: dict[str, np.ndarray] = {}
    order = topo_order(g)
    users: dict[str, int] = {nid: 0 for nid in g.nodes}
    for node in g.nodes.values():
        for s in node.inputs:
            users[s] += 1
    for nid in order:
        node = g.nodes[nid]
        ins = [xs] if nid == g.entry else [vals[s] for s in node.inputs]
        out = hook(nid, node, ins) if hook is not None else None
        vals[nid] = eval_node_fast(node, ins, ws) if out is None else out
        for s in node.inputs:           # free dead values (real-size models)
            users[s] -= 1
            if users[s] == 0 and s != g.exit:
                vals.pop(s, None)
    return vals[g.exit]
