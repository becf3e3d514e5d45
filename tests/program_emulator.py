"""numpy interpreter of a lowered MemberProgram — test infrastructure.

Executes exactly what the GPU would: the launch list over ONE flat activation
arena laid out by ``device.plan_member`` (so an overlap bug in the planner
corrupts results here too), GEMM weights read back from their packed bf16
(r, s, channel-block) K order, epilogue slots in dfx.h order, bf16 rounding
of every stored activation.  Lets the lowering be checked on CPU before any
GPU time is spent.
"""

from __future__ import annotations

import numpy as np

from paper_2410_21120_b200.device import plan_member
from paper_2410_21120_b200.lower import storage_bits_to_f32, to_storage_bits


def _act(kind, v):
    if kind is None:
        return v
    if kind == "relu":
        return np.maximum(v, 0)
    if kind == "hardswish":
        return v * np.clip(v + 3, 0, 6) / 6
    if kind == "hardsigmoid":
        return np.clip(v + 3, 0, 6) / 6
    if kind == "silu":
        return v / (1 + np.exp(-v))
    if kind == "sigmoid":
        return 1 / (1 + np.exp(-v))
    if kind == "gelu":
        from scipy.special import erf
        return (0.5 * v * (1 + erf(v / np.sqrt(2)))).astype(np.float32)
    raise KeyError(kind)


class Emulator:
    def __init__(self, prog, n, round_bf16=True):
        self.p, self.n = prog, n
        self.plan = plan_member(prog, n)
        self.arena = np.full(self.plan.arena_bytes // 2 + 8, np.nan, dtype=np.float32)
        self.round = round_bf16

    def view(self, name):
        v = self.p.values[name]
        b = self.p.buffers[v.buf]
        base = self.plan.offsets[v.buf] // 2
        full = self.arena[base:base + self.n * v.h * v.w * b.pitch].reshape(self.n, v.h, v.w, b.pitch)
        return full[..., v.coff:v.coff + v.c]

    def q(self, x):
        """Round to the program's 16-bit storage type."""
        pr = self.p.precision
        return storage_bits_to_f32(to_storage_bits(np.asarray(x, np.float32), pr), pr)

    def store(self, dst_view, vals):
        dst_view[...] = self.q(vals) if self.round else vals

    def epilogue(self, L, x):
        e = L.epi
        v = x.astype(np.float32)
        if e.alpha is not None:
            v = v * e.alpha
        if e.beta is not None:
            v = v + e.beta
        v = _act(e.act1, v)
        if e.binop == 1:
            v = v + self.view(e.other)
        elif e.binop == 2:
            v = v * self.view(e.other)[:, 0:1, 0:1, :]
        return _act(e.act2, v)

    def run(self, xs):
        p = self.p
        xs = np.asarray(xs, np.float32).reshape((self.n,) + tuple(p.input_dims))
        iv = self.view("<input>")
        ic = getattr(p, "input_im2col", None)
        if ic is not None:                      # im2col of the entry conv, channel order (r, s, c)
            kh, kw, sh, sw, ph, pw = ic
            n, c, h, w = xs.shape
            xp = np.pad(xs, ((0, 0), (0, 0), (ph, ph), (pw, pw)))
            oh, ow = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
            cols = [xp[:, :, r:r + oh * sh:sh, s:s + ow * sw:sw] for r in range(kh) for s in range(kw)]
            xs = np.concatenate(cols, axis=1)   # (n, kh*kw*c, oh, ow), (r, s) major, c minor
            kb = getattr(p, "input_split", 0)
            if kb:                              # [x_hi | x_hi | x_lo], blocks of kb channels
                pad = np.zeros((n, kb - xs.shape[1], oh, ow), np.float32)
                hi = self.q(xs)
                xs = np.concatenate([xs, pad, xs, pad, (xs - hi).astype(np.float32), pad], axis=1)
        if xs.ndim == 4:
            self.store(iv, xs.transpose(0, 2, 3, 1))
        else:
            self.store(iv, xs[:, None, None, :])
        for L in p.launches:
            getattr(self, "do_" + L.kind)(L)
        out = self.view(p.exit_value)        # (n, h, w, c) -> logical CHW flatten
        return out.transpose(0, 3, 1, 2).reshape(self.n, -1)

    def do_gemm(self, L):
        g = L.geom
        x = self.view(L.src)
        key = L.blobs["weight"]
        dbg = getattr(self.p, "debug_f32", {})
        packed = dbg[key] if (not self.round and key in dbg) else \
            storage_bits_to_f32(self.p.blobs[key], self.p.precision)
        w = packed.reshape(g["cout"], g["kh"], g["kw"], g["cblocks"] * g["cb"])[..., :g["cin"]]
        if self.round:
            x = self.q(x)
        if L.pre is not None:                   # A prologue transform, rounded like the smem rewrite
            pe = L.pre
            if pe.binop == 2:
                x = x * self.view(pe.other)[:, 0:1, 0:1, :]
            else:
                if pe.alpha is not None:
                    x = x * pe.alpha
                if pe.beta is not None:
                    x = x + pe.beta
                x = _act(pe.act1, x)
            x = self.q(x) if self.round else x.astype(np.float32)
        n, h, wd, c = x.shape
        xp = np.pad(x, ((0, 0), (g["ph"], g["ph"]), (g["pw"], g["pw"]), (0, 0)))
        out = self.view(L.dst)
        P, Q = out.shape[1], out.shape[2]
        acc = np.zeros((n, P, Q, g["cout"]), np.float64)
        for r in range(g["kh"]):
            for s in range(g["kw"]):
                win = xp[:, r:r + P * g["sh"]:g["sh"], s:s + Q * g["sw"]:g["sw"], :]
                acc += np.einsum("npqc,oc->npqo", win, w[:, r, s, :], optimize=True)
        self.store(out, self.epilogue(L, acc.astype(np.float32)))

    def do_dwconv(self, L):
        g = L.geom
        x = self.view(L.src)
        taps = self.p.blobs[L.blobs["weight"]].reshape(g["kh"], g["kw"], -1)
        xp = np.pad(x, ((0, 0), (g["ph"], g["ph"]), (g["pw"], g["pw"]), (0, 0)))
        out = self.view(L.dst)
        P, Q = out.shape[1], out.shape[2]
        acc = np.zeros(out.shape, np.float32)
        for r in range(g["kh"]):
            for s in range(g["kw"]):
                acc += xp[:, r:r + P * g["sh"]:g["sh"], s:s + Q * g["sw"]:g["sw"], :] * taps[r, s]
        self.store(out, self.epilogue(L, acc))

    def do_dwse(self, L):
        """depthwise conv + epilogue -> 16-bit tile -> SE gate (rounded) -> tile * gate."""
        g = L.geom
        x = self.view(L.src)
        taps = self.p.blobs[L.blobs["weight"]].reshape(g["kh"], g["kw"], -1)
        xp = np.pad(x, ((0, 0), (g["ph"], g["ph"]), (g["pw"], g["pw"]), (0, 0)))
        P, Q = self.view(L.dst).shape[1:3]
        acc = np.zeros((x.shape[0], P, Q, x.shape[3]), np.float32)
        for r in range(g["kh"]):
            for s in range(g["kw"]):
                acc += xp[:, r:r + P * g["sh"]:g["sh"], s:s + Q * g["sw"]:g["sw"], :] * taps[r, s]
        e = L.epi
        if e.alpha is not None:
            acc = acc * e.alpha
        if e.beta is not None:
            acc = acc + e.beta
        t = _act(e.act1, acc)
        t = self.q(t) if self.round else t
        pooled = t.mean(axis=(1, 2))
        w1 = storage_bits_to_f32(self.p.blobs[L.blobs["w1"]], self.p.precision).reshape(g["c"], g["cr"])
        w2 = storage_bits_to_f32(self.p.blobs[L.blobs["w2"]], self.p.precision).reshape(g["c"], g["cr"])
        h = pooled @ w1
        if "b1" in L.blobs:
            h = h + self.p.blobs[L.blobs["b1"]][:h.shape[1]]
        h = _act(g["act1"], h)
        gate = h @ w2.T
        if "b2" in L.blobs:
            gate = gate + self.p.blobs[L.blobs["b2"]][:gate.shape[1]]
        gate = _act(g["act2"], gate)
        gate = self.q(gate) if self.round else gate
        self.store(self.view(L.dst), t * gate[:, None, None, :])

    def do_pool(self, L):
        g = L.geom
        x = self.view(L.src)
        fill = -np.inf if g["is_max"] else 0.0
        xp = np.pad(x, ((0, 0), (g["ph"], g["ph"]), (g["pw"], g["pw"]), (0, 0)), constant_values=fill)
        ones = np.pad(np.ones(x.shape[1:3]), ((g["ph"], g["ph"]), (g["pw"], g["pw"])))
        out = self.view(L.dst)
        P, Q = out.shape[1], out.shape[2]
        acc, cnt = None, np.zeros((P, Q))
        for r in range(g["kh"]):
            for s in range(g["kw"]):
                win = xp[:, r:r + P * g["sh"]:g["sh"], s:s + Q * g["sw"]:g["sw"], :]
                cnt += ones[r:r + P * g["sh"]:g["sh"], s:s + Q * g["sw"]:g["sw"]]
                acc = win.copy() if acc is None else (np.maximum(acc, win) if g["is_max"] else acc + win)
        if not g["is_max"]:
            div = g["kh"] * g["kw"] if g["cip"] else cnt
            acc = acc / (div if np.isscalar(div) else div[None, :, :, None])
        self.store(out, acc)

    def do_gap(self, L):
        x = self.view(L.src)
        self.store(self.view(L.dst), x.mean(axis=(1, 2), keepdims=True))

    def do_se(self, L):
        g = L.geom
        x = self.view(L.src)                                   # (n, h, w, c)
        pooled = x.astype(np.float64).mean(axis=(1, 2))
        w1 = storage_bits_to_f32(self.p.blobs[L.blobs["w1"]], self.p.precision).reshape(g["c"], g["cr"]).T
        w2 = storage_bits_to_f32(self.p.blobs[L.blobs["w2"]], self.p.precision).reshape(g["c"], g["cr"])
        h = pooled @ w1.T.astype(np.float64)
        if "b1" in L.blobs:
            h = h + self.p.blobs[L.blobs["b1"]][:g["cr"]]
        h = _act(g["act1"], h.astype(np.float32))
        o = h.astype(np.float64) @ w2.T.astype(np.float64)
        if "b2" in L.blobs:
            o = o + self.p.blobs[L.blobs["b2"]][:g["c"]]
        o = _act(g["act2"], o.astype(np.float32))
        if g.get("apply"):                                     # fused channel_scale
            self.store(self.view(L.dst), x * o[:, None, None, :])
        else:
            self.store(self.view(L.dst), o[:, None, None, :])

    def do_ln(self, L):
        x = self.view(L.src).astype(np.float64)             # (n, 1, L, c)
        dst = self.view(L.dst)
        rows = dst.shape[2] if dst.ndim == 4 else 1
        x = x[:, :, :rows, :]
        if L.geom["norm"]:
            mu = x.mean(axis=-1, keepdims=True)
            var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
            g = self.p.blobs[L.blobs["gamma"]][:x.shape[-1]]
            b = self.p.blobs[L.blobs["beta"]][:x.shape[-1]]
            x = (x - mu) / np.sqrt(var + L.geom["eps"]) * g + b
        self.store(dst, x.reshape(dst.shape).astype(np.float32))

    def do_tokens(self, L):
        x = self.view(L.src)                                 # (n, h, w, c)
        n, h, w, c = x.shape
        cls = self.p.blobs[L.blobs["class_token"]][:c]
        pos = self.p.blobs[L.blobs["pos_embedding"]][:(1 + h * w) * c].reshape(1 + h * w, c)
        t = np.concatenate([np.broadcast_to(cls, (n, 1, c)), x.reshape(n, h * w, c)], axis=1) + pos
        self.store(self.view(L.dst), t[:, None].astype(np.float32))

    def do_attn(self, L):
        x = self.view(L.src)[:, 0].astype(np.float64)       # (n, L, 3c)
        heads, c = L.geom["heads"], L.geom["c"]
        d = c // heads
        outs = []
        for hd in range(heads):
            q, k, v = (x[..., j * c + hd * d:j * c + (hd + 1) * d] for j in range(3))
            s = q @ np.swapaxes(k, 1, 2) / np.sqrt(d)
            s = np.exp(s - s.max(axis=-1, keepdims=True))
            outs.append((s / s.sum(axis=-1, keepdims=True)) @ v)
        self.store(self.view(L.dst), np.concatenate(outs, axis=-1)[:, None].astype(np.float32))

    def do_ew(self, L):
        self.store(self.view(L.dst), self.epilogue(L, self.view(L.src)))

    def do_copy(self, L):
        cv = self.p.values[L.geom["concat"]]
        b = self.p.buffers[cv.buf]
        base = self.plan.offsets[cv.buf] // 2
        full = self.arena[base:base + self.n * cv.h * cv.w * b.pitch].reshape(self.n, cv.h, cv.w, b.pitch)
        src = self.view(L.src)
        off = L.geom["coff"]
        full[..., off:off + src.shape[3]] = src
