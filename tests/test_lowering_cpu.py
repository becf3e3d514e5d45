"""Lowering + planner + weight packing checked on CPU through the program emulator."""

import numpy as np
import pytest

from conftest import golden_input
from oracle.executor_ref import run_fast
from paper_2410_21120_b200.lower import lower_member
from program_emulator import Emulator


def _rel(a, b):
    a = a.reshape(len(a), -1)
    b = b.reshape(len(b), -1)
    return (np.abs(a - b).max(axis=1) / np.maximum(np.abs(b).max(axis=1), 1e-30)).max()


def test_corpus_lowering_exact_in_fp32(corpus, corpus_golden):
    """Without bf16 rounding the lowered program equals the reference outputs to fp32 noise."""
    for i, (g, w) in enumerate(corpus):
        prog = lower_member(g, w, keep_f32=True)
        xs = np.stack([golden_input(g.input_spec.dims, 7919 * i + t) for t in range(4)])
        got = Emulator(prog, 4, round_bf16=False).run(xs)
        assert _rel(got, corpus_golden[f"{g.model_id}.y"]) < 1e-5, g.model_id


TOL = 2e-2               # north-star tolerance: per sample ||d||inf / ||ref||inf
BF16_TOL_TOY_MAX = 6e-2  # bf16 storage: worst toy model (random init, near-zero logits)


def test_corpus_lowering_fp16_tolerance(corpus, corpus_golden):
    for i, (g, w) in enumerate(corpus):
        prog = lower_member(g, w)                      # default precision: fp16
        xs = np.stack([golden_input(g.input_spec.dims, 7919 * i + t) for t in range(4)])
        got = Emulator(prog, 4).run(xs)
        assert _rel(got, corpus_golden[f"{g.model_id}.y"]) <= TOL, g.model_id


def test_corpus_lowering_bf16_tolerance(corpus, corpus_golden):
    errs = []
    for i, (g, w) in enumerate(corpus):
        prog = lower_member(g, w, precision="bf16")
        xs = np.stack([golden_input(g.input_spec.dims, 7919 * i + t) for t in range(4)])
        got = Emulator(prog, 4).run(xs)
        errs.append(_rel(got, corpus_golden[f"{g.model_id}.y"]))
    errs = np.array(errs)
    assert (errs <= TOL).mean() >= 0.97, np.sort(errs)[-8:]
    assert errs.max() < BF16_TOL_TOY_MAX


def test_zoo_lowering(zoo, zoo_golden):
    for g, w in zoo:
        prog = lower_member(g, w)
        xs = zoo_golden[f"{g.model_id}.x"]
        got = Emulator(prog, len(xs)).run(xs)
        assert _rel(got, zoo_golden[f"{g.model_id}.y"]) < TOL, g.model_id


def test_launch_counts_show_fusion(corpus):
    """Epilogue fusion + zero-copy concat: fewer launches than compute nodes."""
    nodes = launches = 0
    for g, w in corpus:
        prog = lower_member(g, w)
        nodes += sum(1 for n in g.nodes.values() if n.kind not in ("flatten",))
        launches += len(prog.launches)
    assert launches < nodes


def _tiny_vit(res=32, patch=8, **kw):
    from paper_2410_21120_b200 import zoo
    return zoo.vit_b_16(model_id=f"vit_tiny_{res}_{patch}", res=res, patch=patch, hidden=128,
                        layers=2, heads=2, mlp=256, classes=10, **kw)


@pytest.mark.parametrize("res,patch", [(32, 8), (64, 8), (16, 16)])     # L = 17, 65, 2
def test_token_kinds_lowering(res, patch):
    """ViT kinds (tokens, layernorm(+select), attention, GELU, row-wise dense with
    residual epilogue): exact in fp32, north-star tolerance in fp16/bf16."""
    g, w = _tiny_vit(res, patch)
    xs = np.random.default_rng(res).standard_normal((3, 3, res, res)).astype(np.float32)
    ref = run_fast(g, w, xs)
    got = Emulator(lower_member(g, w, keep_f32=True), 3, round_bf16=False).run(xs)
    assert _rel(got, ref) < 1e-5
    for pr in ("fp16", "bf16"):
        got = Emulator(lower_member(g, w, precision=pr), 3).run(xs)
        assert _rel(got, ref) <= TOL, pr


def test_vit_launch_structure():
    """ViT-B/16: 4 GEMMs + 2 LN + 1 attention per block, residuals and GELU folded
    into GEMM epilogues, final LN computes only the class-token row."""
    from paper_2410_21120_b200 import zoo
    g, w = zoo.build("vit_b_16")
    prog = lower_member(g, w)
    kinds = [L.kind for L in prog.launches]
    assert kinds.count("gemm") == 1 + 12 * 4 + 1
    assert kinds.count("ln") == 12 * 2 + 1 and kinds.count("attn") == 12
    assert "ew" not in kinds and kinds.count("tokens") == 1
    last_ln = [L for L in prog.launches if L.kind == "ln"][-1]
    assert last_ln.dst == "cls" and prog.values["cls"].w == 1


def test_gemm_depthwise_epilogue_plan():
    """Host side of the depthwise epilogue (device.gemm_dw_pairs / plan_member):
    every EfficientNetV2-L MBConv expand conv pairs with its depthwise conv; at
    batch 1 the 14x14 / 7x7 ones (not the 28x28 one) absorb it, 14x14 as 2-CTA
    clusters (one M tile per CTA, no m2), never with split-K; at batch 8 none do."""
    from paper_2410_21120_b200 import device, zoo
    g, w = zoo.build("efficientnet_v2_l")
    prog = lower_member(g, w)
    pairs = device.gemm_dw_pairs(prog)
    assert len(pairs) == 61
    by_index = {L.index: L for L in prog.launches}
    for gi, di in pairs.items():
        assert by_index[gi].kind == "gemm" and by_index[di].kind == "dwconv"
        assert by_index[di].src == by_index[gi].dst
    p1 = device.plan_member(prog, 1, 148, True)
    assert len(p1.skip) == 60 and p1.skip <= set(pairs.values())
    fused = [t for t in p1.tilings.values() if t.get("dw") is not None]
    assert len(fused) == 60
    for t in fused:
        assert t["splits"] == 1 and not t["csplit"] and t["m2"] == 0
        mt = t["mt_n"] * t["mt_p"] * t["mt_q"]
        assert mt in (1, 2) and t["tiles"] == t["nt"] * mt
    assert {t["mt_p"] for t in fused} == {1, 2}
    assert not device.plan_member(prog, 8, 148, True).skip


@pytest.mark.parametrize("name", ["efficientnet_v2_l", "mobilenet_v3_large", "densenet161"])
@pytest.mark.parametrize("n", [1, 2])
def test_plan_never_overlays_a_launch_output_on_its_inputs(name, n):
    """No launch writes bytes it (or another CTA of the same grid) still reads: a
    GEMM carrying a depthwise epilogue writes the depthwise output at ITS index,
    so that buffer must be disjoint from the GEMM's own input (first_fit
    used the depthwise launch's later start and overlaid the two)."""
    from paper_2410_21120_b200 import device, zoo
    g, w = zoo.build(name)
    prog = lower_member(g, w)
    plan = device.plan_member(prog, n, 148, True)
    by_index = {L.index: L for L in prog.launches}

    def rng(vname):
        b = prog.values[vname].buf
        off = plan.offsets[b]
        return off, off + prog.buffers[b].bytes_for(n), b

    checked = 0
    for L in prog.launches:
        if L.index in plan.skip:
            continue
        t = plan.tilings.get(L.index, {})
        dst = by_index[t["dw"]].dst if t.get("dw") is not None else L.dst
        w0, w1, wb = rng(dst if L.kind != "copy" else L.geom["concat"])
        for src in (L.src, L.epi.other):
            if src is None:
                continue
            r0, r1, rb = rng(src)
            if rb == wb:
                continue                  # concat windows of one buffer (disjoint channels)
            assert w1 <= r0 or r1 <= w0, (L.index, L.kind, src, dst)
        checked += t.get("dw") is not None
    if name == "efficientnet_v2_l":
        assert checked == 60 if n == 1 else checked >= 0


def test_group_pairing_is_monotone():
    """Grouped-GEMM pairing (device.ExecInstance._pair_chains): members paired two by
    two, matches strictly increasing in both chains (no cross-chain cycle), most
    matches first, short overlaps below GROUP_MIN ignored."""
    from paper_2410_21120_b200 import device, runtime as rt
    G = rt.OP_GEMM

    def chain(keys):
        return [(rt.OP_IN, None, {})] + [(G, None, {"gkey": k}) for k in keys] + [(rt.OP_OUT, None, {})]
    a = chain("abcdabcdxyz")
    b = chain("abcdabcdabcdabcdxyz")       # a deeper model sharing a's shapes
    c = chain("pqrs")
    d = chain("pq")
    pairs = device.ExecInstance._pair_chains(None, [a, b, c, d])
    assert [(x, y) for x, y, _ in pairs] == [(0, 1)]          # c-d share only 2 < GROUP_MIN
    _, _, mt = pairs[0]
    assert len(mt) == 11
    for (i0, j0), (i1, j1) in zip(mt, mt[1:]):
        assert i1 > i0 and j1 > j0
    for i, j in mt:
        assert a[i][2]["gkey"] == b[j][2]["gkey"]
