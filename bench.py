#!/usr/bin/env python3
"""Benchmark of the fused multi-CNN DAG on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1]): VGG16 + MobileNetV3-L + DenseNet161 +
EfficientNetV2-L fused into one DAG, batch 1 per member, synthetic N(0,1)
3x224x224 inputs, calibrated synthetic weights (zoo/, no checkpoints offline).
One step = one fused query = one image through every member (4 images).

  value   images/s of the whole job, device-timed with CUDA events per step
          (inputs resident in HBM); the weights (587 MB packed) exceed the
          126 MB L2, and an L2-flush write of 256 MB runs between timed steps
          outside the events
  e2e     the same metric through the public API ``execute_fused`` with host
          Tensors: pinned H2D of the inputs, graph, D2H of the logits
  + swap-in (one arena, one H2D) vs the unfused per-tensor loader, peak HBM
    fused vs unfused, per-kernel-class roofline, CPU oracle baseline.

Usage: python bench.py [--gpus N --steps K --warmup W] [--impl reference]
N>1 runs under torchrun: rank 0 does the single H2D, the arena is broadcast
over NCCL, every rank runs its own queries (weak scaling), time = max over
ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_PATH = ROOT / "MEASURED_PEAKS.json"
NVLINK_GBS = 900.0          # NVLink 5 per GPU per direction (NVSwitch: full bandwidth to every peer)
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    try:
        d = json.loads(PEAKS_PATH.read_text())
        return d, "measured"
    except Exception:  # noqa: BLE001
        return FALLBACK_PEAKS, "fallback"


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """SM clock + clock-event reasons sampled DURING the timed region.

    NVML (pynvml) polled every ~2 ms from a thread; falls back to
    ``nvidia-smi -lms 20`` when NVML is unavailable."""

    REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc, self.stop_flag = index, [], None, False
        self.thread = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(index)
            self.bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                         "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                         "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                         "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def start(self):
        self.stop_flag = False
        if self.nv is not None:
            def poll():
                nv = self.nv
                while not self.stop_flag:
                    sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    self.rows.append((sm, [n for n, b in self.bits.items() if rs & b]))
                    time.sleep(0.002)
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            p = [x.strip() for x in line.split(",")]
            if len(p) == 6 and p[0].isdigit():
                self.max_mhz = float(p[1])
                self.rows.append((float(p[0]), [n for n, v in zip(self.REASONS, p[2:]) if v.lower() == "active"]))

    def stop(self):
        self.stop_flag = True
        if self.thread is not None:
            self.thread.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for r in self.rows for n in r[1]})
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(min(sm)),
                "sm_max_mhz": float(getattr(self, "max_mhz", max(sm))), "reasons": reasons,
                "samples": len(self.rows), "source": "nvml" if self.nv is not None else "nvidia-smi"}


# ----------------------------------------------------------------------------- helpers

def build_models(names):
    from paper_2410_21120_b200 import zoo
    return [zoo.build(n) for n in names]


def make_inputs(models, batch, seed=1234):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((batch,) + tuple(g.input_spec.dims)).astype(np.float32) for g, _ in models]


def cpu_port_time(models, xs, budget_s=30.0):
    """The reference algorithm (numpy port, BLAS on all host threads) on a bounded sample."""
    from oracle.executor_ref import run_fast
    t0 = time.perf_counter()
    imgs = 0
    while True:
        for (g, w), x in zip(models, xs):
            run_fast(g, w, x[:1])
            imgs += 1
        el = time.perf_counter() - t0
        if el > budget_s / 3 or imgs >= 4 * len(models):
            return imgs / el, imgs, el


def measure_pinned_h2d(rt, nbytes=1 << 30, reps=5):
    host = rt.host_alloc(nbytes)
    dev = rt.malloc(nbytes)
    s = rt.stream_create()
    best = float("inf")
    for _ in range(reps):
        e0, e1 = rt.Event(), rt.Event()
        e0.record(s)
        rt.h2d(dev, host, nbytes, s)
        e1.record(s)
        best = min(best, e0.elapsed_ms(e1))
    rt.free(dev)
    rt.host_free(host)
    rt.stream_destroy(s)
    return nbytes / (best * 1e-3) / 1e9


# ----------------------------------------------------------------------------- reference arm

def reference_executor_sample(x):
    """The UNMODIFIED reference (baseline/_ref, pip-installed from /root/reference/pkg)
    through its own public API: dagfuse.executor.run on VGG16 -- the one north-star
    member made only of the reference's nine kinds -- for one image, on one host
    thread (its fixed-order numpy folds, src/executor.py:56-184).  The model goes
    through the reference's own loaders (JSON graph + FIWT weights written by this
    package's byte-identical writers).  A bounded sample (~20 s) that pins the
    port's speed (the arm's value) to the real reference's."""
    import sys
    import tempfile
    ref_root = Path(__file__).resolve().parent / "baseline" / "_ref"
    if not (ref_root / "dagfuse").is_dir():
        return {"unavailable": "baseline/_ref not installed"}
    sys.path.insert(0, str(ref_root))
    try:
        import dagfuse.executor as rex
        import dagfuse.model_io as rio
        from oracle.executor_ref import run_fast
        from paper_2410_21120_b200 import model_io, zoo
        g, w = zoo.build("vgg16")
        with tempfile.TemporaryDirectory() as td:
            model_io.save_graph(g, Path(td) / "vgg16.graph.json")
            model_io.save_weights(w, Path(td) / "vgg16.weights.fiwt")
            rg = rio.load_graph(Path(td) / "vgg16.graph.json")
            rw = rio.load_weights(Path(td) / "vgg16.weights.fiwt")
        t0 = time.perf_counter()
        y = rex.run(rg, rw, rex.Tensor.from_array(np.asarray(x, np.float32).reshape(g.input_spec.dims)))
        el = time.perf_counter() - t0
        t1 = time.perf_counter()
        port = run_fast(g, w, np.asarray(x, np.float32).reshape((1,) + tuple(g.input_spec.dims)))[0]
        el_port = time.perf_counter() - t1
        ref = np.asarray(y.values, np.float64)
        return {"model": "vgg16", "api": "dagfuse.executor.run (baseline/_ref, unmodified)",
                "s_per_image": el, "images_per_s": 1.0 / el, "threads": 1,
                "port_s_per_image": el_port,
                "port_rel_err_vs_reference": float(np.abs(port - ref).max() / np.abs(ref).max())}
    except Exception as e:                               # report, never fail the arm
        return {"unavailable": f"{type(e).__name__}: {e}"}
    finally:
        sys.path.remove(str(ref_root))


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU algorithm (oracle port) on host cores."""
    if rank != 0:
        return
    from oracle.executor_ref import run_fast
    models = build_models(args.models)
    xs = make_inputs(models, args.batch)
    cores = os.cpu_count() or 1

    # one step = one member's batch, members in rotation: a bounded sample (about a
    # quarter of a fused query) so --steps K of the driver still ends within minutes;
    # images/s is unaffected by the sampling
    k = [0]

    def step():
        (g, w), x = models[k[0] % len(models)], xs[k[0] % len(models)]
        run_fast(g, w, x)
        k[0] += 1

    for _ in range(args.warmup):
        step()
    k[0] = 0
    # whole rotations, so every member weighs equally in the sample
    nsteps = -(-args.steps // len(models)) * len(models)
    t0 = time.perf_counter()
    for _ in range(nsteps):
        step()
    el = time.perf_counter() - t0
    imgs = nsteps * args.batch
    value = imgs / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s",
        "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / nsteps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(args),
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": "port",
                         "sample": f"{nsteps} member batches (members in rotation, whole rotations, batch "
                                   f"{args.batch}) through oracle/executor_ref.run_fast (numpy fp32, "
                                   f"BLAS on {cores} host threads)"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_executor": reference_executor_sample(
            xs[list(args.models).index("vgg16")][0] if "vgg16" in args.models
            else np.random.default_rng(1234).standard_normal((3, 224, 224)).astype(np.float32)),
    }
    print(json.dumps(line), flush=True)


SHARD_BATCH = 32           # configs[2]: per-member batch sharded over the replicas
METRIC = "fused 4-model DAG images/s (batch 1 per member), with latency ms, peak HBM GB, swap-in ms"


def config_dict(args):
    return {"workload": "4-model fused DAG (configs[1])" if args.batch == 1 else
            f"4-model fused DAG, batch {args.batch} per member",
            "models": list(args.models), "batch_per_member": args.batch,
            "input": "3x224x224 fp32 N(0,1)", "precision": args.precision, "mode": args.mode,
            "l2": "weights 587 MB > 126 MB L2; 256 MB L2-flush write between timed steps (untimed)"}


# ----------------------------------------------------------------------------- secondary configs

def time_device_steps(rt, inst, flush, steps, warmup=3, raw=False):
    """Device-timed steps of one instance's graph (L2 flushed between steps);
    (median, mean) ms, or every step's ms with ``raw``."""
    for _ in range(warmup):
        inst.launch_graph()
    inst.sync()
    ms = []
    for _ in range(steps):
        rt.memset(flush, 0, 256 << 20, inst.stream)
        e0, e1 = rt.Event(), rt.Event()
        e0.record(inst.stream)
        inst.launch_graph()
        e1.record(inst.stream)
        ms.append(e0.elapsed_ms(e1))
    inst.sync()
    if raw:
        return ms
    return float(np.median(ms)), float(np.mean(ms))


def gemm_class(inst, tc_peak):
    """Tensor-core view of one instance: GEMM launches replayed alone (profile_nodes)."""
    prof = inst.profile_nodes(reps=4, kinds={"gemm"})
    ms = sum(r["ms"] for r in prof)
    fl = sum(r["flops"] for r in prof)
    best = max(prof, key=lambda r: r["flops"] / r["ms"])
    return {"gemm_launches": len(prof), "gemm_ms": round(ms, 4),
            "gemm_tflops": round(fl / (ms * 1e-3) / 1e12, 1),
            "frac_of_bf16_peak": round(fl / (ms * 1e-3) / 1e12 / tc_peak, 4),
            "best_launch": {"node": best["node"], "tflops": round(best["flops"] / (best["ms"] * 1e-3) / 1e12, 1)}}


def secondary_configs(args, rt, members, programs, arena, flush, P, local_rank):
    """configs[2] (batch 32 on one GPU), configs[3] (swap-in stress) and configs[4]
    (8-model mixed batch) -- measured on the same box after the headline run."""
    from paper_2410_21120_b200.device import DeviceDag, PerTensorArena, WeightArena, program_for
    tc_peak = float(P.get("bf16_tflops", 1590.0))
    out = {}
    # configs[2]: the same fused DAG at batch 32 per member (1 GPU; N>1 shards it over replicas)
    dag = DeviceDag(members, local_rank, args.mode, arena=arena, programs=programs, precision=args.precision)
    b = 32
    inst = dag.acquire(tuple([b] * len(members)))
    inst.upload_inputs(make_inputs([(sg, w) for sg, w in members], b, seed=99))
    med, mean = time_device_steps(rt, inst, flush, steps=20)
    flops = sum(p.gemm_flops_per_sample for p in programs) * b
    out["batch32"] = {"config": "configs[2]: 4-model fused DAG, batch 32 per member, 1 GPU",
                      "ms_per_step": med, "images_per_s": len(members) * b / (med * 1e-3),
                      "step_tflops": round(flops / (med * 1e-3) / 1e12, 1),
                      "step_frac_of_bf16_peak": round(flops / (med * 1e-3) / 1e12 / tc_peak, 4),
                      **gemm_class(inst, tc_peak)}
    dag.free_instances()
    # configs[3]: swap-in stress -- repeated load/unload of the fused arena vs per-model loads
    stress = WeightArena(programs, local_rank)
    fused_ms, fused_copy = [], []
    for _ in range(20):
        stress.upload()
        fused_ms.append(stress.upload_ms)
        fused_copy.append(stress.memcpy_ms)
        stress.unload()
    total = stress.total
    stress.free()
    unf = []
    for _ in range(3):
        pt = PerTensorArena(programs, local_rank)
        unf.append(pt.upload_ms)
        pt.free()
    out["swap_stress"] = {"config": "configs[3]: 20 load/unload cycles of the fused arena vs 3 per-tensor loads",
                          "arena_mb": total / 1e6,
                          "fused_load_ms_median": float(np.median(fused_ms)),
                          "fused_h2d_gbs_median": total / (float(np.median(fused_copy)) * 1e-3) / 1e9,
                          "unfused_load_ms_median": float(np.median(unf)),
                          "speedup": float(np.median(unf) / np.median(fused_ms))}
    # swap-in from disk: the reference's FIWT files -> parse ->
    # lower + pack -> upload, vs one packed-arena file -> pinned read -> ONE H2D
    out["swap_from_disk"] = swap_from_disk(args, members)
    out["member_swap"] = member_swaps(args)
    # configs[4]: 8-model fused DAG with mixed per-member batches
    from paper_2410_21120_b200 import zoo
    names = list(zoo.EIGHT_MODEL)
    batches = (1, 2, 4, 8, 1, 2, 4, 8)
    m8 = build_models(names)
    # ViT-B/16's layernorm / token / attention kernels are 16-bit only: the 8-model
    # DAG runs in the split mode's 16-bit plane type (fp16x2 -> fp16)
    prec8 = args.precision[:4]
    p8 = [program_for(g, w, prec8) for g, w in m8]
    rt.pool_trim(0)            # retained arena-pool pages would hide the allocation from cudaMemGetInfo
    free0, _ = rt.mem_info()
    dag8 = DeviceDag(m8, local_rank, args.mode, programs=p8, precision=prec8)
    inst8 = dag8.acquire(batches)
    inst8.upload_inputs([np.random.default_rng(7 + i).standard_normal((bb,) + tuple(g.input_spec.dims))
                         .astype(np.float32) for i, (bb, (g, _)) in enumerate(zip(batches, m8))])
    med8, _ = time_device_steps(rt, inst8, flush, steps=20)
    free1, _ = rt.mem_info()
    out["eight_model"] = {"config": "configs[4]: 8-model fused DAG, per-member batches "
                                    + ",".join(f"{n}:{bb}" for n, bb in zip(names, batches)),
                          "precision": prec8,
                          "ms_per_step": med8, "images_per_s": sum(batches) / (med8 * 1e-3),
                          "arena_mb": dag8.arena.total / 1e6, "swap_in_ms": dag8.swap_in_ms,
                          "peak_hbm_gb": (free0 - free1) / 1e9, "graph_nodes": inst8.kernel_nodes}
    dag8.free_instances()
    dag8.arena.free()
    return out


def accuracy_modes(args, models, flush, P, local_rank, modes=("fp16x2", "bf16x2", "fp16", "bf16")):
    """The same configs[1] / configs[2] workloads in the other storage precisions
    (the headline line is args.precision): the split modes fp16x2 / bf16x2 (two
    16-bit planes per value, three-product GEMMs) are the ones that meet the full
    north-star parity bar -- identical top-1 on >= 99.9 % of 1000 inputs, raw
    (tests/test_gpu_north_star.py; statistic in profiles/r02/parity_*.json); the
    16-bit fp16 / bf16 modes are the fast ones (within 2e-2 / 1e-1, top-1 only
    where the fp32 margin exceeds the error).
    Each: device-timed batch-1 and batch-32 steps, e2e through execute_fused with
    host tensors, and the logits of one image per member against the CPU oracle."""
    from oracle.executor_ref import run_fast
    from paper_2410_21120_b200 import fuse, runtime as rt
    from paper_2410_21120_b200.executor import Tensor
    out = {}
    xs1 = make_inputs(models, 1, seed=1234)
    xs32 = make_inputs(models, SHARD_BATCH, seed=99)
    refs = [run_fast(g, w, x[:1])[0] for (g, w), x in zip(models, xs1)]
    for prec in modes:
        if prec == args.precision:
            continue
        dag = fuse.fuse_models(models)
        img = fuse.load_fused(dag, local_rank, args.mode, precision=prec)
        inst = img.acquire(tuple([1] * len(models)))
        inst.upload_inputs(xs1)
        med1, _ = time_device_steps(rt, inst, flush, steps=max(20, min(args.steps, 100)))
        img.release(inst)
        inst = img.acquire(tuple([SHARD_BATCH] * len(models)))
        inst.upload_inputs(xs32)
        med32, _ = time_device_steps(rt, inst, flush, steps=20)
        img.release(inst)
        host = {sg.model_id: Tensor(sg.input_spec, x[0]) for sg, x in zip(dag.subgraphs, xs1)}
        for _ in range(3):
            outs = fuse.execute_fused(dag, host)
        n = max(20, min(args.steps, 100))
        t0 = time.perf_counter()
        for _ in range(n):
            outs = fuse.execute_fused(dag, host)
        e2e_ms = (time.perf_counter() - t0) / n * 1e3
        err = {sg.model_id: float(np.abs(outs[sg.model_id].values - r).max() / np.abs(r).max())
               for sg, r in zip(dag.subgraphs, refs)}
        out[prec] = {"ms_per_step": med1, "images_per_s": len(models) / (med1 * 1e-3),
                     "e2e_ms_per_step": e2e_ms, "e2e_images_per_s": len(models) / (e2e_ms * 1e-3),
                     "batch32_ms_per_step": med32,
                     "batch32_images_per_s": len(models) * SHARD_BATCH / (med32 * 1e-3),
                     "arena_mb": img.arena.total / 1e6, "parity_rel_err": err,
                     "north_star_statistic": f"profiles/r02/parity_{{0,1,2}}_{prec}.json"}
        fuse.unload(dag)
    return out


def member_swaps(args):
    """swap_subgraph on the resident 4-model DAG (the measured replacement of the
    reference's simulate_swap, costmodel.py:308-338): each member in turn replaced by
    ResNet-50 and swapped back.  Per swap: the device work (one allocation from the
    arena pool, D2D of the untouched members, ONE H2D of the incoming segment from
    its pinned image) and the whole call (validation, profile of the incoming member,
    DAG rebuild); incoming programs are lowered and pinned once beforehand."""
    from paper_2410_21120_b200 import fuse, zoo
    from paper_2410_21120_b200.device import program_for, stage_segment
    models = build_models(args.models)
    incoming = zoo.build("resnet50")
    for g, w in models + [incoming]:
        stage_segment(program_for(g, w, args.precision))
    dag = fuse.fuse_models(models)
    fuse.load_fused(dag, precision=args.precision)
    rows = []
    for (g, w) in models:
        for out_id, inc in ((g.model_id, incoming), (incoming[0].model_id, (g, w))):
            t0 = time.perf_counter()
            new = fuse.swap_subgraph(dag, out_id, inc)
            wall = (time.perf_counter() - t0) * 1e3
            ls = fuse.device_image(new).last_swap
            fuse.unload(dag)
            dag = new
            rows.append({"out": out_id, "in": inc[0].model_id, "segment_mb": ls["bytes"] / 1e6,
                         "device_ms": ls["ms"], "malloc_ms": ls["malloc_ms"], "d2d_ms": ls["d2d_ms"],
                         "h2d_ms": ls["memcpy_ms"], "call_ms": wall})
    fuse.unload(dag)
    return {"config": "each north-star member swapped out for ResNet-50 and back on the loaded DAG",
            "precision": args.precision, "swaps": rows,
            "device_ms_median": float(np.median([r["device_ms"] for r in rows])),
            "call_ms_median": float(np.median([r["call_ms"] for r in rows]))}


def swap_from_disk(args, members):
    import tempfile
    from paper_2410_21120_b200 import fuse, model_io, pack_io, runtime as rt
    with tempfile.TemporaryDirectory(dir="/tmp") as td:
        td = Path(td)
        graphs = [fuse._as_graph(sg) for sg, _ in members]
        for g, (_, w) in zip(graphs, members):                     # untimed: write the files
            model_io.save_graph(g, td / f"{g.model_id}.graph.json")
            model_io.save_weights(w, td / f"{g.model_id}.weights.fiwt")
        fiwt_bytes = sum((td / f"{g.model_id}.weights.fiwt").stat().st_size for g in graphs)
        pack_io.save_packed(fuse.fuse_models([(g, w) for g, (_, w) in zip(graphs, members)]),
                            td / "dag.dfxpack", precision=args.precision)
        import gc
        gc.collect()
        t0 = time.perf_counter()
        pairs = [(model_io.load_graph(td / f"{g.model_id}.graph.json"),
                  model_io.load_weights(td / f"{g.model_id}.weights.fiwt")) for g in graphs]
        t1 = time.perf_counter()
        d = fuse.fuse_models(pairs)
        img = fuse.load_fused(d, precision=args.precision)
        fiwt_ms = (time.perf_counter() - t0) * 1e3
        parse_ms = (t1 - t0) * 1e3
        fuse.unload(d)
        img.arena.free()
        del pairs, d, img
        gc.collect()                         # the FIWT path's 1.2 GB of arrays, freed untimed
        t0 = time.perf_counter()
        dp = pack_io.load_packed(td / "dag.dfxpack")
        packed_ms = (time.perf_counter() - t0) * 1e3
        a = fuse.device_image(dp).arena
        res = {"config": "4-model DAG swapped in from files on the box's /tmp (page cache warm: "
                         "the files were just written)",
               "fiwt_mb": fiwt_bytes / 1e6, "fiwt_load_ms": fiwt_ms, "fiwt_parse_ms": parse_ms,
               "packed_mb": (td / "dag.dfxpack").stat().st_size / 1e6, "packed_load_ms": packed_ms,
               "packed_phases_ms": {k: round(getattr(a, k + "_ms"), 2) for k in
                                    ("header", "alloc", "read", "malloc", "memcpy", "dag")},
               "speedup": fiwt_ms / packed_ms}
        fuse.unload(dp)
        a.free()
    return res


def ncu_traffic():
    """dram bytes per GEMM launch from the committed ncu capture of this workload
    (profiles/*traffic*.json, written by scripts/summarize_profiles.py), else None."""
    for f in sorted((ROOT / "profiles").glob("*traffic*.json"), reverse=True):
        try:
            d = json.loads(f.read_text())
            return d.get("dram_bytes_per_gemm_launch"), f.name, d.get("note")
        except Exception:  # noqa: BLE001
            continue
    return None, None, None


# ----------------------------------------------------------------------------- our arm

def run_ours(args):
    from paper_2410_21120_b200 import fuse, runtime as rt
    from paper_2410_21120_b200.device import DeviceDag, PerTensorArena, WeightArena, program_for
    from paper_2410_21120_b200.executor import Tensor
    from paper_2410_21120_b200.replicas import ReplicaGroup, measure_sharded

    rg = ReplicaGroup()                       # NCCL process group when WORLD_SIZE > 1
    world, rank, local_rank = rg.world, rg.rank, rg.local_rank
    rt.init_device(local_rank)
    P, peak_kind = peaks()

    models = build_models(args.models)
    dag = fuse.fuse_models(models)
    members = [(sg, sg.weight_binding) for sg in dag.subgraphs]
    programs = [program_for(g, w, args.precision) for g, w in members]

    # ---------------- unfused baseline: per-tensor loads, per-model graphs run one after another
    unfused = None
    if not args.skip_unfused and world == 1:
        # pinned per-tensor A/B (consolidation vs pinning): median of 3 loads, freed
        pinned_loads = []
        for _ in range(3):
            ptp = PerTensorArena(programs, local_rank, pinned=True)
            pinned_loads.append((ptp.upload_ms, ptp.malloc_ms, ptp.memcpy_ms))
            ptp.free()
        free_u0, _ = rt.mem_info()
        # pageable per-tensor loads (the framework default): median of 3, the first of a
        # fresh process pays one-time driver costs (reported apart); the last one stays
        loads = []
        for i in range(3):
            pt = PerTensorArena(programs, local_rank)
            loads.append((pt.upload_ms, pt.malloc_ms, pt.memcpy_ms))
            if i < 2:
                pt.free()
        first_unfused_ms = loads[0][0]
        pt.upload_ms, pt.malloc_ms, pt.memcpy_ms = sorted(loads)[1]
        pp = sorted(pinned_loads)[1]
        solos = [DeviceDag([m], local_rank, "sequential", arena=_SubArena(pt, i), programs=[p],
                           precision=args.precision)
                 for i, (m, p) in enumerate(zip(members, programs))]
        insts = [d.acquire((args.batch,)) for d in solos]
        for si, x in zip(insts, make_inputs(models, args.batch, seed=1234 + rank)):
            si.upload_inputs([x])
        free_u1, _ = rt.mem_info()
        u_ms = []
        for _ in range(max(3, args.steps // 2)):
            e0, e1 = rt.Event(), rt.Event()
            e0.record(insts[0].stream)
            for si in insts:          # one model after another, each its own graph
                si.launch_graph()
                si.sync()
            e1.record(insts[-1].stream)
            u_ms.append(e0.elapsed_ms(e1))
        unfused = {"swap_in_ms": pt.upload_ms, "malloc_ms": pt.malloc_ms, "memcpy_ms": pt.memcpy_ms,
                   "weight_tensors": pt.tensors,
                   "first_load_ms": first_unfused_ms,
                   "pinned_per_tensor": {"swap_in_ms": pp[0], "malloc_ms": pp[1], "memcpy_ms": pp[2],
                                         "note": "same per-tensor cudaMalloc + cudaMemcpyAsync, sources "
                                                 "staged in ONE pinned buffer (untimed, as the fused arena's)"},
                   "peak_hbm_gb": (free_u0 - free_u1) / 1e9,
                   "ms_per_query": float(np.median(u_ms)),
                   "note": "per-tensor cudaMalloc+cudaMemcpyAsync from pageable memory (median of 3 "
                           "loads); one CUDA graph per model, launched one after another"}
        for d in solos:
            d.free_instances()
        pt.free()


    # ---------------- swap-in: one pinned arena, ONE H2D (rank 0), NCCL broadcast to replicas
    rt.pool_trim(0)            # the retained arena pool must not hide the allocation from cudaMemGetInfo
    free0, _ = rt.mem_info()
    first_load_ms = None
    arena = WeightArena(programs, local_rank)
    bcast_ms = bcast_first_ms = None
    if world > 1:
        if rank == 0:
            arena.upload()
        else:
            arena.allocate()
        bcast_ms = rg.broadcast_device(arena.dev, arena.total, local_rank, src=0)
        # a second broadcast of the resident arena: the first one includes NCCL's
        # lazy connection setup
        bcast_first_ms, bcast_ms = bcast_ms, rg.broadcast_device(arena.dev, arena.total, local_rank, src=0)
    else:
        # the swap-in reported is the median of 3 load cycles (the first cudaMalloc of
        # a fresh process is occasionally 10-50x slower); the first is reported too
        loads = []
        for i in range(3):
            if i:
                arena.unload()
            arena.upload()
            loads.append((arena.upload_ms, arena.malloc_ms, arena.memcpy_ms))
        first_load_ms = loads[0][0]
        arena.upload_ms, arena.malloc_ms, arena.memcpy_ms = sorted(loads)[1]
    img = DeviceDag(members, local_rank, args.mode, arena=arena, programs=programs,
                    precision=args.precision)
    batch = tuple([args.batch] * len(members))
    inst = img.acquire(batch)
    xs = make_inputs(models, args.batch, seed=1234 + rank)
    inst.upload_inputs(xs)
    inst.launch_graph()
    inst.sync()
    free1, _ = rt.mem_info()
    fused_peak = free0 - free1

    flush = rt.malloc(256 << 20)
    clocks = ClockSampler(local_rank)

    # ---------------- device-timed steps
    for _ in range(args.warmup):
        inst.launch_graph()
    inst.sync()
    rg.barrier()
    clocks.start()
    step_ms = []
    for _ in range(args.steps):
        rt.memset(flush, rank & 0xFF, 256 << 20, inst.stream)       # L2 flush, outside the events
        e0, e1 = rt.Event(), rt.Event()
        e0.record(inst.stream)
        inst.launch_graph()
        e1.record(inst.stream)
        step_ms.append(e0.elapsed_ms(e1))
    inst.sync()
    clk = clocks.stop()
    total_ms = rg.max(float(np.sum(step_ms)))
    imgs_per_step = len(members) * args.batch
    value = world * imgs_per_step * args.steps / (total_ms * 1e-3)
    ms_per_step = total_ms / args.steps

    # ---------------- e2e through the public API (host tensors, pinned H2D + D2H inside)
    fuse.attach_image(dag, img)
    host_inputs = {sg.model_id: ([Tensor(sg.input_spec, x[i]) for i in range(args.batch)]
                                 if args.batch > 1 else Tensor(sg.input_spec, x[0]))
                   for sg, x in zip(dag.subgraphs, xs)}
    for _ in range(max(args.warmup, 1)):
        fuse.execute_fused(dag, host_inputs)
    rg.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        outs = fuse.execute_fused(dag, host_inputs)
    e2e_s = rg.max(time.perf_counter() - t0)
    e2e_value = world * imgs_per_step * args.steps / e2e_s

    # ---------------- configs[2]: batch 32 per member sharded over the replicas (strong
    # scaling; at N=1 the whole batch on one GPU)
    def run_rows(start, stop, steps):
        rows = stop - start
        si = img.acquire(tuple([rows] * len(members)))
        si.upload_inputs([x[start:stop] for x in make_inputs(models, SHARD_BATCH, seed=99)])
        ms = time_device_steps(rt, si, flush, steps=steps, warmup=3, raw=True)
        img.release(si)
        return ms
    sharded = measure_sharded(rg, run_rows, SHARD_BATCH, steps=max(10, min(args.steps, 50)))
    sharded["images_per_s"] = len(members) * SHARD_BATCH / (sharded["ms_per_step"] * 1e-3)
    sharded["config"] = (f"configs[2]: 4-model fused DAG, batch {SHARD_BATCH} per member sharded over "
                         f"{world} replica(s) (rows per rank {sharded['rows_per_rank']}); step time = slowest rank")

    if rank != 0:
        return

    # ---------------- per-kernel-class roofline (eager replay, CUDA events per launch)
    prof = inst.profile_nodes(reps=8)
    classes = {}
    for r in prof:
        c = classes.setdefault(r["kind"], {"ms": 0.0, "bytes": 0, "flops": 0, "launches": 0})
        c["ms"] += r["ms"]
        c["bytes"] += r["bytes"]
        c["flops"] += r["flops"]
        c["launches"] += 1
    eager_total = sum(c["ms"] for c in classes.values())
    dom = max(classes, key=lambda k: classes[k]["ms"])
    g = classes["gemm"]
    gemm_gbs = g["bytes"] / (g["ms"] * 1e-3) / 1e9
    gemm_tflops = g["flops"] / (g["ms"] * 1e-3) / 1e12
    hbm_peak = float(P["hbm_gbs"])
    tc_peak = float(P.get("bf16_tflops", 1590.0))
    hbm_frac, tc_frac = gemm_gbs / hbm_peak, gemm_tflops / tc_peak
    bound = "hbm" if hbm_frac >= tc_frac else "tensor"
    roofline = {
        "kernel": "dfx::gemm_kernel (tcgen05 implicit-GEMM conv/dense, all launches of one step)",
        "bound": bound,
        "achieved": gemm_gbs if bound == "hbm" else gemm_tflops,
        "peak": hbm_peak if bound == "hbm" else tc_peak,
        "unit": "GB/s" if bound == "hbm" else "TFLOP/s",
        "frac": hbm_frac if bound == "hbm" else tc_frac,
        "traffic": None,
        "peak_source": f"MEASURED_PEAKS.json ({peak_kind}; burst figures, kernels timed alone)",
        "other_view": ({"achieved_tflops": gemm_tflops, "frac_of_bf16_peak": tc_frac} if bound == "hbm"
                       else {"achieved_gbs": gemm_gbs, "frac_of_hbm_peak": hbm_frac}),
        "gemm_share_of_eager_step": g["ms"] / eager_total,
        "gemm_launches_per_step": g["launches"],
        "classes": {k: {"ms": round(v["ms"], 4), "launches": v["launches"],
                        "GB/s": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["ms"] else None,
                        "TFLOP/s": round(v["flops"] / (v["ms"] * 1e-3) / 1e12, 2) if v["ms"] else None}
                    for k, v in sorted(classes.items(), key=lambda kv: -kv[1]["ms"])},
        "dominant_class": dom,
    }

    traffic, traffic_src, traffic_note = ncu_traffic()
    roofline["traffic"] = traffic
    roofline["traffic_source"] = traffic_src
    roofline["traffic_note"] = traffic_note
    roofline["algorithmic_bytes_per_gemm_launch"] = g["bytes"] / max(g["launches"], 1)
    extra = modes = None
    if not args.skip_extra and world == 1:
        extra = secondary_configs(args, rt, members, programs, arena, flush, P, local_rank)
    if not args.skip_modes and world == 1:
        modes = accuracy_modes(args, models, flush, P, local_rank)
    h2d_gbs = measure_pinned_h2d(rt)
    cores = os.cpu_count() or 1
    cpu_baseline = None
    if world == 1:            # the CPU baseline runs on rank 0 at N=1 only
        cpu_ips, cpu_imgs, cpu_s = cpu_port_time(models, xs)
        cpu_baseline = {"value": cpu_ips, "unit": "images/s", "cores": cores, "kind": "port",
                        "sample": f"{cpu_imgs} member-images ({cpu_s:.1f} s) through "
                                  f"oracle/executor_ref.run_fast (numpy fp32, BLAS on {cores} threads)"}
    # check the logits of the e2e run against the CPU oracle (4 members, 1 image)
    from oracle.executor_ref import run_fast
    parity = {}
    for (gph, w), sg, x in zip(models, dag.subgraphs, xs):
        ref = run_fast(gph, w, x[:1])[0]
        got = outs[sg.model_id] if args.batch == 1 else outs[sg.model_id][0]
        parity[sg.model_id] = float(np.abs(got.values - ref).max() / np.abs(ref).max())

    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": {"fp16": "f16", "bf16": "bf16", "fp16x2": "f16x2", "bf16x2": "bf16x2"}[args.precision],
        "data": "synthetic (N(0,1) inputs, seeded calibrated random-init weights)",
        "config": config_dict(args),
        "latency_ms": ms_per_step,
        "swap_in": {"fused_ms": arena.upload_ms, "fused_malloc_ms": getattr(arena, "malloc_ms", None),
                    "fused_memcpy_ms": getattr(arena, "memcpy_ms", None),
                    "arena_mb": arena.total / 1e6, "cuda_mallocs": 1, "h2d_copies": 1,
                    "fused_h2d_gbs": (arena.total / (arena.memcpy_ms * 1e-3) / 1e9
                                      if getattr(arena, "memcpy_ms", None) else None),
                    "pinned_h2d_peak_gbs": h2d_gbs,
                    "h2d_frac_of_pinned_peak": (arena.total / (arena.memcpy_ms * 1e-3) / 1e9 / h2d_gbs
                                                if getattr(arena, "memcpy_ms", None) else None),
                    "nccl_broadcast_ms": bcast_ms,
                    "nccl_broadcast_first_ms": bcast_first_ms,
                    "nccl_broadcast_gbs": arena.total / (bcast_ms * 1e-3) / 1e9 if bcast_ms else None,
                    "nccl_broadcast_frac_of_nvlink": (arena.total / (bcast_ms * 1e-3) / 1e9 / NVLINK_GBS
                                                      if bcast_ms else None),
                    "note": "median of 3 load cycles (one allocation from the retained arena pool + one H2D each; first_load_ms maps the pool pages)",
                    "first_load_ms": first_load_ms,
                    "unfused_ms": unfused["swap_in_ms"] if unfused else None,
                    "unfused_malloc_ms": unfused["malloc_ms"] if unfused else None,
                    "unfused_memcpy_ms": unfused["memcpy_ms"] if unfused else None},
        "peak_hbm_gb": {"fused": fused_peak / 1e9, "unfused": unfused["peak_hbm_gb"] if unfused else None},
        "unfused": unfused,
        "e2e": {"value": e2e_value, "unit": "images/s",
                "h2d_bytes_per_step": int(sum(x.nbytes for x in xs)),
                "d2h_bytes_per_step": int(sum(sg.output_spec.element_count * 4 * args.batch
                                              for sg in dag.subgraphs)),
                "ms_per_step": e2e_s / args.steps * 1e3},
        "gpu_launches": inst.kernel_nodes * args.steps,
        "graph_nodes_per_step": inst.kernel_nodes,
        "roofline": roofline,
        "cpu_baseline": cpu_baseline,
        "parity_rel_err": parity,
        # logits that came out inf / NaN during the whole run (fp16 stores do not
        # saturate, so any activation overflow would show here; dfx_nonfinite_count)
        "nonfinite_logits": fuse.nonfinite_outputs(),
        "clocks": clk,
        "sharded_batch32": sharded,
        "other_configs": extra,
        "precision_modes": modes,
    }
    print(json.dumps(line), flush=True)


class _SubArena:
    """One member's view of a PerTensorArena (member index remapped to 0)."""

    def __init__(self, pt, i):
        self.pt, self.i = pt, i
        self.upload_ms = None

    def addr(self, member, key):
        return self.pt.addr(self.i, key)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--batch", type=int, default=1)
    # default: the split fp16x2 storage -- the precision that meets the whole north-star
    # parity bar (<= 2e-2 AND identical top-1 on >= 99.9 % of 1000 inputs, raw); the
    # 16-bit modes are in the line's precision_modes block
    ap.add_argument("--precision", default="fp16x2", choices=("fp16", "bf16", "fp16x2", "bf16x2"))
    ap.add_argument("--mode", default="concurrent", choices=("concurrent", "sequential"))
    ap.add_argument("--models", nargs="+",
                    default=["vgg16", "mobilenet_v3_large", "densenet161", "efficientnet_v2_l"])
    ap.add_argument("--skip-unfused", action="store_true")
    ap.add_argument("--skip-modes", action="store_true",
                    help="skip the other storage precisions (fp16x2 / bf16x2 / bf16) block")
    ap.add_argument("--skip-extra", action="store_true",
                    help="skip configs[2..4] (batch 32, swap stress, 8-model) after the headline")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args)


def torchrun_cmd(n: int, port: int, argv: list[str]) -> list[str]:
    """One process per GPU on this node (rendezvous on 127.0.0.1)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *argv]


def launch_ranks(n: int) -> int:
    """``bench.py --gpus N`` outside torchrun: spawn the N ranks ourselves (rank 0
    prints the JSON line).  NCCL init logging stays on so the communicator's
    nranks is visible in stderr."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(torchrun_cmd(n, port, sys.argv[1:]), env=env)


if __name__ == "__main__":
    main()
