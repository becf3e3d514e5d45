"""Table V of the paper ("individual model swaps
in a DAG") replayed on the B200 through the manager's run_swap_schedule
(the reference's scheduler.py:438-546 control flow, manager.py), fused vs
unfused, with the zoo's real architectures.

The paper's DAG: VGG-19-BN, ResNet-50, MobileNetV3-L, ResNeXt-50, MNASNet; one
member swapped every 25 iterations (5 swaps, 150 iterations).  The zoo has 8
architectures, so the replay keeps the shape of the experiment with them:

  start  vgg16, resnet50, mobilenet_v3_large, densenet161, resnet152
  @25    vgg16 -> efficientnet_v2_l         (the paper's swap 1: VGG-19 -> EfficientNetV2)
  @50    resnet50 -> inception_v3           (swap 2: ResNet-50 -> Inception v3)
  @75    densenet161 -> vgg16
  @100   mobilenet_v3_large -> resnet50
  @125   resnet152 -> densenet161

Every iteration is launched (replay_iterations), batch 1 per member; every model
is lowered once before either run (cached programs), so loads and swaps time the
device work: allocation, copies, graph build.  Per segment:
measured device footprint (cudaMemGetInfo), cumulative time; per swap: the
measured swap time (fused: the incoming member's segment -- one allocation + one
H2D -- and a graph rebuild; unfused: the incoming model's image load).
Writes gpurun_out/table5_replay.json.
"""

import json
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2410_21120_b200 import costmodel, manager, zoo  # noqa: E402
from paper_2410_21120_b200.repo import Repository  # noqa: E402

START = ["vgg16", "resnet50", "mobilenet_v3_large", "densenet161", "resnet152"]
SWAPS = [(25, "vgg16", "efficientnet_v2_l"), (50, "resnet50", "inception_v3"), (75, "densenet161", "vgg16"),
         (100, "mobilenet_v3_large", "resnet50"), (125, "resnet152", "densenet161")]
SEG = 25


def main():
    ct = costmodel.DEFAULT_COST_TABLE
    out = {"config": "Table V replay (PAPER.md:383-403) with zoo models, batch 1, 25 iterations per segment",
           "start": START, "swaps": SWAPS}
    with tempfile.TemporaryDirectory() as td:
        repo = Repository(Path(td) / "repo", ct)
        names = sorted(set(START) | {s[2] for s in SWAPS})
        for n in names:
            g, w = zoo.build(n)
            repo.register_model(g, w)
        # lower + pack every model once up front (the program cache): both modes then
        # measure the same load work (allocation, H2D, graph build), not who lowered first
        from paper_2410_21120_b200.device import program_for, stage_segment
        for n in names:
            stage_segment(program_for(*repo.load_pair(n)))      # lowered, packed, pinned once
        steps = [manager.SwapStep(a, o, i) for a, o, i in SWAPS]
        for mode in (manager.FUSED, manager.UNFUSED):
            t0 = time.perf_counter()
            log, recs = manager.run_swap_schedule(START, steps, SEG, repo, ct, mode, 1e9,
                                                  replay_iterations=True)
            wall = time.perf_counter() - t0
            swaps = [{"out": e.payload["out"], "in": e.payload["in"], "swap_ms": e.payload["duration_ms"],
                      **{k: e.payload[k] for k in ("segment_upload_ms", "segment_bytes", "malloc_ms", "d2d_ms",
                                                   "memcpy_ms") if k in e.payload}}
                     for e in log.events_of("swap_subgraph")]
            loads = [e.payload["duration_ms"] for e in log.events_of("load")]
            iters = [e.payload["duration_ms"] for e in log.events_of("iterate")]
            out[mode] = {"initial_load_ms": loads[0] if loads else None,
                         "segments": [{"models": list(r.model_ids), "measured_peak_mib": round(r.measured_peak_mib, 1),
                                       "estimate_mib": r.peak_mib, "iterate_ms": round(it, 3),
                                       "cumulative_ms": round(r.cumulative_ms, 3)}
                                      for r, it in zip(recs, iters)],
                         "swaps": swaps, "wall_s": round(wall, 2)}
            print(mode, json.dumps(out[mode])[:2000], flush=True)
    f, u = out[manager.FUSED], out[manager.UNFUSED]
    out["summary"] = [{"segment": i, "fused_mib": a["measured_peak_mib"], "unfused_mib": b["measured_peak_mib"],
                       "fused_cum_ms": a["cumulative_ms"], "unfused_cum_ms": b["cumulative_ms"]}
                      for i, (a, b) in enumerate(zip(f["segments"], u["segments"]))]
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "table5_replay.json").write_text(json.dumps(out, indent=1))
    print(json.dumps(out["summary"], indent=1))


if __name__ == "__main__":
    main()
