"""Multi-replica host logic under gloo, world_size 2, on CPU.

Covers the N>1 path of bench.py without GPUs: the packed weight arena built on
rank 0 is broadcast and must be byte-identical to what every rank packs
itself; request batches are sharded per member and the gathered per-replica
logits (computed here by the CPU emulator of the lowered program) equal the
unsharded run.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2410_21120_b200.replicas import shard_rows  # noqa: E402


def test_shard_rows_partitions():
    for batch in (0, 1, 5, 32, 33):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_rows(batch, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    assert [shard_rows(32, r, 2) for r in range(2)] == [(0, 16), (16, 32)]
    assert shard_rows(32, 3, 8) == (12, 16)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from paper_2410_21120_b200.replicas import ReplicaGroup, measure_sharded
    rg = ReplicaGroup("gloo")
    try:
        from conftest import corpus_models
        from paper_2410_21120_b200.device import arena_layout, fill_arena
        from paper_2410_21120_b200.lower import lower_member
        from paper_2410_21120_b200.replicas import arena_digest, shard_inputs
        from program_emulator import Emulator

        models = corpus_models()[40:43]
        progs = [lower_member(g, w) for g, w in models]
        layout, _, total = arena_layout(progs)
        own = np.zeros(total, np.uint8)
        fill_arena(own, progs, layout)
        buf = own.copy() if rank == 0 else np.zeros(total, np.uint8)
        got = rg.broadcast_bytes(buf, src=0)
        ok_arena = arena_digest(got) == arena_digest(own)

        rng = np.random.default_rng(7)
        batches = [rng.standard_normal((5,) + g.input_spec.dims).astype(np.float32) for g, _ in models]
        mine = shard_inputs(batches, rank, world)
        local = [Emulator(p, len(x)).run(x) if len(x) else np.zeros((0, int(np.prod(p.output_dims))), np.float32)
                 for p, x in zip(progs, mine)]
        full = rg.gather(local)
        ref = [Emulator(p, len(x)).run(x) for p, x in zip(progs, batches)]
        ok_out = all(np.allclose(a, b, rtol=1e-6, atol=1e-6) for a, b in zip(full, ref))
        # bench.py's configs[2] timing: batch 32 sharded 16/16, the step time is the
        # slowest rank's (rank 1 reports 2 ms per step here, rank 0 1 ms)
        seen = []

        def run_rows(start, stop, steps):
            seen.append((start, stop))
            return [1.0 + rank] * steps
        rec = measure_sharded(rg, run_rows, 32, steps=4)
        ok_timing = (seen == [(16 * rank, 16 * rank + 16)] and rec["ms_per_step"] == 2.0
                     and rec["rows_per_rank"] == [16, 16] and rec["local_ms_per_step"] == 1.0 + rank
                     and rg.sum(1) == world)
        q.put((rank, ok_arena, ok_out and ok_timing))
    finally:
        dist.destroy_process_group()


def test_bench_launcher_command():
    """bench.py --gpus N outside torchrun spawns N ranks on 127.0.0.1."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    cmd = bench.torchrun_cmd(4, 29555, ["--gpus", "4", "--steps", "10"])
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "10"] and cmd[-5].endswith("bench.py")


def test_gloo_two_replicas_broadcast_and_shard():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = sorted(q.get(timeout=10) for _ in procs)
    assert [r[0] for r in results] == [0, 1]
    assert all(r[1] for r in results), results
    assert all(r[2] for r in results), results
