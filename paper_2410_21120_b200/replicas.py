"""Multi-GPU replicas of one fused DAG (one process per GPU).

The path shards by request: every replica holds the whole
fused DAG and serves a contiguous slice of each member's batch (configs[2]
splits batch 32 as 16/8/4 per replica at 2/4/8 GPUs).  The one exchange is at
swap-in: the rank that did the single pinned H2D broadcasts the packed weight
arena to the others over NCCL (NVLink 5 / NVSwitch, zero-copy on the arena's
device pointer); a swap re-broadcasts only the incoming member's segment.
Queries need no collective; a caller that wants every rank's logits gathers
them (``execute_sharded``).

The host logic (sharding, max-over-ranks timing, gathers, byte broadcasts)
is backend-agnostic and runs under ``gloo`` on CPU in
tests/test_replicas_cpu.py; bench.py drives the same code with NCCL.
"""

from __future__ import annotations

import hashlib
import os
import time

import numpy as np


def shard_rows(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) rows of a batch for ``rank``; sizes differ by <= 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError((rank, world))
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_inputs(batches: list, rank: int, world: int) -> list:
    """Each member's batch split independently (mixed per-member batch sizes)."""
    return [b[slice(*shard_rows(len(b), rank, world))] for b in batches]


def arena_digest(buf) -> str:
    return hashlib.sha256(memoryview(np.ascontiguousarray(buf)).cast("B")).hexdigest()


class ReplicaGroup:
    """This process's place among the replicas (RANK / WORLD_SIZE / LOCAL_RANK
    from the environment, as torchrun sets them).  World 1 needs no
    torch.distributed at all."""

    def __init__(self, backend: str | None = None):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = None
        self.dist = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            if backend is None:
                backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(self.local_rank)
            if not dist.is_initialized():
                dist.init_process_group(backend)
            self.backend, self.dist = dist.get_backend(), dist

    # ---- plumbing
    def _tensor(self, values, dtype=None):
        import torch
        t = torch.tensor(values, dtype=dtype or torch.float64)
        return t.cuda(self.local_rank) if self.backend == "nccl" else t

    def barrier(self) -> None:
        if self.dist is not None:
            if self.backend == "nccl":
                import torch
                torch.cuda.synchronize(self.local_rank)
            self.dist.barrier()

    def max(self, x: float) -> float:
        """Max over ranks (multi-GPU timings are the slowest rank's)."""
        if self.dist is None:
            return float(x)
        t = self._tensor([float(x)])
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.dist is None:
            return float(x)
        t = self._tensor([float(x)])
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def rows(self, batch: int) -> tuple[int, int]:
        return shard_rows(batch, self.rank, self.world)

    def gather(self, local: list) -> list:
        """Concatenate every rank's per-member row slices in rank order."""
        if self.dist is None:
            return [np.asarray(x) for x in local]
        parts: list = [None] * self.world
        self.dist.all_gather_object(parts, [np.asarray(x) for x in local])
        return [np.concatenate([p[m] for p in parts], axis=0) for m in range(len(local))]

    def broadcast_bytes(self, buf: np.ndarray, src: int = 0) -> np.ndarray:
        """Broadcast a host uint8 buffer (gloo; with NCCL through a device copy)."""
        if self.dist is None:
            return buf
        import torch
        t = torch.from_numpy(np.ascontiguousarray(buf, dtype=np.uint8))
        if self.backend == "nccl":
            t = t.cuda(self.local_rank)
        self.dist.broadcast(t, src=src)
        return t.cpu().numpy()

    # ---- the fused DAG on every replica
    def broadcast_device(self, ptr: int, nbytes: int, device: int, src: int = 0) -> float:
        """ncclBroadcast of ``nbytes`` at device address ``ptr`` (zero-copy via
        __cuda_array_interface__); returns the slowest rank's wall ms, from a
        barrier to the broadcast's completion on every rank."""
        import torch

        class _Iface:
            def __init__(self, p, n):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (p, False),
                                                 "version": 3}

        t = torch.as_tensor(_Iface(ptr, nbytes), device=f"cuda:{device}")
        self.barrier()
        t0 = time.perf_counter()
        self.dist.broadcast(t, src=src)
        torch.cuda.synchronize(device)
        return self.max((time.perf_counter() - t0) * 1e3)

    def load(self, dag, precision: str = "fp16", mode: str = "concurrent", src: int = 0):
        """Swap ``dag`` into every replica: rank ``src`` packs and uploads the arena
        (one allocation, one H2D), the others allocate and receive it by one NCCL
        broadcast.  Binds the image to ``dag`` on every rank; returns
        (DeviceDag, {"h2d_ms", "broadcast_ms", "bytes"})."""
        from . import fuse
        from .device import DeviceDag, WeightArena, program_for
        members = [(sg, sg.weight_binding) for sg in dag.subgraphs]
        programs = [program_for(g, w, precision) for g, w in members]
        arena = WeightArena(programs, self.local_rank)
        stats = {"bytes": arena.total, "h2d_ms": None, "broadcast_ms": None}
        if self.rank == src or self.world == 1:
            arena.upload()
            stats["h2d_ms"] = arena.upload_ms
        else:
            arena.allocate()
        if self.world > 1:
            stats["broadcast_ms"] = self.broadcast_device(arena.dev, arena.total, self.local_rank, src)
        img = DeviceDag(members, self.local_rank, mode, arena=arena, programs=programs, precision=precision)
        fuse.attach_image(dag, img)
        return img, stats

    def swap(self, dag, out_id: str, incoming, src: int = 0):
        """swap_subgraph on every replica: rank ``src`` uploads the incoming
        member's segment, the others receive only that segment by broadcast."""
        from . import fuse
        new = fuse._swap(dag, out_id, incoming, upload=(self.rank == src or self.world == 1))
        img = fuse.device_image(new)
        if self.world > 1:
            idx = [sg.model_id for sg in new.subgraphs].index(incoming[0].model_id)
            ptr, nbytes = img.arena.segment(idx)
            img.last_swap = dict(img.last_swap or {}, broadcast_ms=self.broadcast_device(
                ptr, nbytes, self.local_rank, src))
        return new

    def execute_sharded(self, dag, inputs: dict) -> dict:
        """execute_fused over the replicas: each rank runs its rows of every member's
        batch (a list of Tensors per member), the logits are gathered in rank order
        and every rank returns the whole batch's outputs."""
        from . import fuse
        from .executor import Tensor
        mids = [sg.model_id for sg in dag.subgraphs]
        mine = {m: list(inputs[m])[slice(*self.rows(len(inputs[m])))] for m in mids}
        outs = fuse.execute_fused(dag, mine)
        local = [np.stack([t.values for t in outs[m]]) if outs[m] else
                 np.zeros((0, dag.subgraph(m).output_spec.element_count), np.float32) for m in mids]
        full = self.gather(local)
        return {m: [Tensor(dag.subgraph(m).output_spec, r) for r in f] for m, f in zip(mids, full)}


def measure_sharded(rg: ReplicaGroup, run_rows, global_batch: int, steps: int) -> dict:
    """configs[2]-style strong scaling: a global batch per member sharded over the
    replicas.  ``run_rows(start, stop, steps)`` runs this rank's rows ``steps``
    times and returns the device-timed ms of each step; the job's step time is
    the slowest rank's.  Returns the bench record."""
    start, stop = rg.rows(global_batch)
    rg.barrier()
    ms = run_rows(start, stop, steps)
    local = float(np.sum(ms))
    total = rg.max(local)
    return {"global_batch_per_member": global_batch, "world": rg.world,
            "rows_per_rank": [b - a for a, b in (shard_rows(global_batch, r, rg.world) for r in range(rg.world))],
            "ms_per_step": total / steps, "local_ms_per_step": local / steps, "steps": steps}
