"""Multi-GPU replicas of one fused DAG (one process per GPU).

The path shards by request: every replica holds the whole DAG and serves a
contiguous slice of each member's batch (C3 splits batch 32
as 16/8/4 per replica at 2/4/8 GPUs).  The only exchange is at swap-in: the
rank that did the single pinned H2D broadcasts the packed weight arena to
the others over NCCL (NVLink 5 / NVSwitch).  Forward passes need no
collective; each replica D2H-copies its logits slice.

These helpers are device-agnostic so the host logic runs under ``gloo`` on
CPU in tests (tests/test_replicas_cpu.py); bench.py uses them with NCCL.
"""

from __future__ import annotations

import hashlib

import numpy as np


def shard_rows(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) rows of a batch for ``rank``; sizes differ by <= 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError((rank, world))
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_inputs(batches: list[np.ndarray], rank: int, world: int) -> list[np.ndarray]:
    """Each member's batch split independently (mixed per-member batch sizes)."""
    return [b[slice(*shard_rows(len(b), rank, world))] for b in batches]


def arena_digest(buf) -> str:
    return hashlib.sha256(memoryview(np.ascontiguousarray(buf)).cast("B")).hexdigest()


def broadcast_bytes(buf: np.ndarray, src: int = 0, group=None, device=None) -> np.ndarray:
    """Broadcast a uint8 buffer from ``src`` with torch.distributed (gloo on CPU
    buffers, NCCL when ``device`` is a CUDA device)."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(buf, dtype=np.uint8))
    if device is not None:
        t = t.to(device)
    dist.broadcast(t, src=src, group=group)
    return t.cpu().numpy() if device is not None else t.numpy()


def gather_outputs(local: list[np.ndarray], group=None) -> list[np.ndarray]:
    """Concatenate every rank's logits slices in rank order (per member)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    parts: list = [None] * world
    dist.all_gather_object(parts, [np.asarray(x) for x in local], group=group)
    return [np.concatenate([p[m] for p in parts], axis=0) for m in range(len(local))]
