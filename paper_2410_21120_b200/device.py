"""Device residency of a fused DAG: weight arena, activation plans, CUDA graphs.

Swap-in (the reference simulates it: /root/reference/pkg/src/dagfuse/costmodel.py:277-338)
is real here: every member's packed weights are laid out in ONE pinned host
arena and moved with ONE ``cudaMemcpyAsync`` into ONE device allocation
(``dfx_arena_upload``).  ``swap_subgraph`` re-uploads only the incoming
member's segment.  Replication to other GPUs is a single NCCL broadcast of
the arena (``broadcast_arena``).

Execution: an ``ExecInstance`` owns one activation arena (planned by
``planner.first_fit`` over the lowered buffers' launch-index lifetimes), a
split-K workspace, the GEMM descriptor table, I/O staging buffers and one
instantiated CUDA graph containing every member's launches.  In the default
``concurrent`` mode members are independent graph branches with disjoint
arena segments (the reference's Σ, costmodel.py:264-266); ``sequential``
chains members and overlays their segments (max).  Instances are pooled per
batch signature so concurrent ``execute_fused`` callers never share one.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import sys
import threading
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import runtime as rt
from .graph_ir import LiveInterval
from .lower import (ATTN, COPY, DWCONV, DWSE, EW, GAP, GEMM, LN, POOL, SE, TOKENS, MemberProgram,
                    gemm_tiling, lower_member, planes_of)
from .planner import first_fit

ALIGN = 256
# split-K reduction: "kernel" = a separate deterministic reduction node (default,
# measured faster at batch 1: its launch overlaps via PDL and it is spread over
# the whole GPU); "fixup" = the last-arriving CTA of each tile reduces in-kernel
from .lower import SPLITK_MODE
_program_cache: dict[tuple[int, int], tuple] = {}
_cache_lock = threading.Lock()


def program_for(g, w, precision: str = "fp16") -> MemberProgram:
    """Lowered program of (graph, weights, precision), cached for as long as the
    weight store lives (weak reference + finalizer: the cache never keeps a weight
    store or its packed 16-bit blobs alive).  The key is the weight store's identity
    plus the graph's identity-free fingerprint (model id, entry, exit, node count),
    so a model's ModelGraph and the SubGraph fuse_models made of it -- the same
    immutable structure over the same weights -- share one program (a swap brings
    in a member whose program, and pinned segment, were prepared beforehand)."""
    key = (id(w), g.model_id, g.entry, g.exit, len(g.nodes), precision)
    with _cache_lock:
        hit = _program_cache.get(key)
        if hit is not None and hit[1]() is w:
            return hit[2]
    prog = lower_member(g, w, precision=precision)
    with _cache_lock:
        _program_cache[key] = (None, weakref.ref(w), prog)
    weakref.finalize(w, _program_cache.pop, key, None).atexit = False
    return prog


def _fold_rows(v: "rt.View") -> "rt.View":
    """(n, 1, L, c) token view -> (1, 1, n*L, c): the same bytes, one GEMM M axis."""
    assert v.h == 1
    return rt.View(v.base, 1, 1, v.n * v.w, v.c, v.pitch, v.coff, v.dtype)


def _align(x, a=ALIGN):
    return (x + a - 1) // a * a


GEMM_SMEM_LIMIT = 227 * 1024 - 1024          # minus the kernel's 1 KB alignment slack
GEMM_SMEM_FIXED = 1024 + 2048                # barriers/descriptor + epilogue vectors


GEMM_PERSIST = os.environ.get("DFX_GEMM_PERSIST", "1") != "0"    # A/B switch
# from this batch on the SE gate reads its FC weights from L2 instead of staging
# them in smem per CTA (dfx_fused.cu; apply bit 1)
SE_UNSTAGED_BATCH = int(os.environ.get("DFX_SE_UNSTAGED_BATCH", "8"))
# node priorities by member chain length (DFX_PRIORITY=0: off, A/B) for latency-bound
# (every member batch <= 2) instances: 4-model batch 1 2.63 -> 2.48 ms, 8-model batch 1
# 3.37 -> 2.91 ms; with larger or mixed batches chain length is no proxy for work
# (4-model batch 32 12.3 -> 13.3 ms, 8-model batches 1..8 6.6 -> 7.3 ms), so off
NODE_PRIORITY = os.environ.get("DFX_PRIORITY", "1") != "0"
PRIORITY_MAX_BATCH = 2
SLACK_SPLIT_MAX = int(os.environ.get("DFX_SLACK_SPLIT_MAX", "0"))
# ... applied only to members whose estimated chain is below this fraction of the
# longest one (A/B: the members with the most slack give up SMs)
SLACK_FRAC = float(os.environ.get("DFX_SLACK_FRAC", "1.0"))
SLACK_SMS = int(os.environ.get("DFX_SLACK_SMS", "0"))
SLACK_DELAY = float(os.environ.get("DFX_SLACK_DELAY", "0"))
# batch-1 weight tiles (each read by one or two CTAs) loaded with an L2 evict_first
# policy, so weight streaming does not evict the members' activations (A/B)
W_EVICT_FIRST = os.environ.get("DFX_W_EVICT_FIRST", "0") == "1"
# batch <= 2: every GEMM launch prefetches the member's NEXT weight blobs (the next
# GEMM's weights, and the SE's FC weights when an SE launch comes first) into L2
# (dfx_gemm_launch.l2_pf), so a dependent layer's weight TMA hits L2 (A/B)
L2_PREFETCH = os.environ.get("DFX_L2_PREFETCH", "1") != "0"
L2_PREFETCH_MAX_BATCH = 2
L2_PREFETCH_DEPTH = int(os.environ.get("DFX_L2_PREFETCH_DEPTH", "1"))   # A/B: 2 = one launch further
# persistent GEMM for grids above this many waves (A/B knob)
PERSIST_MIN_WAVES = float(os.environ.get("DFX_PERSIST_MIN_WAVES", "2"))
# split precision: slots twice as large (half the prefetched stages per CTA), so the
# one-tile-per-CTA kernel's per-tile prologue and pipeline fill weigh more -- the
# persistent walk pays from under one wave (fp16x2 batch 32: 2 waves 18.76 ms,
# 1.5: 18.03, 1: 17.23, 0.75: 17.18, 0.5: 17.18)
PERSIST_MIN_WAVES_X2 = float(os.environ.get("DFX_PERSIST_MIN_WAVES_X2", "0.75"))
PERSIST_ONE_CTA_X2 = os.environ.get("DFX_PERSIST_ONE_CTA_X2", "0") == "1"   # A/B (dfx_api.cu reads it too)
GEMM_EARLY_PDL = os.environ.get("DFX_GEMM_EARLY_PDL", "0") == "1"            # A/B switch
GEMM_DRAIN_STAGED = os.environ.get("DFX_GEMM_DRAIN", "direct") == "staged"   # A/B switch
# grouped GEMM across members (north-star subsystem 4): pairs of concurrent members
# whose GEMM sequences share layer shapes run those layers as ONE ndesc = 2 launch
# (ExecInstance._pair_chains).  Measured: configs[4] (8 members) 6.09 ->
# 5.99 ms; ResNet-50 + ResNet-152 alone slower (1.25 -> 1.28 ms at batch 1, 2.28 ->
# 2.54 at batch 8: the coupled chains wait for each other).  "auto": DAGs of >= 6
# concurrent members; "1" always; "0" never.
GROUP_GEMM = {"1": True, "0": False}.get(os.environ.get("DFX_GROUP_GEMM", "auto"), "auto")
GROUP_AUTO_MEMBERS = 6
GROUP_MIN = int(os.environ.get("DFX_GROUP_MIN", "4"))          # matched layers for a pair to group
# e2e queries gather their inputs on a host thread pool, overlapping the H2D (A/B switch)
E2E_GATHER = os.environ.get("DFX_E2E_GATHER", "1") != "0"
# end to end with per-member input gates (dfx_execute_gated): the graph is launched
# first and every member starts as soon as its own input is on the device (the
# longest chain gathered and sent first).  Measured no gain (fp16x2 e2e 3.24 ms
# gathered-then-launched vs 3.27 ms gated: the graph launch call now precedes the
# gather on the host, and the gates add a kernel per chain).  Off (DFX_E2E_GATED=1)
E2E_GATED = os.environ.get("DFX_E2E_GATED", "0") == "1"


def gemm_slots(bn: int, tiles: int, sm_count: int = 148, m2: int = 0, planes: int = 1) -> int:
    """Pipeline depth of a GEMM launch: as deep as shared memory allows (<= 8)
    when the grid fits in one wave -- every extra slot is another weight tile
    requested before griddepcontrol.wait -- else 4, leaving room for two CTAs
    per SM on narrow tiles.  m2 slots hold two A tiles (dfx_common.cuh gemm_slot_bytes)."""
    slot = (128 * 64 * 2 * (1 + m2) + bn * 128) * planes
    fit = (GEMM_SMEM_LIMIT - GEMM_SMEM_FIXED) // slot
    return max(2, min(8 if tiles <= sm_count else 4, fit))


# ------------------------------------------------------------------------------ weights

def arena_layout(programs: list[MemberProgram]):
    """Byte layout of the packed weight arena: member segments in member order,
    blobs in sorted-key order inside a segment, every blob 256-B aligned (TMA
    needs 16 B; 256 keeps every tensor on its own L2 sector group).
    Returns (per-member {key: offset}, per-member (offset, bytes), total)."""
    layout, segments, at = [], [], 0
    for p in programs:
        seg0, offs = at, {}
        for key in sorted(p.blobs):
            offs[key] = at
            at = _align(at + p.blobs[key].nbytes)
        layout.append(offs)
        segments.append((seg0, at - seg0))
    return layout, segments, max(at, ALIGN)


# id(program) -> (weakref, offsets, bytes, pinned _Block): a member's packed weight
# segment staged ONCE in pinned host memory, so a swap_subgraph that brings the
# member in is one allocation + D2D of the untouched members + ONE H2D, with no
# per-swap pinning or packing on the host
_segments: dict[int, tuple] = {}
_segments_lock = threading.Lock()


def _release_segment(key):
    with _segments_lock:
        hit = _segments.pop(key, None)
    if hit is not None:
        hit[3].release()


def stage_segment(prog: MemberProgram) -> tuple[dict, int, int]:
    """(blob offsets, bytes, pinned host address) of a member's packed segment;
    staged on first use and kept while the program lives."""
    offs, size, blk = _stage_block(prog)
    return offs, size, blk.ptr


def _stage_block(prog: MemberProgram):
    key = id(prog)
    with _segments_lock:
        hit = _segments.get(key)
        if hit is not None and hit[0]() is prog:
            return hit[1], hit[2], hit[3]
    offs, at = {}, 0
    for k in sorted(prog.blobs):
        offs[k] = at
        at = _align(at + prog.blobs[k].nbytes)
    size = max(at, ALIGN)
    blk = _Block(rt.host_alloc(size), "host")
    buf = np.frombuffer((C.c_uint8 * size).from_address(blk.ptr), dtype=np.uint8)
    for k, off in offs.items():
        raw = prog.blobs[k].view(np.uint8).reshape(-1)
        buf[off:off + raw.size] = raw
    with _segments_lock:
        _segments[key] = (weakref.ref(prog), offs, size, blk)
    weakref.finalize(prog, _release_segment, key).atexit = False
    return offs, size, blk


def fill_arena(buf: np.ndarray, programs: list[MemberProgram], layout) -> None:
    """Copy every blob into its slot of a uint8 arena buffer."""
    for p, offs in zip(programs, layout):
        for key, off in offs.items():
            raw = p.blobs[key].view(np.uint8).reshape(-1)
            buf[off:off + raw.size] = raw


# weight arenas come from a retained stream-ordered pool (dfx_pool_malloc): a
# swapped-out arena's pages stay mapped for the next swap-in (DFX_ARENA_POOL=0:
# plain cudaMalloc / cudaFree, A/B)
ARENA_POOL = os.environ.get("DFX_ARENA_POOL", "1") != "0"


class _Block:
    """One device (or pinned host) allocation, reference-counted by the arenas
    that read it: a swapped DAG shares every untouched member's bytes with the
    DAG it was swapped from, and the memory goes back when the last one is
    unloaded (release on refs == 0)."""

    _lock = threading.Lock()

    def __init__(self, ptr: int, kind: str):
        self.ptr, self.kind, self.refs = ptr, kind, 1

    def retain(self) -> "_Block":
        with self._lock:
            assert self.refs > 0, "retain of a released block"
            self.refs += 1
        return self

    def release(self) -> None:
        with self._lock:
            self.refs -= 1
            last = self.refs == 0
        if last and self.ptr:
            {"pool": rt.pool_free, "dev": rt.free, "host": rt.host_free}[self.kind](self.ptr)
            self.ptr = 0


def _arena_block(nbytes: int, stream=None) -> _Block:
    if not ARENA_POOL:
        return _Block(rt.malloc(nbytes), "dev")
    return _Block(rt.pool_malloc(nbytes, stream), "pool")


class WeightArena:
    """Packed weights of all members: host pinned staging + device copy.

    Ownership: the device allocation(s) and the pinned staging are _Blocks.
    ``clone_for_swap`` shares them (retain); ``replace_member`` puts the incoming
    member in a NEW device block, so the source DAG's bytes are never written
    and it stays valid; ``free`` releases this arena's references."""

    def __init__(self, programs: list[MemberProgram], device: int = 0):
        self.device = device
        self.layout, self.segments, self.total = arena_layout(programs)
        rt.init_device(device)
        if len(programs) == 1:
            # one member: its staged pinned segment (stage_segment) IS the arena's
            # host copy -- no pinning or packing per load
            offs, size, blk = _stage_block(programs[0])
            assert size == self.total and offs == self.layout[0]
            self._host_block = blk.retain()
            self.host_pinned = True
            self._init_device_state()
            return
        host = rt.host_alloc(self.total)
        self._host_block = _Block(host, "host")
        self.host_pinned = True
        view = (C.c_uint8 * self.total).from_address(host)
        fill_arena(np.frombuffer(view, dtype=np.uint8), programs, self.layout)
        self._init_device_state()

    @classmethod
    def from_host(cls, layout, segments, total, host: int, device: int = 0, pinned: bool = True,
                  keep=None) -> "WeightArena":
        """An arena over an already-filled host buffer (pack_io: read from a file).
        Pinned buffers are owned (freed with the arena); pageable ones are kept
        alive through ``keep``."""
        a = cls.__new__(cls)
        a.device = device
        a.layout, a.segments, a.total = layout, segments, total
        a._host_block = _Block(host, "host") if pinned else None
        a.host_pinned = pinned
        a._host_keep = keep
        a._host_ptr = host
        a._init_device_state()
        return a

    def _init_device_state(self):
        self._dev_block: _Block | None = None
        self._swap_blocks: list[_Block] = []
        self.member_base: list[int] = []       # device base of each member's segment
        self.upload_ms = None
        self.last_swap = None

    @property
    def host(self) -> int:
        return self._host_block.ptr if self._host_block is not None else getattr(self, "_host_ptr", 0)

    @property
    def dev(self) -> int:
        return self._dev_block.ptr if self._dev_block is not None else 0

    @property
    def shared(self) -> bool:
        return any(b.refs > 1 for b in self._blocks())

    def _blocks(self):
        out = [self._dev_block] if self._dev_block is not None else []
        return out + list(self._swap_blocks)

    def upload(self, stream=None) -> float:
        """ONE device allocation + ONE H2D copy of the whole arena; returns ms.

        The two phases are timed apart (the reference's cost model books them
        as separate cudaMalloc / cudaMemcpyAsync rows, costmodel.py:297-300):
        ``malloc_ms`` by wall clock, ``memcpy_ms`` by CUDA events."""
        if self._dev_block is not None:
            raise RuntimeError("arena already resident (unload() first)")
        t0 = time.perf_counter()
        self._dev_block = _arena_block(self.total, stream)
        self.malloc_ms = (time.perf_counter() - t0) * 1e3
        e0, e1 = rt.Event(), rt.Event()
        e0.record(stream)
        rt.h2d(self.dev, self.host, self.total, stream)
        e1.record(stream)
        self.memcpy_ms = e0.elapsed_ms(e1)
        rt.stream_sync(stream)
        self.upload_ms = (time.perf_counter() - t0) * 1e3
        self.member_base = [self.dev + off for off, _ in self.segments]
        return self.upload_ms

    def unload(self) -> None:
        """Swap-out: free the device copy, keep a pinned host copy (the next upload()
        is again one allocation + one H2D).  An arena made by a swap has no host
        staging of its own layout yet: the device bytes are first read back into a
        fresh pinned buffer (one D2H).  Only for an arena no other DAG shares."""
        if self.shared:
            raise RuntimeError("arena shared with a swapped DAG: unload the DAGs instead")
        if self._dev_block is not None and getattr(self, "host_stale", False):
            host = rt.host_alloc(self.total)
            rt.d2h(host, self.dev, self.total, None)
            rt.stream_sync(None)
            if self._host_block is not None:
                self._host_block.release()
            self._host_block, self.host_pinned, self.host_stale = _Block(host, "host"), True, False
        for b in self._blocks():
            b.release()
        self._dev_block, self._swap_blocks = None, []
        self.member_base = []

    def allocate(self) -> None:
        """Device allocation only (a replica that receives the arena by broadcast)."""
        self._dev_block = _arena_block(self.total)
        self.member_base = [self.dev + off for off, _ in self.segments]

    def addr(self, member: int, key: str) -> int:
        return self.member_base[member] + (self.layout[member][key] - self.segments[member][0])

    def segment(self, member: int) -> tuple[int, int]:
        """(device address, bytes) of one member's weights."""
        return self.member_base[member], self.segments[member][1]

    def replace_member(self, member: int, prog: MemberProgram, stream=None, upload: bool = True) -> float:
        """swap_subgraph on a resident arena: a NEW contiguous device block for the
        post-swap DAG -- the untouched members' segments copied device-to-device
        from the source blocks (HBM speed), ONLY the incoming member uploaded from
        the host.  The source DAG's bytes are never written (it stays valid, and
        queries on it may run concurrently); when it is unloaded its block goes
        back whole, so the outgoing member's bytes do not outlive it (no dead
        segments accumulate over a swap sequence).  Returns the wall ms of
        allocation + copies; ``last_swap`` has the phases.  ``upload=False`` (a
        replica): the incoming segment is left for the broadcast."""
        offs, size, host = stage_segment(prog) if upload else (None, 0, 0)
        if not upload:
            offs, at = {}, 0
            for key in sorted(prog.blobs):
                offs[key] = at
                at = _align(at + prog.blobs[key].nbytes)
            size = max(at, ALIGN)
        # the new layout: members in order, each segment 256-B aligned
        old_base, old_layout, old_segments = list(self.member_base), self.layout, self.segments
        layout, segments, total = [], [], 0
        for i in range(len(old_segments)):
            if i == member:
                rel, nbytes = offs, size
            else:
                o0, nbytes = old_segments[i]
                rel = {k: v - o0 for k, v in old_layout[i].items()}
            segments.append((total, nbytes))
            layout.append({k: total + v for k, v in rel.items()})
            total = _align(total + nbytes)
        t0 = time.perf_counter()
        blk = _arena_block(total, stream)
        t1 = time.perf_counter()
        e0, e1, e2 = rt.Event(), rt.Event(), rt.Event()
        e0.record(stream)
        for i, (off, nbytes) in enumerate(segments):
            if i != member:
                rt.d2d(blk.ptr + off, old_base[i], nbytes, stream)
        e1.record(stream)
        if upload:
            rt.h2d(blk.ptr + segments[member][0], host, size, stream)
        e2.record(stream)
        rt.stream_sync(stream)
        ms = (time.perf_counter() - t0) * 1e3
        self.last_swap = {"bytes": size, "arena_bytes": total, "malloc_ms": (t1 - t0) * 1e3,
                          "d2d_ms": e0.elapsed_ms(e1), "memcpy_ms": e1.elapsed_ms(e2) if upload else None,
                          "ms": ms if upload else 0.0}
        for b in self._blocks():                  # this arena now reads only the new block
            b.release()
        self._dev_block, self._swap_blocks = blk, []
        self.layout, self.segments, self.total = layout, segments, total
        self.member_base = [blk.ptr + off for off, _ in segments]
        self.host_stale = True                    # the pinned staging has the old layout
        return self.last_swap["ms"]

    def clone_for_swap(self) -> "WeightArena":
        """A second arena over the same blocks (each retained once more)."""
        twin = object.__new__(WeightArena)
        twin.__dict__.update(self.__dict__)
        twin.layout = list(self.layout)
        twin.segments = list(self.segments)
        twin.member_base = list(self.member_base)
        twin._dev_block = self._dev_block.retain() if self._dev_block is not None else None
        twin._swap_blocks = [b.retain() for b in self._swap_blocks]
        twin._host_block = self._host_block.retain() if self._host_block is not None else None
        return twin

    def free(self):
        """Release this arena's references (device blocks, pinned staging);
        idempotent."""
        for b in self._blocks():
            b.release()
        if self._host_block is not None:
            self._host_block.release()
        self._dev_block, self._swap_blocks, self._host_block = None, [], None
        self._host_keep = None
        self._host_ptr = 0
        self.member_base = []


class PerTensorArena:
    """The UNFUSED baseline loader (what per-model framework loading does):
    one cudaMalloc + one cudaMemcpyAsync per weight tensor, model by model.
    Same interface as WeightArena so the same kernels run on it; used only to
    measure the fused-vs-unfused claims.

    ``pinned=False``: each tensor is copied from its own pageable host array (the
    copy completes before cudaMemcpyAsync returns).  ``pinned=True``: the A/B that
    separates consolidation from pinning -- every tensor is first staged (untimed,
    like WeightArena's packed staging) in ONE pinned host buffer, then still gets
    its own cudaMalloc and its own asynchronous cudaMemcpyAsync."""

    def __init__(self, programs: list[MemberProgram], device: int = 0, stream=None, pinned: bool = False):
        rt.init_device(device)
        self.device = device
        self.ptrs: list[dict[str, int]] = []
        self.tensors = 0
        self.total = 0
        self.malloc_ms = self.memcpy_ms = 0.0
        self.pinned = pinned
        host = None
        if pinned:
            sizes = [_align(np.asarray(p.blobs[k]).nbytes) for p in programs for k in sorted(p.blobs)]
            host = rt.host_alloc(max(sum(sizes), 16))
            hb = np.frombuffer((C.c_uint8 * max(sum(sizes), 16)).from_address(host), dtype=np.uint8)
            at = 0
            for p in programs:
                for key in sorted(p.blobs):
                    raw = np.ascontiguousarray(p.blobs[key]).view(np.uint8).reshape(-1)
                    hb[at:at + raw.size] = raw
                    at += _align(raw.size)
        t0 = time.perf_counter()
        at = 0
        for p in programs:
            table = {}
            for key in sorted(p.blobs):
                blob = np.ascontiguousarray(p.blobs[key])
                src = host + at if pinned else blob.ctypes.data
                ta = time.perf_counter()
                ptr = rt.malloc(blob.nbytes)
                tb = time.perf_counter()
                rt.call("dfx_memcpy_h2d", C.c_void_p(ptr), C.c_void_p(src),
                        C.c_size_t(blob.nbytes), C.c_void_p(stream))
                if not pinned:
                    rt.stream_sync(stream)        # pageable source: copy completes before return
                self.malloc_ms += (tb - ta) * 1e3
                self.memcpy_ms += (time.perf_counter() - tb) * 1e3
                table[key] = ptr
                self.tensors += 1
                self.total += blob.nbytes
                at += _align(blob.nbytes)
            self.ptrs.append(table)
        if pinned:
            tc = time.perf_counter()
            rt.stream_sync(stream)                # the queued copies drain
            self.memcpy_ms += (time.perf_counter() - tc) * 1e3
            rt.host_free(host)
        self.upload_ms = (time.perf_counter() - t0) * 1e3

    def addr(self, member: int, key: str) -> int:
        return self.ptrs[member][key]

    def free(self):
        for table in self.ptrs:
            for p in table.values():
                rt.free(p)
        self.ptrs = []


def broadcast_arena(arena: WeightArena, src: int = 0, group=None) -> None:
    """Replicate the device arena from rank ``src`` over NCCL (torch.distributed
    plumbing; the arena is wrapped zero-copy through __cuda_array_interface__)."""
    import torch
    import torch.distributed as dist

    class _Iface:
        def __init__(self, ptr, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1",
                                             "data": (ptr, False), "version": 3}

    t = torch.as_tensor(_Iface(arena.dev, arena.total), device=f"cuda:{arena.device}")
    dist.broadcast(t, src=src, group=group)


# ------------------------------------------------------------------------------ plans

@dataclass
class MemberPlan:
    offsets: list[int]          # per buffer, relative to the member segment
    arena_bytes: int
    ws_bytes: int
    tilings: dict[int, dict]    # launch index -> gemm tiling
    skip: frozenset = frozenset()   # launch indices absorbed by a GEMM's depthwise epilogue


# GEMM -> depthwise conv in one launch when one CTA holds the whole GEMM output map
# (batch-1 MBConv expand convs at 14x14 / 7x7; dfx_gemm.cu dw_k > 0).  DFX_GEMM_DW=0: off
GEMM_DW = os.environ.get("DFX_GEMM_DW", "1") != "0"
GEMM_DW_BN = int(os.environ.get("DFX_GEMM_DW_BN", "32"))
GEMM_DW_BN_M2 = int(os.environ.get("DFX_GEMM_DW_BN_M2", "16"))     # two M tiles per CTA
# two M tiles (14x14 maps): a 2-CTA cluster, one tile each, halo rows over DSMEM
# ("cluster"), or both tiles in one m2 CTA ("m2")
GEMM_DW_PAIR = os.environ.get("DFX_GEMM_DW_PAIR", "cluster")
GEMM_DW_BN_PAIR = int(os.environ.get("DFX_GEMM_DW_BN_PAIR", "32"))
# "nosplit": only where the GEMM alone would not split K (the fused launch never does);
# "single": only where one 128-row M tile holds the map (no m2)
GEMM_DW_MODE = os.environ.get("DFX_GEMM_DW_MODE", "all")
# the squeeze-excitation after a fused depthwise conv absorbed too (dfx_epi.cuh
# se_finish: one grid-wide barrier instead of an SE launch).  Measured slower
# (EfficientNetV2-L batch 1 node sum 1.95 -> 2.02 ms fp16; 4-model DAG 2.17 -> 2.49 ms):
# the barrier waits out the CTA skew (~3.5 us) and the partial-sum gather + hidden
# vector run serialised after it, where the separate SE launch overlaps its prologue
# with the GEMM's tail under PDL.  Off by default (DFX_GEMM_DW_SE=1: on, A/B)
GEMM_DW_SE = os.environ.get("DFX_GEMM_DW_SE", "0") == "1"
# the SE launch after a depthwise-epilogue GEMM keeps running, but the GEMM's CTAs --
# which hold every depthwise output of their channels -- write the channel means
# (dfx_se_fuse mode 1), so the SE skips its pooling pass over x.  Measured slower:
# the means (butterflies, syncs, a pair's DSMEM exchange) add 2.5 us to the GEMM
# and save 0.8 us in the SE (EfficientNetV2-L fp16x2 node classes; 4-model batch 1
# 3.04 -> 3.10 ms fp16x2, 2.19 -> 2.28 ms fp16).  Off (DFX_GEMM_DW_SQUEEZE=1: A/B)
GEMM_DW_SQUEEZE = os.environ.get("DFX_GEMM_DW_SQUEEZE", "0") == "1"
_DW_ACTS = (None, "relu", "hardswish", "silu")


def gemm_dw_pairs(prog: MemberProgram) -> dict[int, int]:
    """GEMM launch index -> index of the depthwise launch right after it that is
    the ONLY reader of its output (structure only; the batch decides in plan_member).
    The depthwise must be a shape dwconv_tile_kernel takes (square 3x3 / 5x5,
    stride 1 / 2) with BN + one of its templated activations."""
    readers: dict[str, int] = {}
    for L in prog.launches:
        for v in (L.src, L.epi.other):
            if v is not None:
                readers[v] = readers.get(v, 0) + 1
    bufs: dict[int, int] = {}
    for v in prog.values.values():
        bufs[v.buf] = bufs.get(v.buf, 0) + 1
    out = {}
    ls = prog.launches
    for i in range(len(ls) - 1):
        L, D = ls[i], ls[i + 1]
        if L.kind != GEMM or D.kind != DWCONV or D.src != L.dst or readers.get(L.dst) != 1:
            continue
        if L.dst == prog.exit_value or bufs.get(prog.values[L.dst].buf) != 1:
            continue
        if L.geom.get("tokens") or L.pre is not None or L.epi.binop or L.epi.act2 is not None:
            continue
        g = D.geom
        if not (g["kh"] == g["kw"] and g["kh"] in (3, 5) and g["sh"] == g["sw"] and g["sh"] in (1, 2)
                and g["ph"] == g["pw"]):
            continue
        if D.epi.binop or D.epi.act2 is not None or D.epi.act1 not in _DW_ACTS:
            continue
        vi, vo = prog.values[L.dst], prog.values[D.dst]
        if L.geom["cout"] % 8 or vi.c != L.geom["cout"] or vo.coff % 8 or \
                prog.buffers[vo.buf].pitch % 8:
            continue
        out[L.index] = D.index
    return out


def dw_se_pairs(prog: MemberProgram, dw_pairs: dict[int, int]) -> dict[int, int]:
    """GEMM launch index -> the SE launch its depthwise epilogue can absorb: the SE
    (with its channel_scale fused, apply = 1) reads the depthwise output and nothing
    else does (dfx_gemm_desc.se, dfx_epi.cuh se_finish)."""
    readers: dict[str, int] = {}
    for L in prog.launches:
        for v in (L.src, L.epi.other):
            if v is not None:
                readers[v] = readers.get(v, 0) + 1
    by_index = {L.index: L for L in prog.launches}
    out = {}
    for gi, di in dw_pairs.items():
        D = by_index[di]
        S = by_index.get(di + 1)
        if S is None or S.kind != SE or S.src != D.dst or not S.geom.get("apply") or readers.get(D.dst) != 1:
            continue
        if D.dst == prog.exit_value or S.geom["cr"] > 512 or S.geom["c"] != D.geom["cout"]:
            continue
        vo = prog.values[S.dst]
        if vo.coff % 8 or prog.buffers[vo.buf].pitch % 8:
            continue
        out[gi] = S.index
    return out


def _dw_smem_need(n, h, w, oh, ow, bn, planes, se_cr=0, nt=0) -> int:
    """Operand-slot bytes a depthwise-epilogue GEMM CTA needs after its main loop: the
    GEMM output map, and with a fused SE (hidden width se_cr, nt channel tiles) the
    depthwise-output tile + reduction scratch + gathered fc1 partials (dfx_api.cu
    DFX_OP_GEMM, dfx_epi.cuh se_finish)."""
    need = (n * h * w * (bn + 8) * 2 * planes + 15) & ~15
    if se_cr:
        need += (((n * oh * ow * bn * 2 * planes + 15) & ~15) + 256 * 16 * 4 +
                 (4 * bn + 2 * ((se_cr + 3) & ~3) + nt * n * se_cr + 4) * 4)
    return need


def plan_member(prog: MemberProgram, n: int, sm_count: int = 148, cluster_ok: bool = False,
                max_splits: int = 0, se_cta_limit: int = 0) -> MemberPlan:
    """Activation plan + GEMM tilings of one member at batch n.  ``cluster_ok``: the
    DAG is small enough for cluster split-K (lower.SPLITK_MODE "auto").
    ``se_cta_limit`` > 0: depthwise-epilogue GEMMs may absorb the SE after them when
    their grid has at most this many CTAs (a fused SE meets at a grid-wide barrier:
    the concurrent members' fused grids must fit the GPU together)."""
    ws = 0
    tilings = {}
    skip: set[int] = set()
    planes = planes_of(prog.precision)
    dw_pairs = gemm_dw_pairs(prog) if GEMM_DW else {}
    se_pairs = dw_se_pairs(prog, dw_pairs) if GEMM_DW_SE and se_cta_limit and n <= 2 else {}
    sq_pairs = dw_se_pairs(prog, dw_pairs) if GEMM_DW_SQUEEZE and n <= 2 else {}
    for L in prog.launches:
        if L.kind != GEMM:
            continue
        out = prog.values[L.dst]
        if L.geom.get("tokens"):        # token rows of all images are one contiguous M
            t = gemm_tiling(L.geom, 1, 1, n * out.w, sm_count, cluster_ok=cluster_ok and n <= 2,
                            max_splits=max_splits, planes=planes)
        else:
            t = gemm_tiling(L.geom, n, out.h, out.w, sm_count, cluster_ok=cluster_ok, max_splits=max_splits,
                            planes=planes)
        if L.index in dw_pairs and n * out.h * out.w <= 256 and \
                (GEMM_DW_MODE == "all" or t["splits"] == 1):
            # one CTA (m2: two M tiles) holds the whole output map of its channels
            mt = t["mt_n"] * t["mt_p"] * t["mt_q"]
            pair = mt == 2 and GEMM_DW_PAIR == "cluster" and t["mt_p"] == 2
            m2 = int(mt == 2 and not pair)
            bn = min(GEMM_DW_BN_M2 if m2 else GEMM_DW_BN_PAIR if pair else GEMM_DW_BN, t["bn"])
            nt = -(-L.geom["cout"] // bn)
            xs = n * out.h * out.w * (bn + 8) * 2 * planes  # the map in smem (dfx_gemm.cu)
            nsl = gemm_slots(bn, nt * (2 if pair else 1), sm_count, m2, planes)
            if mt <= (1 if GEMM_DW_MODE == "single" else 2) and not (m2 and planes > 1) and \
                    xs <= nsl * (128 * 64 * 2 * (1 + m2) + bn * 128) * planes:
                t = dict(t, bn=bn, nt=nt, splits=1, sps=t["stages"], csplit=0, m2=m2,
                         tiles=nt * (2 if pair else 1), dw=dw_pairs[L.index])
                skip.add(dw_pairs[L.index])
                si = se_pairs.get(L.index)
                if si is not None and not m2:
                    # fused SE: the grid meets at one barrier -- widen the channel tile
                    # until it fits its share of the SMs (and the tile fits smem)
                    D = next(x for x in prog.launches if x.index == t["dw"])
                    S = next(x for x in prog.launches if x.index == si)
                    dv, cr = prog.values[D.dst], S.geom["cr"]
                    for bn2 in sorted({bn, 64, 128}):
                        if bn2 < bn:
                            continue
                        nt2 = -(-L.geom["cout"] // bn2)
                        tiles2 = nt2 * (2 if pair else 1)
                        slot = (128 * 64 * 2 + bn2 * 128) * planes
                        extra = ((D.geom["kh"] ** 2 + 2) * bn2 * 4 +         # taps + BN vectors
                                 2 * planes * bn2 * cr * 2)                  # staged fc1^T / fc2 rows
                        nsl2 = min(gemm_slots(bn2, tiles2, sm_count, 0, planes),
                                   (GEMM_SMEM_LIMIT - GEMM_SMEM_FIXED - extra) // slot)
                        need = _dw_smem_need(n, out.h, out.w, dv.h, dv.w, bn2, planes, cr, nt2)
                        if tiles2 <= se_cta_limit and nsl2 >= 2 and need <= nsl2 * slot:
                            t = dict(t, bn=bn2, nt=nt2, tiles=tiles2, se=si, nslots=nsl2, se_cr=cr)
                            skip.add(si)
                            break
                sq = sq_pairs.get(L.index)
                if sq is not None and t.get("se") is None and not m2:
                    # the SE's squeeze from the depthwise epilogue (means' scratch after the map)
                    need = xs + (256 * 16 + 4 * bn) * 4 + 16
                    if need <= nsl * (128 * 64 * 2 + bn * 128) * planes:
                        t = dict(t, squeeze=sq)
        tilings[L.index] = t
        if t["splits"] > 1 and not t["csplit"]:      # cluster split-K needs no workspace
            ws = max(ws, t["splits"] * n * out.h * out.w * t["nt"] * t["bn"] * 4)
    # buffer lifetimes AFTER the fusion decisions: a GEMM that absorbs its depthwise
    # conv writes the depthwise output at its own launch index, one launch before
    # the (skipped) depthwise launch would have -- while its own input is still
    # being read by slower CTAs of the same grid.  The output's interval must
    # therefore start at the GEMM, or first_fit could overlay it on that input.
    first = {b.bid: b.first for b in prog.buffers}
    by_index = {L.index: L for L in prog.launches}
    for gi, t in tilings.items():
        for role in ("dw", "se"):              # absorbed launches write at the GEMM's index
            if t.get(role) is not None:
                D = by_index[t[role]]
                ob = prog.values[D.dst].buf
                first[ob] = min(first[ob], gi)
    ivs = [LiveInterval(str(b.bid).zfill(6), b.bytes_for(n), first[b.bid], b.last)
           for b in prog.buffers]
    places = first_fit(ivs, align=ALIGN)
    offsets = [0] * len(prog.buffers)
    for pl in places:
        offsets[int(pl.name)] = pl.offset
    arena = max((pl.offset + pl.size for pl in places), default=0)
    return MemberPlan(offsets, _align(arena), _align(ws), tilings, frozenset(skip))


# ------------------------------------------------------------------------------ instances

class ExecInstance:
    """One instantiated CUDA graph of the whole fused DAG for a batch signature."""

    def __init__(self, dag: "DeviceDag", batch: tuple[int, ...]):
        self.dag, self.batch = dag, batch
        self.dtype = rt.DTYPES[dag.precision]
        progs, arena = dag.programs, dag.arena
        rt.init_device(dag.device)
        self.stream = rt.stream_create()
        # cluster split-K only in small concurrent DAGs: its clusters need free GPC
        # slices, which many concurrent branches rarely leave
        cluster_ok = sum(1 for n in batch if n > 0) <= 4
        # A/B (DFX_SLACK_SPLIT_MAX=k): at small batch, members off the critical chain
        # split K at most k ways, leaving SMs to the longest chain
        caps = [0] * len(progs)
        # A/B (DFX_SLACK_SMS=k): the same members instead run every GEMM unsplit on
        # the persistent kernel with at most k CTAs, so they never hold more than
        # ~k SMs while the critical chain's kernels wait for free SMs
        self.sm_budget = [0] * len(progs)
        self.sm_budget_slack = [False] * len(progs)
        if SLACK_DELAY > 0 and dag.mode == "concurrent" and max(batch) <= PRIORITY_MAX_BATCH:
            est = [sum(_NODE_BASE_US.get(L.kind, 2.5) for L in p.launches) if n > 0 else 0
                   for p, n in zip(progs, batch)]
            crit = est.index(max(est))
            self.sm_budget_slack = [i != crit and e < SLACK_FRAC * est[crit] for i, e in enumerate(est)]
        if (SLACK_SPLIT_MAX or SLACK_SMS) and dag.mode == "concurrent" and max(batch) <= PRIORITY_MAX_BATCH:
            est = [sum(_NODE_BASE_US.get(L.kind, 2.5) for L in p.launches) if n > 0 else 0
                   for p, n in zip(progs, batch)]
            crit = est.index(max(est))
            slack = [i != crit and e < SLACK_FRAC * est[crit] for i, e in enumerate(est)]
            caps = [(1 if SLACK_SMS else SLACK_SPLIT_MAX) if s else 0 for s in slack]
            self.sm_budget = [SLACK_SMS if s else 0 for s in slack]
            if os.environ.get("DFX_SLACK_DEBUG"):
                print(f"slack caps: est {[round(e) for e in est]} caps {caps} sms {self.sm_budget}",
                      file=sys.stderr)
        # fused SE grids meet at a grid-wide barrier: the members that may run one at the
        # same time share the SMs (concurrent mode; sequential members never overlap)
        se_members = sum(1 for p, n in zip(progs, batch) if 0 < n <= 2 and any(L.kind == SE for L in p.launches))
        se_limit = (dag.sm_count if dag.mode == "sequential" else dag.sm_count // max(se_members, 1))
        self.plans = [plan_member(p, n, dag.sm_count, cluster_ok, caps[i], se_limit) if n > 0
                      else MemberPlan([], 0, 0, {})
                      for i, (p, n) in enumerate(zip(progs, batch))]
        seq = dag.mode == "sequential"
        # activation arena: disjoint member segments (concurrent) or overlaid (sequential)
        self.seg_off, at = [], 0
        for pl in self.plans:
            self.seg_off.append(0 if seq else at)
            at = max(at, pl.arena_bytes) if seq else at + pl.arena_bytes
        self.act_bytes = _align(max(at, ALIGN))
        ws_each = [pl.ws_bytes for pl in self.plans]
        self.ws_off, wat = [], 0
        for wb in ws_each:
            self.ws_off.append(0 if seq else wat)
            wat = max(wat, wb) if seq else wat + wb
        self.ws_bytes = _align(max(wat, ALIGN))
        self.in_sizes = [n * int(np.prod(p.input_dims)) * 4 for p, n in zip(progs, batch)]
        self.out_sizes = [n * int(np.prod(p.output_dims)) * 4 for p, n in zip(progs, batch)]
        self.in_off = np.cumsum([0] + self.in_sizes).tolist()
        self.out_off = np.cumsum([0] + self.out_sizes).tolist()
        self.in_bytes, self.out_bytes = self.in_off[-1], self.out_off[-1]
        n_gemm = sum(1 for p, n in zip(progs, batch) for L in p.launches if L.kind == GEMM and n)
        self.act = rt.malloc(self.act_bytes)
        self.ws = rt.malloc(self.ws_bytes)
        n_ctr = sum(t["mt_n"] * t["mt_p"] * t["mt_q"] * t["nt"]
                    for pl in self.plans for t in pl.tilings.values() if t["splits"] > 1)
        self.counters = rt.malloc(max(4 * n_ctr, 16))
        self._ctr_used = 0
        self.desc_capacity = 2 * max(n_gemm, 1)       # room for the grouped launches' copies
        self.descs = rt.malloc(self.desc_capacity * C.sizeof(rt.GemmDesc))
        # fused SE (dfx_se_fuse per absorbing GEMM): descriptors, fc1 partial scratch,
        # barrier words (zeroed once; the barrier leaves them reusable)
        self.se_count = sum(1 for pl in self.plans for t in pl.tilings.values()
                            if t.get("se") is not None or t.get("squeeze") is not None)
        self.pool_bytes = sum(_align(n * 4 * 4096) for pl, n in zip(self.plans, batch)
                              for t in pl.tilings.values() if t.get("squeeze") is not None)
        self.se_pooled = rt.malloc(max(self.pool_bytes, 16))
        self._pool_used = 0
        self._squeeze_ptr: dict = {}
        self.se_scratch_bytes = sum(_align(t["nt"] * n * 512 * 4) for pl, n in zip(self.plans, batch)
                                    for t in pl.tilings.values() if t.get("se") is not None)
        self.se_structs = rt.malloc(max(self.se_count, 1) * C.sizeof(rt.SeFuse))
        self.se_sync = rt.malloc(max(self.se_count, 1) * 16)
        self.se_scratch = rt.malloc(max(self.se_scratch_bytes, 16))
        self._se_host: list = []
        self._se_scratch_used = 0
        self.dev_in = rt.malloc(max(self.in_bytes, 16))
        self.dev_out = rt.malloc(max(self.out_bytes, 16))
        # per-member input gates: device flags, a pinned 1, a copy stream
        self.gated = E2E_GATED and E2E_GATHER
        self.gate_flags = rt.malloc(4 * max(len(progs), 4))
        self.gate_one = rt.host_alloc(16)
        C.c_uint32.from_address(self.gate_one).value = 1
        self.copy_stream = rt.stream_create()
        self.host_in = rt.host_alloc(max(self.in_bytes, 16))
        self.host_out = rt.host_alloc(max(self.out_bytes, 16))
        rt.memset(self.act, 0, self.act_bytes, self.stream)
        rt.memset(self.se_sync, 0, max(self.se_count, 1) * 16, self.stream)
        rt.memset(self.gate_flags, 0, 4 * max(len(progs), 4), self.stream)
        rt.memset(self.counters, 0, max(4 * n_ctr, 16), self.stream)
        self.gemm_count = 0
        self.kernel_nodes = 0
        self.graph = self._build(progs, arena)
        rt.stream_sync(self.stream)

    # --- views
    def _view(self, m: int, prog: MemberProgram, name: str, n: int) -> rt.View:
        v = prog.values[name]
        b = prog.buffers[v.buf]
        base = self.act + self.seg_off[m] + self.plans[m].offsets[v.buf]
        return rt.View(base, n, v.h, v.w, v.c, b.phys_pitch, v.coff, self.dtype)

    def _epi(self, m, prog, L, n) -> rt.Epilogue:
        e = rt.Epilogue()
        arena = self.dag.arena
        e.alpha = arena.addr(m, L.blobs["alpha"]) if "alpha" in L.blobs else None
        e.beta = arena.addr(m, L.blobs["beta"]) if "beta" in L.blobs else None
        e.act1 = rt.ACT[L.epi.act1]
        e.act2 = rt.ACT[L.epi.act2]
        e.binop = L.epi.binop
        if L.epi.binop:
            e.other = self._view(m, prog, L.epi.other, n)
        return e

    def _build(self, progs, arena) -> rt.Graph:
        g = rt.Graph()
        host_descs = []
        self._keep = []                                # keep param structs alive
        self.nodes = []                                # (op, params, algorithmic info)
        self._node_member = []                         # member index of every graph node
        # 1. every member's launches as a chain of (op, params, info) items
        chains: list[list[tuple]] = []
        for m, (prog, n) in enumerate(zip(progs, self.batch)):
            items = []
            if n == 0:
                chains.append(items)
                continue
            ic = prog.input_im2col or (0, 0, 0, 0, 0, 0)
            ind = tuple(prog.input_dims) if len(prog.input_dims) == 3 else (prog.input_dims[0], 1, 1)
            pin = rt.InParams(self.dev_in + self.in_off[m], self._view(m, prog, "<input>", n),
                              *ic, *ind, getattr(prog, "input_split", 0))
            if self.gated:                             # the member waits for its input (dfx_execute_gated)
                gp = rt.GateParams(self.gate_flags + 4 * m)
                items.append((rt.OP_GATE, gp, dict(member=m, kind="gate", flops=0, bytes=0)))
            items.append((rt.OP_IN, pin, dict(member=m, kind="in", flops=0, bytes=self.in_sizes[m] * 3 // 2)))
            for L in prog.launches:
                if L.index in self.plans[m].skip:      # absorbed by the GEMM before it
                    continue
                for op, params in self._params(m, prog, L, n, host_descs):
                    info = self._algo(prog, L, n, op)
                    info["node"] = L.nodes[0]
                    if op == rt.OP_GEMM:
                        info["tiling"] = self.plans[m].tilings[L.index]
                        info["geom"] = {k: L.geom[k] for k in ("cin", "cout", "kh", "kw", "cb")}
                        info["gkey"] = self._group_key(prog, L, params)
                    items.append((op, params, info))
            pout = rt.OutParams(self._view(m, prog, prog.exit_value, n), self.dev_out + self.out_off[m])
            items.append((rt.OP_OUT, pout, dict(member=m, kind="out", flops=0, bytes=self.out_sizes[m] * 3 // 2)))
            chains.append(items)
        # 2. grouped GEMMs across members (north-star subsystem 4, DFX_GROUP_GEMM)
        active = sum(1 for c in chains if c)
        group = GROUP_GEMM if GROUP_GEMM != "auto" else active >= GROUP_AUTO_MEMBERS
        pairs = self._pair_chains(chains) if group and self.dag.mode == "concurrent" else []
        partner = {}                                   # (m, i) -> (m', i') matched item
        for (a, b, matches) in pairs:
            for ia, ib in matches:
                partner[(a, ia)] = (b, ib)
                partner[(b, ib)] = (a, ia)
        self.grouped_launches = sum(len(mt) for _, _, mt in pairs)
        # 3. graph nodes in dependency order: a matched pair becomes ONE launch once
        # both chains reach it (monotone matching: no cross-chain cycle)
        tail: dict[int, int] = {}                      # member -> last node id
        pos = [0] * len(chains)
        prev_tail = None
        seq = self.dag.mode == "sequential"

        def add(op, params, info, members):
            deps = sorted({tail[mm] for mm in members if mm in tail})
            nid = g.add(op, params, deps)
            for mm in members:
                tail[mm] = nid
            self._node_member.append(members[0])
            self.nodes.append((op, params, info))
            return nid

        order = [m for m in range(len(chains)) if chains[m]]
        # A/B (DFX_SLACK_DELAY=f): the members with slack (DFX_SLACK_FRAC) start only
        # once the critical member's chain is f of the way through (a graph edge from
        # that node to their first node), so their big-grid layers meet its late,
        # narrow layers instead of its wide early ones
        delay_after, delayed = None, set()
        if SLACK_DELAY > 0 and self.dag.mode == "concurrent" and any(self.sm_budget_slack):
            crit = max(order, key=lambda mm: len(chains[mm]))
            delayed = {mm for mm in order if self.sm_budget_slack[mm]}
            delay_after = (crit, int(SLACK_DELAY * len(chains[crit])))
            order = [crit] + [mm for mm in order if mm != crit]
        delay_nid = None
        progressed = True
        while progressed:
            progressed = False
            for m in order:
                items = chains[m]
                while pos[m] < len(items):
                    i = pos[m]
                    if seq and i == 0 and prev_tail is not None:
                        tail[m] = prev_tail            # sequential mode: after the previous member
                    op, params, info = items[i]
                    mate = partner.get((m, i))
                    if mate is not None:
                        b, ib = mate
                        if pos[b] != ib:                # wait for the partner chain to get there
                            break
                        gl = self._group_launch([items[i], chains[b][ib]], host_descs)
                        gi = dict(kind="gemm", member=m, node=f"{info['node']}+{chains[b][ib][2]['node']}",
                                  flops=info["flops"] + chains[b][ib][2]["flops"],
                                  bytes=info["bytes"] + chains[b][ib][2]["bytes"],
                                  weight_bytes=info.get("weight_bytes", 0) + chains[b][ib][2].get("weight_bytes", 0),
                                  grouped=[info["node"], chains[b][ib][2]["node"]],
                                  tiling=info["tiling"], geom=info["geom"])
                        add(rt.OP_GEMM, gl, gi, [m, b])
                        pos[b] += 1
                    elif i == 0 and m in delayed and delay_nid is not None:
                        tail[m] = delay_nid              # start after the critical chain's node
                        add(op, params, info, [m])
                    else:
                        add(op, params, info, [m])
                    if delay_after is not None and (m, i) == delay_after:
                        delay_nid = tail[m]
                    pos[m] += 1
                    progressed = True
                if pos[m] == len(items) and seq:
                    prev_tail = tail[m]
        assert all(p == len(c) for p, c in zip(pos, chains)), "grouped GEMM matching left a chain blocked"
        chain: dict[int, float] = {}
        for mm, (op_, _, info_) in zip(self._node_member, self.nodes):
            chain[mm] = chain.get(mm, 0.0) + _node_cost_us(info_)
        self.gate_order = sorted(range(len(progs)), key=lambda mm: (-chain.get(mm, 0.0), mm))
        if NODE_PRIORITY and self.dag.mode == "concurrent" and max(self.batch) <= PRIORITY_MAX_BATCH:
            self._prioritise(g)
        self._keep = [p for _, p, _ in self.nodes]
        if self._se_host:
            arr = (rt.SeFuse * len(self._se_host))(*self._se_host)
            rt.h2d(self.se_structs, C.addressof(arr), C.sizeof(arr), self.stream)
            rt.stream_sync(self.stream)
        if host_descs:
            assert len(host_descs) <= self.desc_capacity
            arr = (rt.GemmDesc * len(host_descs))(*host_descs)
            rt.h2d(self.descs, C.addressof(arr), C.sizeof(arr), self.stream)
            rt.stream_sync(self.stream)
        g.instantiate()
        self.kernel_nodes = len(g.kinds)
        return g

    # --- grouped GEMM across members
    @staticmethod
    def _group_key(prog, L, gl):
        """Launches that may share ONE grouped gemm_kernel launch: the one-tile kernel
        (no persistent walk, cluster split-K or depthwise epilogue), the same
        weight geometry and input map, same storage type and M2 form."""
        if gl.flags & (2 | 4 | 8 | 16) or gl.desc0.dw_k or gl.desc0.pre_mode or gl.m2:
            return None
        gm = L.geom
        src = prog.values[L.src]
        return (gm["cin"], gm["cout"], gm["kh"], gm["kw"], gm["sh"], gm["sw"], gm["ph"], gm["pw"], gm["cb"],
                src.h, src.w, bool(gm.get("tokens")), gl.dtype)

    def _pair_chains(self, chains):
        """Members paired two by two (most matchable GEMMs first); within a pair the
        GEMMs of equal group key are matched in order (longest common subsequence),
        so every cross-member edge points forward in both chains."""
        keyseq = [[(i, it[2].get("gkey")) for i, it in enumerate(c) if it[0] == rt.OP_GEMM and it[2].get("gkey")]
                  for c in chains]

        def lcs(x, y):
            nx, ny = len(x), len(y)
            dp = np.zeros((nx + 1, ny + 1), np.int32)
            for i in range(nx - 1, -1, -1):
                xi = x[i][1]
                row, nxt = dp[i], dp[i + 1]
                for j in range(ny - 1, -1, -1):
                    row[j] = nxt[j + 1] + 1 if xi == y[j][1] else max(nxt[j], row[j + 1])
            out, i, j = [], 0, 0
            while i < nx and j < ny:
                if x[i][1] == y[j][1]:
                    out.append((x[i][0], y[j][0]))
                    i += 1
                    j += 1
                elif dp[i + 1][j] >= dp[i][j + 1]:
                    i += 1
                else:
                    j += 1
            return out

        cands = []
        for a in range(len(chains)):
            for b in range(a + 1, len(chains)):
                if keyseq[a] and keyseq[b] and {k for _, k in keyseq[a]} & {k for _, k in keyseq[b]}:
                    mt = lcs(keyseq[a], keyseq[b])
                    if len(mt) >= GROUP_MIN:
                        cands.append((len(mt), a, b, mt))
        used, pairs = set(), []
        for _, a, b, mt in sorted(cands, key=lambda t: (-t[0], t[1], t[2])):
            if a not in used and b not in used:
                used |= {a, b}
                pairs.append((a, b, mt))
        return pairs

    def _group_launch(self, items, host_descs) -> rt.GemmLaunch:
        """ONE gemm_kernel launch over the problems of several members (ndesc > 1):
        descriptors copied contiguously into the device array, tiles numbered
        problem after problem (dfx_gemm.cu picks its problem by tile_begin)."""
        descs, at = [], 0
        for _, gl, _ in items:
            d = rt.GemmDesc()
            C.memmove(C.addressof(d), C.addressof(gl.desc0), C.sizeof(d))
            d.tile_begin = at
            at += d.tiles
            descs.append(d)
        slot = len(host_descs)
        host_descs.extend(descs)
        bn = max(d.bn for d in descs)
        planes = 2 if items[0][1].dtype in (rt.DT_F16X2, rt.DT_BF16X2) else 1
        gl = rt.GemmLaunch(self.descs + slot * C.sizeof(rt.GemmDesc), len(descs), at, bn, items[0][1].dtype,
                           gemm_slots(bn, at, self.dag.sm_count, 0, planes))
        return gl

    def _prioritise(self, g) -> None:
        """Concurrent members are independent branches of one graph; the query
        ends when the LONGEST dependent chain ends.  Members get node priorities
        by estimated chain latency (_node_cost_us summed over the member's nodes):
        the longest chain most urgent, so other branches' CTAs fill in around it
        instead of delaying it."""
        chain: dict[int, float] = {}
        for m, (op, _, info) in zip(self._node_member, self.nodes):
            chain[m] = chain.get(m, 0.0) + _node_cost_us(info)
        order = sorted(chain, key=lambda m: (-chain[m], m))
        least, greatest = g.set_priority(0, 0)
        prio = {m: min(least, greatest + r) for r, m in enumerate(order)}
        for nid, m in enumerate(self._node_member):
            g.set_priority(nid, prio[m])

    @staticmethod
    def _algo(prog: MemberProgram, L, n: int, op: int) -> dict:
        """Algorithmic FLOPs and HBM bytes of one launch (16-bit activations,
        unpadded weights): what a perfect kernel must move / compute."""
        es = 2 * planes_of(prog.precision)      # bytes per stored element
        def vbytes(name):
            v = prog.values[name]
            return n * v.h * v.w * v.c * es
        info = dict(member=prog.model_id, kind=L.kind, flops=0, bytes=0)
        out_b = vbytes(L.dst) if L.kind != COPY else vbytes(L.src)
        in_b = vbytes(L.src)
        other_b = vbytes(L.epi.other) if L.epi.other is not None else 0
        if L.epi.binop == 2:                      # per-(n, c) scale vector
            other_b = n * prog.values[L.epi.other].c * 2
        if L.kind == GEMM:
            g = L.geom
            out = prog.values[L.dst]
            macs = n * out.h * out.w * g["cout"] * g["cin"] * g["kh"] * g["kw"]
            wbytes = g["cout"] * g["cin"] * g["kh"] * g["kw"] * es
            if op == rt.OP_SPLITK:
                info.update(kind="splitk", bytes=out_b + other_b)
            else:
                info.update(flops=2 * macs, bytes=wbytes + in_b + out_b + other_b, weight_bytes=wbytes)
        elif L.kind == DWCONV:
            g = L.geom
            out = prog.values[L.dst]
            info.update(flops=2 * n * out.h * out.w * out.c * g["kh"] * g["kw"],
                        bytes=in_b + out_b + out.c * g["kh"] * g["kw"] * 4)
        elif L.kind == SE:
            g = L.geom
            info.update(flops=4 * n * g["c"] * g["cr"], bytes=in_b + out_b + 2 * 2 * g["c"] * g["cr"])
        elif L.kind == DWSE:
            g = L.geom
            out = prog.values[L.dst]
            info.update(flops=2 * n * out.h * out.w * out.c * g["kh"] * g["kw"] + 4 * n * g["c"] * g["cr"],
                        bytes=in_b + out_b + out.c * g["kh"] * g["kw"] * 4 + 2 * 2 * g["c"] * g["cr"])
        elif L.kind == ATTN:
            g = L.geom
            info.update(flops=4 * n * g["seq"] * g["seq"] * g["c"], bytes=in_b + out_b)
        elif L.kind == LN:
            out = prog.values[L.dst]            # rows actually normalised
            info.update(bytes=2 * n * out.w * out.c * 2)
        else:
            info.update(bytes=in_b + out_b + other_b)
        return info

    def profile_nodes(self, reps: int = 8, kinds=None) -> list[dict]:
        """Per-node device time: each graph node (same params as in the step) is
        put ``reps`` times in a chain inside its own CUDA graph, launched once to
        warm up and once between CUDA events on this instance's stream; the
        node time is the event interval / reps (host launch gaps excluded, the
        ~1 us graph node-to-node gap included, as inside the real step).
        A GEMM node that uses split-K is timed together with its reduction."""
        out = []
        i = 0
        nodes = self.nodes
        while i < len(nodes):
            op, params, info = nodes[i]
            group = [(op, params)]
            if op == rt.OP_GEMM and i + 1 < len(nodes) and nodes[i + 1][0] == rt.OP_SPLITK:
                group.append(nodes[i + 1][:2])
                i += 1
            i += 1
            if op == rt.OP_GATE or (kinds is not None and info["kind"] not in kinds):
                continue
            g = rt.Graph()
            last = None
            for _ in range(reps):
                for o, p in group:
                    last = g.add(o, p, [] if last is None else [last])
            g.instantiate()
            g.launch(self.stream)
            e0, e1 = rt.Event(), rt.Event()
            e0.record(self.stream)
            g.launch(self.stream)
            e1.record(self.stream)
            ms = e0.elapsed_ms(e1) / reps
            g.destroy()
            out.append(dict(info, op=op, ms=ms, split=len(group) > 1))
        return out

    def _set_l2_prefetch(self, gl, m, prog: MemberProgram, L) -> None:
        """Ranges for dfx_gemm_launch.l2_pf: the weight blob of the member's next GEMM
        launch and the next SE launch's blobs (one span) when it comes before that
        GEMM; else (DFX_L2_PREFETCH_DEPTH=2) the weight-bearing launch after the next
        GEMM.  Each capped at 16 MB (256-B units in 16 bits)."""
        arena, skip = self.dag.arena, self.plans[m].skip

        def span(X):
            if X.kind == GEMM:
                k = X.blobs["weight"]
                return arena.addr(m, k), prog.blobs[k].nbytes
            keys = list(X.blobs.values())
            lo = min(arena.addr(m, k) for k in keys)
            hi = max(arena.addr(m, k) + prog.blobs[k].nbytes for k in keys)
            total = sum(prog.blobs[k].nbytes for k in keys)
            if hi - lo > 2 * total:              # not adjacent in the segment: the largest blob
                k = max(keys, key=lambda k: prog.blobs[k].nbytes)
                lo, hi = arena.addr(m, k), arena.addr(m, k) + prog.blobs[k].nbytes
            return lo, hi - lo

        after = False
        gemm_span = se_span = extra = None
        for X in prog.launches:
            if X.index == L.index:
                after = True
                continue
            if not after or X.index in skip or X.kind not in (GEMM, SE):
                continue
            if gemm_span is None:
                if X.kind == SE:
                    se_span = se_span or span(X)
                else:
                    gemm_span = span(X)
                    if se_span is not None or L2_PREFETCH_DEPTH < 2:
                        break
            else:
                extra = span(X)
                break
        units, ptrs = 0, []
        for sp in (gemm_span, se_span or extra):
            if sp is None:
                continue
            u = min(sp[1] >> 8, 0xFFFF)
            if u:
                units |= u << (16 * len(ptrs))
                ptrs.append(sp[0])
        gl.l2_pf_units = units
        for i, a in enumerate(ptrs):
            gl.l2_pf[i] = a

    def _params(self, m, prog: MemberProgram, L, n, host_descs):
        arena = self.dag.arena
        src = self._view(m, prog, L.src, n)
        if L.kind == GEMM:
            geo, t = L.geom, self.plans[m].tilings[L.index]
            out = self._view(m, prog, L.dst, n)
            if geo.get("tokens"):            # fold (n, 1, L) token rows into one M axis
                src, out = _fold_rows(src), _fold_rows(out)
            d = rt.GemmDesc()
            d.tmap_a = rt.tmap_act(src, geo["cb"], t["tq"], t["tp"], t["tn"], geo["sw"], geo["sh"])
            # split precision: [W_hi; W_lo] rows, the kernel loads lo rows at cout + co
            d.tmap_b = rt.tmap_weights(arena.addr(m, L.blobs["weight"]), geo["cout"] * planes_of(prog.precision),
                                       geo["k"], geo["cb"], t["bn"], self.dtype)
            d.n, d.p, d.q = out.n, out.h, out.w
            d.tn, d.tp, d.tq = t["tn"], t["tp"], t["tq"]
            d.mt_n, d.mt_p, d.mt_q, d.nt = t["mt_n"], t["mt_p"], t["mt_q"], t["nt"]
            d.r, d.s = geo["kh"], geo["kw"]
            d.stride_h, d.stride_w, d.pad_h, d.pad_w = geo["sh"], geo["sw"], geo["ph"], geo["pw"]
            d.cb, d.cblocks, d.ksteps, d.kpack = geo["cb"], geo["cblocks"], geo["ksteps"], t["kpack"]
            d.stages, d.splits, d.stages_per_split = t["stages"], t["splits"], t["sps"]
            d.bn, d.cout, d.tile_begin, d.tiles = t["bn"], geo["cout"], 0, t["tiles"]
            d.m2 = t.get("m2", 0)
            d.out = out
            if t.get("dw") is not None:      # depthwise epilogue: `out` is the dw output
                D = next(x for x in prog.launches if x.index == t["dw"])
                dg = D.geom
                d.out = self._view(m, prog, D.dst, n)
                d.dw_w = arena.addr(m, D.blobs["weight"])
                d.dw_alpha = arena.addr(m, D.blobs["alpha"]) if "alpha" in D.blobs else None
                d.dw_beta = arena.addr(m, D.blobs["beta"]) if "beta" in D.blobs else None
                d.dw_k, d.dw_s, d.dw_pad = dg["kh"], dg["sh"], dg["ph"]
                d.dw_act = rt.ACT[D.epi.act1]
                if t.get("se") is not None:  # the SE after it too: `out` is the SE's output
                    S = next(x for x in prog.launches if x.index == t["se"])
                    sg = S.geom
                    d.out = self._view(m, prog, S.dst, n)
                    addr = (lambda r: arena.addr(m, S.blobs[r]) if r in S.blobs else None)
                    k = len(self._se_host)
                    f = rt.SeFuse()
                    f.w1, f.b1, f.w2, f.b2 = addr("w1"), addr("b1"), addr("w2"), addr("b2")
                    f.scratch = self.se_scratch + self._se_scratch_used
                    self._se_scratch_used += _align(t["nt"] * n * 512 * 4)
                    f.sync = self.se_sync + 16 * k
                    f.c, f.cr = sg["c"], sg["cr"]
                    f.act1, f.act2 = rt.ACT[sg["act1"]], rt.ACT[sg["act2"]]
                    f.ctas = t["tiles"]
                    self._se_host.append(f)
                    d.se = self.se_structs + k * C.sizeof(rt.SeFuse)
                elif t.get("squeeze") is not None:   # the SE after it reads our channel means
                    S = next(x for x in prog.launches if x.index == t["squeeze"])
                    k = len(self._se_host)
                    f = rt.SeFuse()
                    f.mode, f.c = 1, S.geom["c"]
                    f.pooled = self.se_pooled + self._pool_used
                    self._pool_used += _align(n * 4 * 4096)
                    self._squeeze_ptr[(m, S.index)] = f.pooled
                    self._se_host.append(f)
                    d.se = self.se_structs + k * C.sizeof(rt.SeFuse)
            epi = self._epi(m, prog, L, n)
            if geo.get("tokens") and epi.binop:
                epi.other = _fold_rows(epi.other)
            d.epi = epi
            if L.pre is not None:            # A prologue transform (lower.fold_pre_transforms)
                if L.pre.binop == 2:
                    gv = self._view(m, prog, L.pre.other, n)
                    d.pre_mode, d.pre_scale, d.pre_pitch = 2, gv.base + 2 * gv.coff, gv.pitch
                else:
                    d.pre_mode = 1
                    d.pre_scale = arena.addr(m, L.blobs["pre_alpha"])
                    d.pre_shift = arena.addr(m, L.blobs["pre_beta"]) if "pre_beta" in L.blobs else None
                d.pre_act = rt.ACT[L.pre.act1]
                d.pre_cin = geo["cin"]
            csplit = bool(t["csplit"])
            d.ws = (self.ws + self.ws_off[m]) if t["splits"] > 1 and not csplit else None
            fixup = t["splits"] > 1 and SPLITK_MODE == "fixup"
            if fixup:                  # per-output-tile arrival counters (in-kernel fixup)
                d.counters = self.counters + 4 * self._ctr_used
                self._ctr_used += t["mt_n"] * t["mt_p"] * t["mt_q"] * t["nt"]
            slot = len(host_descs)
            host_descs.append(d)
            self.gemm_count += 1
            planes = planes_of(prog.precision)
            slot_bytes = (128 * 64 * 2 + t["bn"] * 128) * planes     # dfx_common.cuh gemm_slot_bytes
            gl = rt.GemmLaunch(self.descs + slot * C.sizeof(rt.GemmDesc), 1, t["tiles"], t["bn"],
                               self.dtype, t.get("nslots") or gemm_slots(t["bn"], t["tiles"], self.dag.sm_count,
                                                                         t.get("m2", 0), planes))
            gl.m2 = t.get("m2", 0)
            gl.se_cr = t.get("se_cr", 0)
            if csplit:
                gl.flags |= 8                # cluster split-K (DSMEM reduction, no splitk node)
                need = 128 * (t["bn"] + 4) * 4          # the fp32 partial tile parks in the slots
                gl.nslots = max(gl.nslots, -(-need // slot_bytes))
            budget = self.sm_budget[m] if t.get("dw") is None and not csplit else 0
            if GEMM_PERSIST and not gl.m2 and t["splits"] == 1 and t.get("dw") is None and \
                    (t["tiles"] > (PERSIST_MIN_WAVES_X2 if planes > 1 else PERSIST_MIN_WAVES)
                     * self.dag.sm_count or budget):
                gl.max_ctas = budget
                gl.flags |= 2                # persistent kernel for multi-wave layers
                # bn > 64: one CTA per SM, as deep a ring as smem allows; bn <= 64: two
                # CTAs per SM (dfx_api.cu), 4 slots each
                if t["bn"] > 64:
                    vec = 2 * ((geo["cout"] + 15) // 16 * 16) * 4 if geo["cout"] <= 1024 else 0
                    gl.nslots = max(2, min(8, (GEMM_SMEM_LIMIT - GEMM_SMEM_FIXED - vec
                                               - (8 * 2560 if GEMM_DRAIN_STAGED else 0))
                                           // slot_bytes))
                elif planes > 1 and PERSIST_ONE_CTA_X2:      # one CTA per SM, deeper ring (A/B)
                    gl.nslots = max(2, min(8, (GEMM_SMEM_LIMIT - GEMM_SMEM_FIXED) // slot_bytes))
                else:
                    gl.nslots = 4 if planes == 1 else 2
            if W_EVICT_FIRST and not gl.flags & 2 and t["mt_n"] * t["mt_p"] * t["mt_q"] <= 2:
                gl.flags |= 32               # weights read by <= 2 CTAs each: L2 evict_first
            if L2_PREFETCH and n <= L2_PREFETCH_MAX_BATCH:
                self._set_l2_prefetch(gl, m, prog, L)
            if GEMM_DRAIN_STAGED:
                gl.flags |= 4                # smem-transposed epilogue drain (A/B)
            if GEMM_EARLY_PDL:
                gl.flags |= 16               # launch_dependents right after the prologue (A/B)
            gl.desc0 = d                    # single problem: descriptor in kernel-param space
            yield rt.OP_GEMM, gl
            if t["splits"] > 1 and not fixup and not csplit:
                yield rt.OP_SPLITK, rt.SplitKParams(self.ws + self.ws_off[m], t["splits"],
                                                    out.n * out.h * out.w, geo["cout"],
                                                    t["nt"] * t["bn"], out, epi)
        elif L.kind == DWCONV:
            geo = L.geom
            p = rt.DwconvParams(src, self._view(m, prog, L.dst, n), arena.addr(m, L.blobs["weight"]),
                                geo["kh"], geo["kw"], geo["sh"], geo["sw"], geo["ph"], geo["pw"],
                                self._epi(m, prog, L, n))
            yield rt.OP_DWCONV, p
        elif L.kind == POOL:
            geo = L.geom
            yield rt.OP_POOL, rt.PoolParams(src, self._view(m, prog, L.dst, n), geo["kh"], geo["kw"],
                                            geo["sh"], geo["sw"], geo["ph"], geo["pw"],
                                            geo["is_max"], geo["cip"])
        elif L.kind == GAP:
            yield rt.OP_GAP, rt.GapParams(src, self._view(m, prog, L.dst, n))
        elif L.kind == EW:
            yield rt.OP_EW, rt.EwParams(src, self._view(m, prog, L.dst, n), self._epi(m, prog, L, n))
        elif L.kind == COPY:
            cv = self._view(m, prog, L.geom["concat"], n)
            out = rt.View(cv.base, n, src.h, src.w, src.c, cv.pitch, L.geom["coff"], self.dtype)
            yield rt.OP_EW, rt.EwParams(src, out, rt.Epilogue())
        elif L.kind == LN:
            addr = (lambda r: arena.addr(m, L.blobs[r]) if r in L.blobs else None)
            yield rt.OP_LN, rt.LnParams(src, self._view(m, prog, L.dst, n), addr("gamma"),
                                        addr("beta"), L.geom["eps"], L.geom["norm"])
        elif L.kind == TOKENS:
            yield rt.OP_TOKENS, rt.TokensParams(src, self._view(m, prog, L.dst, n),
                                                arena.addr(m, L.blobs["class_token"]),
                                                arena.addr(m, L.blobs["pos_embedding"]))
        elif L.kind == ATTN:
            yield rt.OP_ATTN, rt.AttnParams(src, self._view(m, prog, L.dst, n), L.geom["heads"],
                                            1.0 / math.sqrt(L.geom["c"] // L.geom["heads"]))
        elif L.kind == SE:
            geo = L.geom
            addr = (lambda r: arena.addr(m, L.blobs[r]) if r in L.blobs else None)
            yield rt.OP_SE, rt.SeParams(src, self._view(m, prog, L.dst, n), addr("w1"), addr("b1"),
                                        addr("w2"), addr("b2"), geo["cr"], rt.ACT[geo["act1"]],
                                        rt.ACT[geo["act2"]],
                                        geo.get("apply", 0) | self._se_unstaged(prog, geo, n),
                                        self._squeeze_ptr.get((m, L.index)))
        elif L.kind == DWSE:
            geo = L.geom
            addr = (lambda r: arena.addr(m, L.blobs[r]) if r in L.blobs else None)
            dep = self._epi(m, prog, L, n)
            yield rt.OP_DWSE, rt.DwseParams(src, self._view(m, prog, L.dst, n), addr("weight"),
                                            geo["kh"], geo["kw"], geo["sh"], geo["sw"], geo["ph"], geo["pw"],
                                            dep, addr("w1"), addr("b1"), addr("w2"), addr("b2"), geo["cr"],
                                            rt.ACT[geo["act1"]], rt.ACT[geo["act2"]],
                                            int(n < SE_UNSTAGED_BATCH))
        else:
            raise AssertionError(L.kind)

    @staticmethod
    def _se_unstaged(prog, geo, n) -> int:
        """se_params.apply bits for the FC weights: 2 = read from L2 instead of staged
        per CTA (large batches: the clusters of smem-heavy CTAs could not be
        co-scheduled), 2|4 = stage only the fc1 slices (split precision, hi + lo
        slices of both FCs beyond the cluster kernel's smem budget,
        dfx_common.cuh se_smem_bytes / kSeSmemBudget)."""
        if n >= SE_UNSTAGED_BATCH:
            return 2
        cs = -(-geo["c"] // 128) * 8
        one = ((cs * geo["cr"] * 2 + 15) & ~15) * planes_of(prog.precision)
        if 2 * one <= 190 * 1024:
            return 0
        return 2 | 4 if one <= 190 * 1024 else 2

    # --- execution
    def stage_inputs(self, xs) -> None:
        """Copy each member's inputs into the pinned staging buffer.  A member's entry
        is one (batch, ...) array or a list of per-sample arrays (copied straight
        in: no intermediate np.stack, which doubled the host copy per query)."""
        hb = np.frombuffer((C.c_uint8 * max(self.in_bytes, 16)).from_address(self.host_in),
                           dtype=np.uint8)
        for m, x in enumerate(xs):
            if isinstance(x, (list, tuple)):
                at = self.in_off[m]
                for t in x:
                    raw = np.ascontiguousarray(t, dtype=np.float32).view(np.uint8).reshape(-1)
                    hb[at:at + raw.size] = raw
                    at += raw.size
            else:
                raw = np.ascontiguousarray(x, dtype=np.float32).view(np.uint8).reshape(-1)
                hb[self.in_off[m]:self.in_off[m] + raw.size] = raw

    def read_outputs(self) -> list[np.ndarray]:
        hb = np.frombuffer((C.c_uint8 * max(self.out_bytes, 16)).from_address(self.host_out),
                           dtype=np.uint8)
        outs = []
        for m, p in enumerate(self.dag.programs):
            raw = hb[self.out_off[m]:self.out_off[m + 1]].copy().view(np.float32)
            outs.append(raw.reshape((self.batch[m],) + tuple(p.output_dims)))
        return outs

    def run(self, xs: list[np.ndarray]) -> list[np.ndarray]:
        """End to end: gather -> H2D -> graph -> D2H -> sync (dfx_execute_gather: the
        host copies into the pinned staging run on a thread pool and overlap the
        H2D).  DFX_E2E_GATHER=0: one-thread staging + dfx_execute."""
        if not E2E_GATHER:
            self.stage_inputs(xs)
            self.open_gates()
            self.graph.execute(self.host_in, self.dev_in, self.in_bytes, self.host_out, self.dev_out,
                               self.out_bytes, self.stream)
            return self.read_outputs()
        keep = []
        for m, x in enumerate(xs):
            parts = x if isinstance(x, (list, tuple)) else [x]
            total = 0
            for t in parts:
                a = np.ascontiguousarray(t, dtype=np.float32)
                keep.append(a)
                total += a.nbytes
            if total != self.in_sizes[m]:
                raise ValueError(f"member {m}: {total} input bytes, expected {self.in_sizes[m]}")
        if self.gated:
            # sources member by member, the longest chain first (its branch starts first)
            per = []
            at = 0
            for m, x in enumerate(xs):
                k = len(x) if isinstance(x, (list, tuple)) else 1
                per.append(keep[at:at + k])
                at += k
            order = self.gate_order
            lst = [(m, a) for m in order for a in per[m]]
            srcs = (C.c_void_p * len(lst))(*[a.ctypes.data for _, a in lst])
            sizes = (C.c_size_t * len(lst))(*[a.nbytes for _, a in lst])
            smem = (C.c_int * len(lst))(*[m for m, _ in lst])
            moff = (C.c_size_t * len(xs))(*self.in_off[:len(xs)])
            mbytes = (C.c_size_t * len(xs))(*self.in_sizes)
            self.graph.execute_gated(srcs, sizes, smem, moff, mbytes, self.host_in, self.dev_in, self.gate_flags,
                                     self.gate_one, self.host_out, self.dev_out, self.out_bytes, self.stream,
                                     self.copy_stream)
            return self.read_outputs()
        srcs = (C.c_void_p * len(keep))(*[a.ctypes.data for a in keep])
        sizes = (C.c_size_t * len(keep))(*[a.nbytes for a in keep])
        self.graph.execute_gather(srcs, sizes, self.host_in, self.dev_in, self.host_out, self.dev_out,
                                  self.out_bytes, self.stream)
        return self.read_outputs()

    def upload_inputs(self, xs):
        self.stage_inputs(xs)
        rt.h2d(self.dev_in, self.host_in, self.in_bytes, self.stream)
        rt.stream_sync(self.stream)

    def open_gates(self):
        """Every member's gate open (inputs already resident: device-timed steps,
        profiling, the manager's replays): 0x01010101 in each flag, stream-ordered."""
        if self.gated:
            rt.memset(self.gate_flags, 1, 4 * max(len(self.dag.programs), 4), self.stream)

    def launch_graph(self):
        self.open_gates()
        self.graph.launch(self.stream)

    def sync(self):
        rt.stream_sync(self.stream)

    def download_outputs(self) -> list[np.ndarray]:
        rt.d2h(self.host_out, self.dev_out, self.out_bytes, self.stream)
        rt.stream_sync(self.stream)
        return self.read_outputs()

    def free(self):
        self.graph.destroy()
        for p in (self.act, self.ws, self.counters, self.descs, self.dev_in, self.dev_out,
                  self.se_structs, self.se_sync, self.se_scratch, self.se_pooled, self.gate_flags):
            rt.free(p)
        rt.host_free(self.gate_one)
        rt.stream_destroy(self.copy_stream)
        rt.host_free(self.host_in)
        rt.host_free(self.host_out)
        rt.stream_destroy(self.stream)


# measured batch-1 latency floor of one dependent node per kind, us (layer tables
# of the B200 bench: GEMM ~6.5, SE cluster ~7, depthwise ~4.5, split-K ~3, rest ~2.5)
_NODE_BASE_US = {"gemm": 6.5, "se": 7.0, "dwconv": 4.5, "splitk": 3.0, "dwse": 9.0}


def _node_cost_us(info: dict) -> float:
    """Latency estimate of one graph node for the priority ranking: a per-kind
    floor plus its bytes at 3 TB/s and its FLOPs at 300 TFLOP/s."""
    return (_NODE_BASE_US.get(info.get("kind"), 2.5) + info.get("bytes", 0) / 3e6
            + info.get("flops", 0) / 3e8)


class DeviceDag:
    """A fused DAG resident on one GPU."""

    def __init__(self, members, device: int = 0, mode: str = "concurrent", arena=None,
                 programs=None, precision: str = "fp16"):
        if mode not in ("concurrent", "sequential"):
            raise ValueError(mode)
        self.device, self.mode, self.precision = device, mode, precision
        rt.init_device(device)
        sm = C.c_int()
        rt.call("dfx_device_info", C.c_int(device), C.byref(sm), None, None, None)
        self.sm_count = sm.value
        self.members = list(members)
        self.programs = programs or [program_for(g, w, precision) for g, w in self.members]
        if arena is None:
            arena = WeightArena(self.programs, device)
            arena.upload()
        self.arena = arena
        self._pool: dict[tuple, list[ExecInstance]] = {}
        self._all: list[ExecInstance] = []
        self._lock = threading.Lock()

    @property
    def swap_in_ms(self) -> float:
        return self.arena.upload_ms

    def acquire(self, batch: tuple[int, ...]) -> ExecInstance:
        with self._lock:
            free = self._pool.setdefault(batch, [])
            if free:
                return free.pop()
        inst = ExecInstance(self, batch)
        with self._lock:
            self._all.append(inst)
        return inst

    def release(self, inst: ExecInstance) -> None:
        with self._lock:
            self._pool.setdefault(inst.batch, []).append(inst)

    def execute(self, xs: list) -> list[np.ndarray]:
        """xs[m]: a (batch, ...) array, or a list of per-sample arrays."""
        batch = tuple(len(x) if isinstance(x, (list, tuple)) else int(x.shape[0]) for x in xs)
        inst = self.acquire(batch)
        try:
            return inst.run(xs)
        finally:
            self.release(inst)

    def swapped(self, index: int, incoming, upload: bool = True) -> "DeviceDag":
        g, w = incoming
        prog = program_for(g, w, self.precision)
        arena = self.arena.clone_for_swap()
        ms = arena.replace_member(index, prog, upload=upload)
        members = list(self.members)
        members[index] = incoming
        programs = list(self.programs)
        programs[index] = prog
        out = DeviceDag(members, self.device, self.mode, arena=arena, programs=programs,
                        precision=self.precision)
        out.last_swap_ms = ms
        out.last_swap = dict(arena.last_swap, member=index)
        return out

    def free_instances(self):
        with self._lock:
            for inst in self._all:
                inst.free()
            self._all.clear()
            self._pool.clear()

    def free(self):
        """Swap-out: every execution instance and this image's arena references
        (device blocks shared with a swapped DAG stay until it is freed too)."""
        self.free_instances()
        self.arena.free()
