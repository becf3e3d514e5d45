"""Packed-arena files: a fused DAG's device weight arena on disk, so swap-in is
one file read into pinned memory + ONE H2D, with no FIWT parse and no lowering
(SURVEY.md §8(f) row 2, next to the reference's FIWT format,
/root/reference/pkg/src/dagfuse/model_io.py:83-127).

Layout (little-endian):

    b"DFXPACK1" | u64 H | H bytes JSON header | u64 P | P bytes program table
    | zero pad to a 4096-B boundary | the arena bytes (``header["total"]``)

* The JSON header holds the format version, precision, dag id, every member's
  graph (``model_io.graph_to_dict``, the reference's graph JSON), its weight
  tensor specs, its arena segment and the byte offset of every packed blob.
* The program table is the lowered launch list of each member
  (``lower.MemberProgram`` with the blob arrays left out) as JSON: dataclasses
  from a fixed whitelist and base64 arrays, so reading a file never runs code
  from it.  It is a cache written by ``save_packed`` for the same library
  build (the layout is re-derived and checked at load), not an interchange
  format.
* The arena bytes are exactly what ``device.WeightArena`` uploads: 16-bit GEMM
  weights, fp32 epilogue vectors, 256-B aligned, member segments in member
  order.

``load_packed`` reads the arena straight into its host staging buffer (parallel
``preadv`` chunks, no intermediate copy), rebuilds the blobs as zero-copy views
of it, uploads with one cudaMalloc + one cudaMemcpyAsync and returns a FusedDag
whose device image is attached -- ``execute_fused`` / ``swap_subgraph`` work
on it as on any loaded DAG.  Its members carry ``PackedWeights`` (specs only):
the fp32 weights never leave the disk, so the CPU oracle cannot run on them.
"""

from __future__ import annotations

import copy
import ctypes as C
import json
import struct
import time
from pathlib import Path

import numpy as np

from . import fuse, model_io
from .graph_ir import TensorSpec, WeightStore

MAGIC = b"DFXPACK1"
VERSION = 2                  # 2: program table as JSON (was pickle)
PAGE = 4096


class PackedWeights(WeightStore):
    """Weight specs of a member loaded from a packed file; the values exist only
    in the device arena (16-bit, packed), so reading them raises."""

    def __init__(self, specs: dict[str, TensorSpec]):
        super().__init__()
        self._t = {name: (spec, None) for name, spec in specs.items()}

    def put(self, name, spec, values) -> None:
        raise TypeError("PackedWeights is read-only")

    def values(self, name: str):
        raise LookupError(f"weight {name!r} of a packed DAG lives only in the device arena")

    array = values


# The lowered programs travel as JSON: dataclasses of lower.py (a fixed whitelist)
# and numpy arrays (dtype, shape, base64 bytes).  Loading a packed file therefore
# never executes code from it (no pickle).
def _program_classes():
    from .lower import Buffer, Epi, Launch, MemberProgram, Value
    return {c.__name__: c for c in (Buffer, Epi, Launch, MemberProgram, Value)}


def _enc(x):
    import base64
    import dataclasses
    if dataclasses.is_dataclass(x) and not isinstance(x, type):
        return {"__dc__": type(x).__name__,
                "f": {f.name: _enc(getattr(x, f.name)) for f in dataclasses.fields(x)}}
    if isinstance(x, np.ndarray):
        a = np.ascontiguousarray(x)
        return {"__nd__": a.dtype.str, "shape": list(a.shape), "b64": base64.b64encode(a.tobytes()).decode()}
    if isinstance(x, np.generic):
        return x.item()
    if isinstance(x, tuple):
        return {"__t__": [_enc(v) for v in x]}
    if isinstance(x, list):
        return [_enc(v) for v in x]
    if isinstance(x, dict):
        if not all(isinstance(k, str) for k in x):
            return {"__kv__": [[_enc(k), _enc(v)] for k, v in x.items()]}
        return {"__d__": {k: _enc(v) for k, v in x.items()}}
    if x is None or isinstance(x, (bool, int, float, str)):
        return x
    raise TypeError(f"cannot serialise {type(x).__name__} in a program table")


def _dec(x, classes):
    import base64
    if isinstance(x, list):
        return [_dec(v, classes) for v in x]
    if not isinstance(x, dict):
        return x
    if "__dc__" in x:
        cls = classes.get(x["__dc__"])
        if cls is None:
            raise ValueError(f"unexpected type {x['__dc__']!r} in a program table")
        return cls(**{k: _dec(v, classes) for k, v in x["f"].items()})
    if "__nd__" in x:
        return np.frombuffer(base64.b64decode(x["b64"]), dtype=np.dtype(x["__nd__"])).reshape(x["shape"]).copy()
    if "__t__" in x:
        return tuple(_dec(v, classes) for v in x["__t__"])
    if "__kv__" in x:
        return {_dec(k, classes): _dec(v, classes) for k, v in x["__kv__"]}
    if "__d__" in x:
        return {k: _dec(v, classes) for k, v in x["__d__"].items()}
    raise ValueError("malformed program table")


def _program_table(programs) -> bytes:
    metas = []
    for p in programs:
        m = copy.copy(p)
        m.blobs = {k: (str(v.dtype), tuple(v.shape)) for k, v in p.blobs.items()}
        metas.append(m)
    return json.dumps([_enc(m) for m in metas]).encode()


def _read_program_table(raw: bytes) -> list:
    classes = _program_classes()
    out = []
    for d in json.loads(raw):
        m = _dec(d, classes)
        m.debug_f32 = {}
        out.append(m)
    return out


def save_packed(dag: fuse.FusedDag, path, precision: str = "fp16") -> dict:
    """Lower + pack ``dag`` and write it to ``path``; returns the header."""
    from .device import arena_layout, fill_arena, program_for
    graphs = [fuse._as_graph(sg) for sg in dag.subgraphs]
    programs = [program_for(g, sg.weight_binding, precision) for g, sg in zip(graphs, dag.subgraphs)]
    layout, segments, total = arena_layout(programs)
    header = dict(version=VERSION, precision=precision, dag_id=dag.dag_id, total=total,
                  mem_estimate_mib=dag.total_mem_estimate_mib, members=[
        dict(model_id=sg.model_id, graph=model_io.graph_to_dict(g),
             weights={n: list(sg.weight_binding.spec(n).dims) for n in sg.weight_binding.names()},
             segment=list(seg), blobs={k: int(off) for k, off in lay.items()})
        for sg, g, seg, lay in zip(dag.subgraphs, graphs, segments, layout)])
    hdr = json.dumps(header, sort_keys=True).encode()
    table = _program_table(programs)
    head = MAGIC + struct.pack("<Q", len(hdr)) + hdr + struct.pack("<Q", len(table)) + table
    data_off = -(-len(head) // PAGE) * PAGE
    buf = np.zeros(total, np.uint8)
    fill_arena(buf, programs, layout)
    with open(path, "wb") as f:
        f.write(head)
        f.write(b"\0" * (data_off - len(head)))
        buf.tofile(f)
    return header


def read_header(path) -> tuple[dict, list, int]:
    """(header, program table, byte offset of the arena) of a packed file."""
    with open(path, "rb") as f:
        if f.read(8) != MAGIC:
            raise ValueError(f"{path}: not a packed-arena file")
        (hn,) = struct.unpack("<Q", f.read(8))
        header = json.loads(f.read(hn))
        if header.get("version") != VERSION:
            raise ValueError(f"{path}: packed-arena version {header.get('version')} != {VERSION}")
        (pn,) = struct.unpack("<Q", f.read(8))
        table = _read_program_table(f.read(pn))
        data_off = -(-(16 + hn + 8 + pn) // PAGE) * PAGE
    return header, table, data_off


READ_THREADS = 8
READ_CHUNK = 16 << 20


def _pread_all(path, buf: np.ndarray, offset: int) -> int:
    """Fill ``buf`` from ``path`` at ``offset`` with READ_THREADS parallel preadv
    calls (the GIL is released in the syscall; one thread copies page cache at
    ~4.5 GB/s); returns the bytes read."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    fd = os.open(path, os.O_RDONLY)
    try:
        mv = memoryview(buf)
        chunks = [(o, min(READ_CHUNK, buf.size - o)) for o in range(0, buf.size, READ_CHUNK)]

        def rd(c):
            o, n = c
            done = 0
            while done < n:
                k = os.preadv(fd, [mv[o + done:o + n]], offset + o + done)
                if k <= 0:
                    break
                done += k
            return done

        with ThreadPoolExecutor(READ_THREADS) as ex:
            return sum(ex.map(rd, chunks))
    finally:
        os.close(fd)


def load_packed(path, device: int = 0, mode: str = "concurrent", pinned: bool = False) -> fuse.FusedDag:
    """Swap a packed DAG in: one file read, one cudaMalloc, one H2D.

    ``pinned=False`` (default) reads into pageable memory and lets the driver
    stage the H2D: allocating and pinning 0.6 GB with cudaHostAlloc costs more
    (measured ~0.3 s) than the pageable copy loses.  ``pinned=True`` reads into
    a pinned buffer (worth it when the same arena is re-uploaded many times).
    The returned DAG has its device image attached; the phase timings are on
    ``fuse.device_image(dag).arena`` (header_ms, alloc_ms, read_ms, malloc_ms,
    memcpy_ms, dag_ms, load_ms)."""
    from . import runtime as rt
    from .device import DeviceDag, WeightArena, arena_layout
    t0 = time.perf_counter()
    header, programs, data_off = read_header(path)
    total = int(header["total"])
    rt.init_device(device)
    t1 = time.perf_counter()
    if pinned:
        host = rt.host_alloc(total)
        hb = np.frombuffer((C.c_uint8 * total).from_address(host), dtype=np.uint8)
    else:
        hb = np.empty(total, np.uint8)
        host = hb.ctypes.data
    t2 = time.perf_counter()
    got = _pread_all(path, hb, data_off)
    t3 = time.perf_counter()
    if got != total:
        if pinned:
            rt.host_free(host)
        raise ValueError(f"{path}: truncated arena ({got} of {total} bytes)")
    members = []
    for p, m in zip(programs, header["members"]):
        blobs = {}
        for key in sorted(p.blobs):
            dt, shape = p.blobs[key]
            off = m["blobs"][key]
            n = int(np.prod(shape, dtype=np.int64)) * np.dtype(dt).itemsize
            blobs[key] = hb[off:off + n].view(dt).reshape(shape)
        p.blobs = blobs
        p.precision = header["precision"]
        g = model_io.graph_from_dict(m["graph"])
        members.append((g, PackedWeights({n: TensorSpec(tuple(d)) for n, d in m["weights"].items()})))
    layout, segments, tot2 = arena_layout(programs)
    if tot2 != total or [dict(l) for l in layout] != [m["blobs"] for m in header["members"]]:
        if pinned:
            rt.host_free(host)
        raise ValueError(f"{path}: arena layout does not match this library build")
    arena = WeightArena.from_host(layout, segments, total, host, device, pinned=pinned, keep=hb)
    arena.upload()
    t4 = time.perf_counter()
    if "mem_estimate_mib" in header:        # the packed DAG's estimate: no profile_graph pass
        dag = fuse.FusedDag(header["dag_id"], fuse.build_preamble(len(members), True, None),
                            tuple(fuse._subgraph(g, w) for g, w in members), header["mem_estimate_mib"], 1)
    else:
        dag = fuse.fuse_models(members, dag_id=header["dag_id"], validate=False)
    img = DeviceDag([(sg, sg.weight_binding) for sg in dag.subgraphs], device, mode, arena=arena,
                    programs=programs, precision=header["precision"])
    fuse.attach_image(dag, img)
    t5 = time.perf_counter()
    arena.header_ms, arena.alloc_ms, arena.read_ms = (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3
    arena.dag_ms, arena.load_ms = (t5 - t4) * 1e3, (t5 - t0) * 1e3
    return dag
