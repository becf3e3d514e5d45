"""ctypes binding of libdfx (include/dfx.h).

The product path has no CPU fallback: if ``libdfx.so`` is missing or no
sm_100 device is visible, ``lib()`` / ``init_device()`` raise ``DeviceError``.
Structures mirror dfx.h field for field; ``check_abi()`` compares every
``sizeof`` with the library's own ``dfx_sizeof`` so a layout drift fails at
load time instead of corrupting kernel parameters.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import DeviceError

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libdfx.so"

(OP_GEMM, OP_SPLITK, OP_DWCONV, OP_POOL, OP_GAP, OP_EW, OP_IN, OP_OUT, OP_SE, OP_LN, OP_TOKENS,
 OP_ATTN, OP_DWSE, OP_GATE) = range(1, 15)
ACT = {None: 0, "relu": 1, "hardswish": 2, "hardsigmoid": 3, "silu": 4, "sigmoid": 5, "gelu": 6}
BIN_NONE, BIN_ADD, BIN_SCALE = 0, 1, 2
DT_BF16, DT_F16, DT_BF16X2, DT_F16X2 = 0, 1, 2, 3
DTYPES = {"bf16": DT_BF16, "fp16": DT_F16, "bf16x2": DT_BF16X2, "fp16x2": DT_F16X2}
ABI_VERSION = 5

i32, i64, u64, vp, u8 = C.c_int32, C.c_int64, C.c_uint64, C.c_void_p, C.c_uint8
fptr = C.POINTER(C.c_float)


class View(C.Structure):
    _fields_ = [("base", vp), ("n", i32), ("h", i32), ("w", i32), ("c", i32),
                ("pitch", i32), ("coff", i32), ("dtype", i32), ("_pad", i32)]


class Epilogue(C.Structure):
    _fields_ = [("alpha", vp), ("beta", vp), ("act1", i32), ("act2", i32), ("binop", i32),
                ("_pad", i32), ("other", View)]


class GemmDesc(C.Structure):
    _pack_ = 8
    _fields_ = [("tmap_a", u64 * 16), ("tmap_b", u64 * 16),
                ("n", i32), ("p", i32), ("q", i32), ("tn", i32), ("tp", i32), ("tq", i32),
                ("mt_n", i32), ("mt_p", i32), ("mt_q", i32), ("nt", i32),
                ("r", i32), ("s", i32), ("stride_h", i32), ("stride_w", i32),
                ("pad_h", i32), ("pad_w", i32), ("cb", i32), ("cblocks", i32), ("ksteps", i32),
                ("kpack", i32), ("stages", i32), ("splits", i32), ("stages_per_split", i32),
                ("bn", i32), ("cout", i32), ("tile_begin", i32), ("tiles", i32), ("m2", i32),
                ("out", View), ("epi", Epilogue), ("ws", vp), ("counters", vp),
                ("pre_scale", vp), ("pre_shift", vp), ("pre_mode", i32), ("pre_act", i32),
                ("pre_cin", i32), ("pre_pitch", i32), ("dw_w", vp), ("dw_alpha", vp),
                ("dw_beta", vp), ("dw_k", i32), ("dw_s", i32), ("dw_pad", i32), ("dw_act", i32),
                ("se", vp)]


class SeFuse(C.Structure):
    _fields_ = [("w1", vp), ("b1", vp), ("w2", vp), ("b2", vp), ("scratch", vp), ("sync", vp),
                ("pooled", vp), ("c", i32), ("cr", i32), ("act1", i32), ("act2", i32), ("ctas", i32),
                ("mode", i32), ("_pad", i32 * 2)]


class GemmLaunch(C.Structure):
    _fields_ = [("descs", vp), ("ndesc", i32), ("total_tiles", i32), ("bn_max", i32),
                ("dtype", i32), ("nslots", i32), ("flags", i32), ("m2", i32), ("se_cr", i32), ("max_ctas", i32), ("l2_pf_units", C.c_uint32), ("l2_pf", vp * 2),
                ("desc0", GemmDesc)]


class SplitKParams(C.Structure):
    _fields_ = [("ws", vp), ("splits", i32), ("pixels", i32), ("cout", i32), ("ldw", i32),
                ("out", View), ("epi", Epilogue)]


class DwconvParams(C.Structure):
    _fields_ = [("inp", View), ("out", View), ("weight", vp), ("kh", i32), ("kw", i32),
                ("stride_h", i32), ("stride_w", i32), ("pad_h", i32), ("pad_w", i32),
                ("epi", Epilogue)]


class PoolParams(C.Structure):
    _fields_ = [("inp", View), ("out", View), ("kh", i32), ("kw", i32), ("stride_h", i32),
                ("stride_w", i32), ("pad_h", i32), ("pad_w", i32), ("is_max", i32),
                ("count_include_pad", i32)]


class GapParams(C.Structure):
    _fields_ = [("inp", View), ("out", View)]


class EwParams(C.Structure):
    _fields_ = [("inp", View), ("out", View), ("epi", Epilogue)]


class InParams(C.Structure):
    _fields_ = [("src", vp), ("out", View), ("kh", i32), ("kw", i32), ("sh", i32), ("sw", i32),
                ("ph", i32), ("pw", i32), ("c", i32), ("h", i32), ("w", i32), ("split", i32)]


class OutParams(C.Structure):
    _fields_ = [("inp", View), ("dst", vp)]


class GateParams(C.Structure):
    _fields_ = [("flag", vp), ("_pad", i32 * 2)]


class SeParams(C.Structure):
    _fields_ = [("inp", View), ("out", View), ("w1", vp), ("b1", vp), ("w2", vp), ("b2", vp),
                ("cr", i32), ("act1", i32), ("act2", i32), ("apply", i32), ("pooled", vp)]


class DwseParams(C.Structure):
    _fields_ = [("inp", View), ("out", View), ("dw_weight", vp), ("kh", i32), ("kw", i32),
                ("stride_h", i32), ("stride_w", i32), ("pad_h", i32), ("pad_w", i32),
                ("dw_epi", Epilogue), ("w1", vp), ("b1", vp), ("w2", vp), ("b2", vp),
                ("cr", i32), ("act1", i32), ("act2", i32), ("staged", i32)]


class LnParams(C.Structure):
    _fields_ = [("inp", View), ("out", View), ("gamma", vp), ("beta", vp), ("eps", C.c_float),
                ("norm", i32), ("_pad", i32 * 2)]


class TokensParams(C.Structure):
    _fields_ = [("inp", View), ("out", View), ("cls", vp), ("pos", vp)]


class AttnParams(C.Structure):
    _fields_ = [("qkv", View), ("out", View), ("heads", i32), ("scale", C.c_float), ("_pad", i32 * 2)]


STRUCTS = {
    "dfx_view": View, "dfx_epilogue": Epilogue, "dfx_gemm_desc": GemmDesc,
    "dfx_gemm_launch": GemmLaunch, "dfx_splitk_params": SplitKParams,
    "dfx_dwconv_params": DwconvParams, "dfx_pool_params": PoolParams,
    "dfx_gap_params": GapParams, "dfx_ew_params": EwParams, "dfx_in_params": InParams,
    "dfx_out_params": OutParams, "dfx_se_params": SeParams, "dfx_ln_params": LnParams,
    "dfx_tokens_params": TokensParams, "dfx_attn_params": AttnParams, "dfx_dwse_params": DwseParams,
    "dfx_se_fuse": SeFuse, "dfx_gate_params": GateParams,
}
OP_PARAMS = {OP_GEMM: GemmLaunch, OP_SPLITK: SplitKParams, OP_DWCONV: DwconvParams,
             OP_POOL: PoolParams, OP_GAP: GapParams, OP_EW: EwParams, OP_IN: InParams,
             OP_OUT: OutParams, OP_SE: SeParams, OP_LN: LnParams, OP_TOKENS: TokensParams,
             OP_ATTN: AttnParams, OP_DWSE: DwseParams, OP_GATE: GateParams}

# every symbol include/dfx.h declares (tests check the .so exports all of them)
EXPORTS = (
    "dfx_last_error", "dfx_abi_version", "dfx_sizeof", "dfx_init", "dfx_device_info", "dfx_mem_info", "dfx_nonfinite_count",
    "dfx_malloc", "dfx_free", "dfx_memset", "dfx_pool_malloc", "dfx_pool_free", "dfx_pool_trim", "dfx_pool_stats", "dfx_host_alloc", "dfx_host_free",
    "dfx_host_register", "dfx_host_unregister", "dfx_memcpy_h2d", "dfx_memcpy_d2h",
    "dfx_memcpy_d2d", "dfx_arena_upload", "dfx_stream_create", "dfx_stream_destroy",
    "dfx_stream_sync", "dfx_event_create", "dfx_event_destroy", "dfx_event_record",
    "dfx_event_elapsed", "dfx_tmap_act", "dfx_tmap_weights", "dfx_launch", "dfx_graph_create",
    "dfx_graph_add", "dfx_graph_set_priority", "dfx_graph_instantiate", "dfx_graph_launch", "dfx_graph_node_count",
    "dfx_graph_destroy", "dfx_execute", "dfx_execute_gather", "dfx_execute_gated", "dfx_nvtx_range_push",
    "dfx_nvtx_range_pop",
)

_lock = threading.Lock()
_lib = None
_inited: set[int] = set()


def lib():
    """Load libdfx.so (once).  Raises DeviceError if it is not built."""
    global _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("DFX_LIBRARY", str(LIB_PATH))
            if not Path(path).exists():
                raise DeviceError(-6, f"{path} is not built (run __graft_entry__.build())",
                                  "load libdfx")
            L = C.CDLL(path)
            L.dfx_last_error.restype = C.c_char_p
            L.dfx_sizeof.argtypes = [C.c_char_p]
            L.dfx_sizeof.restype = C.c_int
            _lib = L
            check_abi(L)
        return _lib


def check_abi(L) -> None:
    if L.dfx_abi_version() != ABI_VERSION:
        raise DeviceError(-2, "ABI version mismatch", "dfx_abi_version")
    for name, cls in STRUCTS.items():
        got = L.dfx_sizeof(name.encode())
        if got != C.sizeof(cls):
            raise DeviceError(-2, f"sizeof({name}) = {got} in C, {C.sizeof(cls)} in ctypes",
                              "check_abi")


def call(name: str, *args) -> None:
    L = lib()
    rc = getattr(L, name)(*args)
    if rc != 0:
        raise DeviceError(rc, L.dfx_last_error().decode(errors="replace"), name)


def init_device(device: int = 0) -> None:
    if device in _inited:
        call("dfx_init", C.c_int(device))   # cheap; re-selects the device on this thread
        return
    call("dfx_init", C.c_int(device))
    _inited.add(device)


# ---- small helpers ---------------------------------------------------------------

def malloc(nbytes: int) -> int:
    p = vp()
    call("dfx_malloc", C.byref(p), C.c_size_t(nbytes))
    return p.value


def free(ptr: int) -> None:
    if ptr:
        call("dfx_free", vp(ptr))


def pool_malloc(nbytes: int, stream=None) -> int:
    """Weight-arena allocation from the device's retained pool (dfx_pool_malloc)."""
    p = vp()
    call("dfx_pool_malloc", C.byref(p), C.c_size_t(nbytes), vp(stream))
    return p.value


def pool_free(ptr: int, stream=None) -> None:
    if ptr:
        call("dfx_pool_free", vp(ptr), vp(stream))


def pool_trim(keep_bytes: int = 0) -> None:
    call("dfx_pool_trim", C.c_size_t(keep_bytes))


def pool_stats() -> tuple[int, int]:
    """(bytes the arena pool keeps mapped, bytes of it in use)."""
    r, u = C.c_size_t(), C.c_size_t()
    call("dfx_pool_stats", C.byref(r), C.byref(u))
    return r.value, u.value


def host_alloc(nbytes: int) -> int:
    p = vp()
    call("dfx_host_alloc", C.byref(p), C.c_size_t(nbytes))
    return p.value


def host_free(ptr: int) -> None:
    if ptr:
        call("dfx_host_free", vp(ptr))


def memset(ptr: int, value: int, nbytes: int, stream=None) -> None:
    call("dfx_memset", vp(ptr), C.c_int(value), C.c_size_t(nbytes), vp(stream))


def h2d(dst: int, src: int, nbytes: int, stream=None) -> None:
    call("dfx_memcpy_h2d", vp(dst), vp(src), C.c_size_t(nbytes), vp(stream))


def d2h(dst: int, src: int, nbytes: int, stream=None) -> None:
    call("dfx_memcpy_d2h", vp(dst), vp(src), C.c_size_t(nbytes), vp(stream))


def d2d(dst: int, src: int, nbytes: int, stream=None) -> None:
    call("dfx_memcpy_d2d", vp(dst), vp(src), C.c_size_t(nbytes), vp(stream))


def stream_create() -> int:
    s = vp()
    call("dfx_stream_create", C.byref(s))
    return s.value


def stream_sync(stream) -> None:
    call("dfx_stream_sync", vp(stream))


def stream_destroy(stream) -> None:
    call("dfx_stream_destroy", vp(stream))


def nonfinite_count(device: int = 0, reset: bool = False) -> int:
    """Non-finite logits the output kernels wrote on ``device`` since the last reset
    (an fp16 overflow upstream becomes inf / NaN instead of a clamped value)."""
    n = C.c_ulonglong()
    call("dfx_nonfinite_count", C.c_int(device), C.byref(n), C.c_int(1 if reset else 0))
    return n.value


def mem_info() -> tuple[int, int]:
    f, t = C.c_size_t(), C.c_size_t()
    call("dfx_mem_info", C.byref(f), C.byref(t))
    return f.value, t.value


def launch(op: int, params, stream=None) -> None:
    call("dfx_launch", C.c_int(op), C.byref(params), C.c_size_t(C.sizeof(params)), vp(stream))


class Event:
    def __init__(self):
        e = vp()
        call("dfx_event_create", C.byref(e))
        self.ptr = e.value

    def record(self, stream=None):
        call("dfx_event_record", vp(self.ptr), vp(stream))

    def elapsed_ms(self, end: "Event") -> float:
        ms = C.c_float()
        call("dfx_event_elapsed", vp(self.ptr), vp(end.ptr), C.byref(ms))
        return ms.value

    def __del__(self):
        try:
            if self.ptr and _lib is not None:
                _lib.dfx_event_destroy(vp(self.ptr))
        except Exception:   # noqa: BLE001 - interpreter teardown
            pass


class Graph:
    """A CUDA graph of libdfx kernel nodes with explicit dependencies."""

    def __init__(self):
        g = vp()
        call("dfx_graph_create", C.byref(g))
        self.ptr = g.value
        self.kinds: list[int] = []

    def add(self, op: int, params, deps=()) -> int:
        deps = list(deps)
        arr = (C.c_int * max(len(deps), 1))(*deps)
        nid = C.c_int()
        call("dfx_graph_add", vp(self.ptr), C.c_int(op), C.byref(params),
             C.c_size_t(C.sizeof(params)), arr, C.c_int(len(deps)), C.byref(nid))
        self.kinds.append(op)
        return nid.value

    def set_priority(self, node_id: int, priority: int) -> tuple[int, int]:
        """Node scheduling priority (lower = more urgent); returns (least, greatest)."""
        rng = (C.c_int * 2)()
        call("dfx_graph_set_priority", vp(self.ptr), C.c_int(node_id), C.c_int(priority), rng)
        return rng[0], rng[1]

    def instantiate(self):
        call("dfx_graph_instantiate", vp(self.ptr))

    def launch(self, stream=None):
        call("dfx_graph_launch", vp(self.ptr), vp(stream))

    def execute(self, host_in, dev_in, in_bytes, host_out, dev_out, out_bytes, stream):
        call("dfx_execute", vp(self.ptr), vp(host_in), vp(dev_in), C.c_size_t(in_bytes),
             vp(host_out), vp(dev_out), C.c_size_t(out_bytes), vp(stream))

    def execute_gather(self, srcs, sizes, host_in, dev_in, host_out, dev_out, out_bytes, stream):
        """srcs / sizes: ctypes arrays of host pointers and byte counts."""
        call("dfx_execute_gather", vp(self.ptr), srcs, sizes, C.c_int(len(srcs)), vp(host_in),
             vp(dev_in), vp(host_out), vp(dev_out), C.c_size_t(out_bytes), vp(stream))

    def execute_gated(self, srcs, sizes, src_member, member_off, member_bytes, host_in, dev_in, flags, one,
                      host_out, dev_out, out_bytes, stream, copy_stream):
        """dfx_execute_gated: graph launched first, members' inputs staged behind it."""
        call("dfx_execute_gated", vp(self.ptr), srcs, sizes, src_member, C.c_int(len(srcs)), member_off,
             member_bytes, C.c_int(len(member_off)), vp(host_in), vp(dev_in), vp(flags), vp(one),
             vp(host_out), vp(dev_out), C.c_size_t(out_bytes), vp(stream), vp(copy_stream))

    def destroy(self):
        if self.ptr:
            call("dfx_graph_destroy", vp(self.ptr))
            self.ptr = 0


def tmap_act(view: View, cb: int, tq: int, tp: int, tn: int, sw: int, sh: int):
    buf = (u64 * 16)()
    call("dfx_tmap_act", buf, C.byref(view), C.c_int(cb), C.c_int(tq), C.c_int(tp), C.c_int(tn),
         C.c_int(sw), C.c_int(sh))
    return buf


def tmap_weights(base: int, rows: int, k: int, cb: int, bn: int, dtype: int):
    buf = (u64 * 16)()
    call("dfx_tmap_weights", buf, vp(base), C.c_int(rows), C.c_int(k), C.c_int(cb), C.c_int(bn),
         C.c_int(dtype))
    return buf


class nvtx_range:
    """``with rt.nvtx_range("fuse_models"):`` -- an NVTX range through libdfx (a no-op
    unless a profiler is attached); silently absent when the library is not loaded."""

    def __init__(self, msg: str):
        self.msg = msg.encode()

    def __enter__(self):
        if _lib is not None:
            _lib.dfx_nvtx_range_push(self.msg)
        return self

    def __exit__(self, *exc):
        if _lib is not None:
            _lib.dfx_nvtx_range_pop()
        return False
