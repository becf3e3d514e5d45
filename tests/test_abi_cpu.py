"""The C-ABI library loads without a GPU, exports every symbol include/dfx.h
declares, and every ctypes mirror has the C struct's size."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2410_21120_b200 import runtime

ROOT = Path(__file__).resolve().parents[1]


def _declared_functions():
    text = (ROOT / "include" / "dfx.h").read_text()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(dfx_\w+)\(", text, flags=re.M)))


def test_header_and_binding_agree():
    assert _declared_functions() == sorted(runtime.EXPORTS)


def test_library_exports_every_declared_symbol():
    if not runtime.LIB_PATH.exists():
        pytest.skip("libdfx.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(runtime.LIB_PATH))
    for name in _declared_functions():
        assert hasattr(lib, name), name


def test_struct_layouts_match():
    if not runtime.LIB_PATH.exists():
        pytest.skip("libdfx.so not built")
    L = runtime.lib()           # runs check_abi: every dfx_sizeof == ctypes.sizeof
    for name, cls in runtime.STRUCTS.items():
        assert L.dfx_sizeof(name.encode()) == ctypes.sizeof(cls)
    assert L.dfx_abi_version() == runtime.ABI_VERSION


def test_no_device_fails_loudly():
    """Without an sm_100 GPU the product path raises DeviceError (no CPU fallback)."""
    if not runtime.LIB_PATH.exists():
        pytest.skip("libdfx.so not built")
    import numpy as np
    from paper_2410_21120_b200 import errors, graph_ir
    from paper_2410_21120_b200.executor import Tensor, run
    try:
        runtime.init_device(0)
    except errors.DeviceError:
        g = graph_ir.ModelGraph("m", [graph_ir.OpNode("r", "relu")], "r", "r",
                                graph_ir.TensorSpec((3,)), graph_ir.TensorSpec((3,)))
        with pytest.raises(errors.DeviceError):
            run(g, graph_ir.WeightStore(), Tensor(g.input_spec, np.zeros(3)))
        return
    pytest.skip("a GPU is visible; covered by the gpu tests")
