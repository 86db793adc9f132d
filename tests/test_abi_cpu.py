"""CPU: the C-ABI library loads and exports every function include/fpx.h
declares (no compute calls without a GPU), and the product refuses to run
without CUDA (no CPU fallback)."""
import ctypes
import os
import re

import pytest

from paper_2501_12349_b200 import _C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "fpx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fpx_[a-z0-9_]+)\s*\(", src)))


@pytest.mark.skipif(not os.path.exists(_C.LIB_PATH), reason="library not built")
def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_C.LIB_PATH)
    names = header_functions()
    assert len(names) >= 18
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(_C.exported_symbols()) == names
    L = _C.lib()
    assert L.fpx_abi_version() == _C.ABI_VERSION
    assert L.fpx_supported(3, 3, 5) == 1 and L.fpx_supported(3, 3, 40) == 0


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2501_12349_b200 import engine, toolkit
    with pytest.raises(_C.FpxNativeError):
        engine.setup(toolkit.kershaw_mesh(2, 2))


def test_mesh_struct_layout():
    # fpx_mesh_t: 4 int32, int64, 8 pointers, 2 int32, 2 pointers, int32 + pad,
    # 6 doubles, 2 doubles, (ABI 2) frec + nodes_pad pointers, (ABI 7) fbox
    assert ctypes.sizeof(_C.MeshT) == 16 + 8 + 8 * 8 + 8 + 16 + 8 + 48 + 16 + 16 + 8
