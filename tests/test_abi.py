"""The C ABI library loads, exports every symbol include/tnsample.h declares, and rejects
bad arguments with the documented codes (no GPU compute calls)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2507_11424_b200 import build
    build.build()
    from paper_2507_11424_b200 import _lib
    return _lib.load_library()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tnsample.h")).read()
    return sorted(set(re.findall(r"\b(tn_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = declared_symbols()
    assert "tn_sample" in names and "tn_amplitude" in names and "tn_load_state" in names
    for name in names:
        assert hasattr(lib, name), name


def test_graph_errors_before_device(lib):
    from paper_2507_11424_b200 import _lib
    t = np.zeros(2, dtype=np.complex128)
    tensors = (C.c_void_p * 2)(t.ctypes.data, t.ctypes.data)
    h = C.c_void_p()

    def load(edges, bd, chi=2, n=2):
        e = np.asarray(edges, dtype=np.int32).reshape(-1, 2)
        b = np.asarray(bd, dtype=np.int32)
        g = _lib._Graph(n, len(b), e.ctypes.data_as(C.POINTER(C.c_int32)), b.ctypes.data_as(C.POINTER(C.c_int32)))
        return lib.tn_load_state(C.byref(g), tensors, chi, C.byref(h))

    assert load([[0, 0]], [1]) == -2          # self-loop
    assert load([[0, 5]], [1]) == -2          # out of range
    assert load([[0, 1], [1, 0]], [1, 1]) == -2  # duplicate
    assert load([[0, 1]], [3]) == -2          # bond > chi
    assert load([[0, 1]], [1], chi=0) == -1   # chi < 1
    assert lib.tn_load_state(None, tensors, 2, C.byref(h)) == -1
    assert b"duplicate" in lib.tn_last_error() or lib.tn_last_error()


def test_no_device_fails_loudly(lib):
    """Without a CUDA device a valid state is refused with TN_E_CUDA (no CPU fallback)."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    from paper_2507_11424_b200 import _lib
    t = np.zeros(2, dtype=np.complex128)
    t[0] = 1
    tensors = (C.c_void_p * 1)(t.ctypes.data)
    e = np.zeros((0, 2), dtype=np.int32)
    b = np.zeros(0, dtype=np.int32)
    g = _lib._Graph(1, 0, e.ctypes.data_as(C.POINTER(C.c_int32)), b.ctypes.data_as(C.POINTER(C.c_int32)))
    h = C.c_void_p()
    assert lib.tn_load_state(C.byref(g), tensors, 1, C.byref(h)) == -5
