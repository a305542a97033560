"""The C-ABI library loads on CPU and exports every symbol include/hs_api.h declares
(no compute calls without a GPU)."""
import os

import pytest

from paper_2503_12886_b200 import _lib as L
from paper_2503_12886_b200 import build as B


def test_library_built_in_tree():
    B.build()
    assert os.path.exists(L.LIB_PATH)
    assert L.LIB_PATH.startswith(os.path.dirname(os.path.dirname(os.path.abspath(B.__file__))))


def test_exports_every_header_symbol():
    lib = L.load()
    syms = L.header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
        assert s in L.SIGNATURES, f"{s} has no ctypes signature"


def test_pure_queries():
    lib = L.load()
    assert lib.hs_version() == 1
    assert lib.hs_scan_blocks(1000) == 4
    assert lib.hs_mlp_size(13, 128, 20) == 128 * 13 + 128 + 128 * 128 + 128 + 20 * 128 + 20
    assert lib.hs_sort_workspace_size(1 << 20) > 0
    assert 1 <= lib.hs_blend_bwd_partials(100) <= lib.hs_blend_bwd_partials(50176) <= 592


def test_device_error_mapping():
    with pytest.raises(FloatingPointError, match="non-finite scale at Gaussian index 7"):
        L.raise_device_error((1 << 62) | (2 << 32) | 7)
    with pytest.raises(FloatingPointError, match="zero-norm quaternion at Gaussian index 3"):
        L.raise_device_error((1 << 32) | 3)
    with pytest.raises(ValueError, match="non-finite"):
        L.raise_device_error(0)
    L.raise_device_error(L.HS_NO_ERROR)


def test_status_mapping():
    with pytest.raises(ValueError):
        L.check(L.HS_ERR_SHAPE)
    with pytest.raises(RuntimeError):
        L.check(L.HS_ERR_COLOR_INIT)


def test_u8_unit_is_exact():
    """hs_common.cuh:u8_unit (x * r, then the FMA residual correction) is the correctly
    rounded float32 x / 255 for every byte value: checked with exact rationals."""
    from fractions import Fraction as Fr
    import numpy as np

    def r32(x):
        c = np.float32(float(x))
        cands = [np.nextafter(c, np.float32(-np.inf)), c, np.nextafter(c, np.float32(np.inf))]
        return min(cands, key=lambda v: (abs(Fr(float(v)) - x), int(np.float32(v).view(np.uint32)) & 1))

    r = np.float32(1.0) / np.float32(255.0)
    for x in range(256):
        q = r32(Fr(x) * Fr(float(r)))
        res = r32(-Fr(float(q)) * 255 + x)
        got = r32(Fr(float(res)) * Fr(float(r)) + Fr(float(q)))
        assert got == np.float32(x) / np.float32(255.0), x
