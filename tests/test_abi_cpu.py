"""Host-side checks of the C-ABI library that need no GPU: it loads, exports every symbol
include/axq.h declares, and rejects invalid arguments before touching the device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "axq.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(axq_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2203_04071_b200 import _lib
    from paper_2203_04071_b200.build import build
    build()
    return _lib.load()


def test_header_declares_expected_entry_points():
    names = _declared()
    for n in ("axq_quantize", "axq_lut_gemm", "axq_lut_conv2d", "axq_dequantize"):
        assert n in names          # the four calls BASELINE.json north_star names


def test_library_exports_every_declared_symbol(L):
    from paper_2203_04071_b200 import _lib
    names = _declared()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert sorted(_lib.EXPORTED) == names


def test_binding_names_match_abi():
    import paper_2203_04071_b200 as pkg
    for n in ("axq_quantize", "axq_lut_gemm", "axq_lut_conv2d", "axq_dequantize", "axq_amax",
              "axq_scale", "axq_lut_gemm_dq", "axq_lut_conv2d_dq", "axq_lut_create"):
        assert callable(getattr(pkg, n))


def test_invalid_arguments_rejected_on_host(L):
    from paper_2203_04071_b200._lib import (AXQ_ERR_INVALID, AXQ_ERR_UNSUPPORTED, AXQ_OK,
                                            axq_conv_desc)
    assert L.axq_version() >= 100
    assert L.axq_status_string(0) == b"ok"
    h = ctypes.c_void_p()
    assert L.axq_lut_create(9, None, ctypes.byref(h)) == AXQ_ERR_INVALID
    assert L.axq_lut_create(1, None, ctypes.byref(h)) == AXQ_ERR_INVALID
    assert L.axq_amax(None, -1, None, None) == AXQ_ERR_INVALID
    assert L.axq_scale(None, 8, None, None) == AXQ_ERR_INVALID
    assert L.axq_quantize(None, 10, None, 8, None, None) == AXQ_ERR_INVALID
    assert L.axq_lut_gemm(-1, 1, 1, None, 1, None, 1, None, None, 1, None) == AXQ_ERR_INVALID
    assert L.axq_lut_gemm(1, 1, 1, None, 1, None, 1, None, None, 1, None) == AXQ_ERR_INVALID
    assert L.axq_dequantize(4, 4, None, 4, None, None, None, None, 4, None) == AXQ_ERR_INVALID
    d = axq_conv_desc(1, 8, 8, 4, 4, 3, 3, 1, 1, 1, 1, 1, 1, 2)
    # groups > 1 is supported (NEXT-3): with no table handle the call is invalid, and a group
    # count that does not divide the channels is invalid too
    assert L.axq_lut_conv2d(ctypes.byref(d), None, None, None, None, None) == AXQ_ERR_INVALID
    d3 = axq_conv_desc(1, 8, 8, 4, 4, 3, 3, 1, 1, 1, 1, 1, 1, 3)
    assert L.axq_lut_conv2d(ctypes.byref(d3), None, None, None, None, None) == AXQ_ERR_INVALID
    ho, wo = ctypes.c_int64(), ctypes.c_int64()
    assert L.axq_conv2d_out_hw(ctypes.byref(d), ctypes.byref(ho), ctypes.byref(wo)) == AXQ_OK
    assert (ho.value, wo.value) == (8, 8)
    d7 = axq_conv_desc(1, 224, 224, 3, 64, 7, 7, 2, 2, 3, 3, 1, 1, 1)
    assert L.axq_conv2d_out_hw(ctypes.byref(d7), ctypes.byref(ho), ctypes.byref(wo)) == AXQ_OK
    assert (ho.value, wo.value) == (112, 112)


def test_ste_workspace_queries(L):
    """axq_ste_*_workspace_elems: host-only sizing (no GPU needed).  The pre-converted operands
    of a product are 3 bf16 terms of the fp32 operand (128 x 32 tiles) and the bf16 codes."""
    from paper_2203_04071_b200._lib import axq_conv_desc
    L.axq_ste_linear_workspace_elems.restype = ctypes.c_int64
    L.axq_ste_linear_workspace_elems.argtypes = [ctypes.c_int64] * 3
    L.axq_ste_conv2d_workspace_elems.restype = ctypes.c_int64
    L.axq_ste_conv2d_workspace_elems.argtypes = [ctypes.c_void_p]
    assert L.axq_ste_linear_workspace_elems(-1, 4, 4) == -1
    assert L.axq_ste_conv2d_workspace_elems(None) == -1
    assert L.axq_ste_linear_workspace_elems(0, 0, 0) == 0
    M, N, K = 256, 1024, 1024
    cdiv = lambda a, b: -(-a // b)
    gx = cdiv(M, 128) * cdiv(N, 32) * 3 * 128 * 32 // 2 + cdiv(K, 128) * cdiv(N, 32) * 128 * 32 // 2
    gw = cdiv(N, 128) * cdiv(M, 32) * 3 * 128 * 32 // 2 + cdiv(K, 128) * cdiv(M, 32) * 128 * 32 // 2
    need = L.axq_ste_linear_workspace_elems(M, N, K)
    assert need >= max(gx, gw)
    assert L.axq_ste_linear_workspace_elems(2 * M, N, K) >= need
    d = axq_conv_desc(32, 56, 56, 64, 64, 3, 3, 1, 1, 1, 1, 1, 1, 1)
    Mc, Kc = 32 * 56 * 56, 9 * 64
    assert L.axq_ste_conv2d_workspace_elems(ctypes.byref(d)) >= cdiv(Mc, 128) * cdiv(64, 32) * 3 * 128 * 32 // 2


def test_product_package_does_not_import_oracle():
    """The product path must not route through the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2203_04071_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dp, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "axq_oracle" not in src and "liboracle" not in src, f
