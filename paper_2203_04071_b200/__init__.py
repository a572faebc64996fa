"""B200-native approximate-multiplier LUT inference (AdaPT, arXiv 2203.04071).

The product path is libaxq.so (hand-written sm_100a CUDA behind the C ABI in
include/axq.h) reached through the thin ctypes binding in ``_lib``.  There is no CPU
fallback: importing the package raises if the library has not been built.
"""
from . import _lib
from ._lib import (  # noqa: F401
    EXPORTED, AxqError, Lut, axq_amax, axq_conv2d_out_hw, axq_dequantize,
    axq_dequantize_nhwc_to_nchw, axq_lut_conv2d, axq_lut_conv2d_dq, axq_lut_create,
    axq_lut_destroy, axq_lut_gemm, axq_lut_gemm_dq, axq_quantize, axq_quantize_nchw_to_nhwc,
    axq_scale, conv_desc,
)

_lib.load()
