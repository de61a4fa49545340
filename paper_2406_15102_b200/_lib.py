"""ctypes binding of libhlq_b200.so (include/hlq_b200.h).

The shared library is the only compute path: there is no CPU or PyTorch
fallback.  Loading fails loudly when the library is missing, and every call
into it raises the reference's exception classes on a non-zero status.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import DimensionError, FormatError, ParameterError, StateError

_HERE = os.path.dirname(os.path.abspath(__file__))
# HLQ_LIB_PATH: load an alternative in-tree build (A/B kernel experiments)
LIB_PATH = os.environ.get("HLQ_LIB_PATH") or os.path.join(_HERE, "libhlq_b200.so")

(HLQ_OK, HLQ_ERR_DIMENSION, HLQ_ERR_PARAMETER, HLQ_ERR_STATE, HLQ_ERR_NONFINITE, HLQ_ERR_CUDA,
 HLQ_ERR_FORMAT) = range(7)
HLQ_F32, HLQ_BF16 = 0, 1
HLQ_EPI_EXACT, HLQ_EPI_FAST = 0, 1

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_U32 = ctypes.c_uint32
_D = ctypes.c_double
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/hlq_b200.h exactly
SIGNATURES = {
    "hlq_version": (ctypes.c_char_p, []),
    "hlq_last_error": (ctypes.c_char_p, []),
    "hlq_device_ok": (_I, []),
    "hlq_quantize_ht_cols": (_I, [_P, _I, _I64, _I64, _I64, _I, _P, _P, _I64, _P, _P]),
    "hlq_quantize_proj_rows": (_I, [_P, _I, _I64, _I64, _I64, _I64, _I64, _U32, _I, _P, _P, _I64,
                                    _P, _P]),
    "hlq_quantize_dual": (_I, [_P, _I, _I64, _I64, _I64, _I64, _I64, _U32, _I, _I, _P, _P, _I64, _P,
                               _I64, _P, _P, _P]),
    "hlq_transform_pass": (_I, [_P, _I, _I64, _I64, _I64, _I64, _I64, _I, _I, _U32, _I, _I, _I, _P,
                                _P, _I64, _P, _I64, _P, _P, _P]),
    "hlq_proj_rows_amax": (_I, [_P, _I, _I64, _I64, _I64, _I64, _I64, _U32, _P, _P]),
    "hlq_proj_rows_quant": (_I, [_P, _I, _I64, _I64, _I64, _I64, _I64, _U32, _I, _P, _P, _I64, _P,
                                 _P]),
    "hlq_gemm_i8": (_I, [_P, _I64, _P, _I64, _I64, _I64, _I64, _I, _I, _P, _P, _D, _I, _P, _I, _I64,
                         _P, _I64, _P]),
    "hlq_gemm_i8_grouped": (_I, [_P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I, _I, _P,
                                 _P, _D, _I, _P, _I, _I64, _P, _I64, _P]),
    "hlq_gemm_i8_ws": (_SZ, [_I64, _I64, _I64, _I64]),
    "hlq_gemm_i8_ws_bits": (_SZ, [_I64, _I64, _I64, _I64, _I, _I]),
    "hlq_conv_acbp_pass": (_I, [_P, _I, _I64, _I64, _I64, _I64, _I, _I, _I, _U32, _I, _I, _P, _P, _I64, _P, _P]),
    "hlq_set_reserved_sms": (_I, [_I]),
    "hlq_nonfinite_fetch": (_I, [_P, _I, _P]),
    "hlq_acbp_container_bytes": (_I64, [_I64, _I64, _I]),
    "hlq_acbp_ws": (_SZ, [_I64]),
    "hlq_acbp_pack": (_I, [_P, _I64, _I64, _I64, _I, _I, _U32, _I64, _I64, _I64, _P, _P, _I64, _P, _SZ, _P]),
    "hlq_acbp_parse": (_I, [_P, _I64, _P, _P]),
    "hlq_acbp_unpack": (_I, [_P, _I64, _P, _P, _I64, _P, _P, _SZ, _P]),
    "hlq_last_error_offset": (_I64, []),
    "hlq_gemm_i8_multi": (_I, [_I, _P, _P]),
    "hlq_gemm_i4a_ex": (_I, [_P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I, _P, _P, _D, _I, _P,
                             _I, _I64, _P, _SZ, _P]),
    "hlq_quantize_dual_ex": (_I, [_P, _I, _I64, _I64, _I64, _I64, _I64, _U32, _I, _I, _P, _P, _I64, _I, _P, _I64,
                                  _P, _P, _P, _P, _SZ, _P]),
    "hlq_gemm_i8_ex": (_I, [_P, _I64, _I64, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I, _I, _P, _P,
                            _D, _I, _P, _I, _I64, _P, _I64, _P, _SZ, _P]),
    "hlq_quantize_weights_ws": (_SZ, [_I]),
    "hlq_basis_energy": (_I, [_P, _I, _I64, _I64, _I64, _I64, _I64, _P, _P]),
    "hlq_quantize_dual_colsum_ws": (_SZ, [_I64, _I64, _I64, _U32]),
    "hlq_quantize_dual_colsum": (_I, [_P, _I, _I64, _I64, _I64, _I64, _I64, _U32, _I, _I, _P, _P, _I64, _P,
                                      _I64, _P, _P, _P, _P, _SZ, _P]),
    "hlq_xform_quantize": (_I, [_P, _I, _I, ctypes.c_uint64, ctypes.c_uint64, _P, _P, _P, _P]),
    "hlq_xform_project_f32": (_I, [_P, _P, _P]),
    "hlq_xform_unproject_f32": (_I, [_P, _P, _P]),
    "hlq_quantize_stochastic": (_I, [_P, _I, _I64, _I64, _I64, _I64, _I64, _I, _U32, _I, ctypes.c_uint64,
                                     ctypes.c_uint64, _I, _I64, _I64, _P, _P, _I64, _P, _P]),
    "hlq_quantize_weights": (_I, [_I, _P, _P, _P, _I, _P, _P, _P, _P, _SZ, _P]),
    "hlq_quantize_weights_ex": (_I, [_I, _P, _P, _P, _I, _P, _P, _P, _P, _P, _SZ, _P]),
    "hlq_conv_dgrad_i8_ex": (_I, [_P, _I64, _I64, _I64, _I64, _I64, _P, _I64, _I64, _I, _I, _I, _I64, _I64, _I,
                                  _P, _P, _I, _P, _I, _P, _P]),
    "hlq_conv_dgrad_i8": (_I, [_P, _I64, _I64, _I64, _I64, _I64, _P, _I64, _I64, _I, _I, _I, _I, _P, _P,
                               _I, _P, _I, _P, _P]),
    "hlq_conv_acbp_compress": (_I, [_P, _I, _I64, _I64, _I64, _I64, _I, _I, _I, _U32, _I, _P, _I64,
                                    _P, _P, _P]),
    "hlq_col2im": (_I, [_P, _I, _I64, _I64, _I64, _I64, _I64, _I, _I, _I, _P, _I, _P]),
    "hlq_col2im_ex": (_I, [_P, _I, _I64, _I64, _I64, _I64, _I64, _I, _I, _I, _I, _P, _I, _P]),
    "hlq_acbp_k": (_I64, [_I64, _I64, _I, _I]),
    "hlq_acbp_rows": (_I64, [_I64, _I64, _I]),
    "hlq_acbp_compress": (_I, [_P, _I, _I64, _I64, _I64, _I, _U32, _I, _P, _I64, _P, _P, _P]),
    "hlq_hq_grad_input_ws": (_SZ, [_I64, _I64, _I64]),
    "hlq_grad_weight_ws_ex": (_SZ, [_I64, _I64, _I64, _I64, _I, _I, _I]),
    "hlq_grad_weight_ws": (_SZ, [_I64, _I64, _I64, _I, _I]),
    "hlq_hq_grad_input": (_I, [_P, _I, _I64, _I64, _P, _I64, _I, _P, _I, _I, _P, _SZ, _P]),
    "hlq_grad_weight": (_I, [_P, _I64, _P, _P, _I, _I64, _I64, _I64, _I64, _I, _U32, _I, _D, _P, _I,
                             _I, _P, _SZ, _P]),
}

class AcbpInfo(ctypes.Structure):
    """hlq_acbp_info (include/hlq_b200.h)."""
    _fields_ = [("B", _I64), ("L", _I64), ("I", _I64), ("bits", _I), ("block", _I), ("rank", _I),
                ("bitmap", _U32), ("axis", _I), ("rows", _I64), ("K", _I64), ("payload_bytes", _I64),
                ("total_bytes", _I64)]


class Xform(ctypes.Structure):
    """hlq_xform (include/hlq_b200.h)."""
    _fields_ = [("src", _P), ("src_dtype", ctypes.c_int32), ("segs", _I64), ("rows", _I64), ("cols", _I64),
                ("src_stride", _I64 * 3), ("bitmap", _U32), ("dst_stride", _I64 * 3), ("idx_stride", _I64 * 3)]


class GemmDesc(ctypes.Structure):
    """hlq_gemm_desc (include/hlq_b200.h)."""
    _fields_ = [("A", _P), ("lda", _I64), ("a_gstride", _I64), ("B", _P), ("ldb", _I64), ("b_gstride", _I64),
                ("M", _I64), ("N", _I64), ("K", _I64), ("groups", _I64), ("bits_a", _I), ("bits_b", _I),
                ("sa", _P), ("sb", _P), ("extra", _D), ("epilogue", _I), ("out", _P), ("out_dtype", _I),
                ("ldo", _I64), ("acc_out", _P), ("ld_acc", _I64), ("a_packed", _I)]


_lock = threading.Lock()
_lib = None


class HLQLibraryError(RuntimeError):
    """The CUDA library is missing or unusable (there is deliberately no fallback)."""


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise HLQLibraryError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2406_15102_b200.build` "
                "(the HLQ path has no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def exported_symbols() -> list:
    return list(SIGNATURES)


def version() -> str:
    return load().hlq_version().decode()


def check(status: int) -> None:
    if status == HLQ_OK:
        return
    msg = load().hlq_last_error().decode()
    if status == HLQ_ERR_DIMENSION:
        raise DimensionError(msg)
    if status == HLQ_ERR_PARAMETER:
        raise ParameterError(msg)
    if status == HLQ_ERR_STATE:
        raise StateError(msg)
    if status == HLQ_ERR_NONFINITE:
        raise ValueError(msg)
    if status == HLQ_ERR_FORMAT:
        raise FormatError(msg, int(load().hlq_last_error_offset()))
    raise HLQLibraryError(f"CUDA error in libhlq_b200: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
