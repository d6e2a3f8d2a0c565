"""ctypes binding of the C ABI (include/q8g_b200.h).

The CUDA library is the only compute path: if libq8g_b200.so is missing or
fails to load, every entry point raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("Q8G_LIB", _PKG / "libq8g_b200.so"))

Q8G_OK, Q8G_EINVAL, Q8G_ENOMEM, Q8G_ECUDA, Q8G_ENOTSUP = 0, 1, 2, 3, 4
ROUND_REF, ROUND_F32_RNE = 0, 1


class Q8GError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(Q8GError, ValueError):
    """Maps the reference's std::invalid_argument (engine.hpp:66-84)."""


class Blocking(C.Structure):
    _fields_ = [("mcb", C.c_int), ("ncb", C.c_int), ("kcb", C.c_int), ("mr", C.c_int), ("nr", C.c_int)]


class RequantParamsC(C.Structure):
    _fields_ = [
        ("multiplier", C.c_double),
        ("zp_a", C.c_int32),
        ("zp_b", C.c_int32),
        ("zp_c", C.c_int32),
        ("k_total", C.c_int32),
        ("bias_host", C.POINTER(C.c_int32)),
        ("zp_b_per_channel_host", C.POINTER(C.c_int32)),
        ("multiplier_f32_per_channel_host", C.POINTER(C.c_float)),
        ("multiplier_per_channel_host", C.POINTER(C.c_double)),
        ("col_offsets_host", C.POINTER(C.c_int32)),
        ("rounding", C.c_int),
        ("relu", C.c_int),
    ]


class PipelineArgsC(C.Structure):  # q8g_pipeline_args
    _fields_ = [
        ("sparse", C.c_void_p),
        ("bias_add_dev", C.c_void_p),
        ("writer", C.c_int),
        ("ep", C.c_void_p),
        ("dq_scale", C.c_double),
        ("dq_zero_point", C.c_int32),
    ]


Q8G_WRITE_RAW_I32, Q8G_WRITE_REQUANT_U8, Q8G_WRITE_DEQUANT_F32 = 0, 1, 2


# (name, restype, argtypes)
_P = C.c_void_p
_I = C.c_int
_SIGS = [
    ("q8g_last_error", C.c_char_p, []),
    ("q8g_version", _I, []),
    ("q8g_launch_count", C.c_uint64, []),
    ("q8g_launch_stats", _I, [C.POINTER(C.c_uint64), _I]),
    ("q8g_debug_tc_trace", _I, [C.POINTER(C.c_uint64), _I]),
    ("q8g_debug_kernel_clock", _I, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("q8g_blocking_defaults", _I, [C.POINTER(Blocking)]),
    ("q8g_blocking_validate", _I, [C.POINTER(Blocking)]),
    ("q8g_select_blocking", _I, [_I, _I, _I, C.POINTER(Blocking), C.POINTER(Blocking)]),
    ("q8g_partition_stripes", _I, [_I, _I, _I, C.POINTER(_I), C.POINTER(_I)]),
    ("q8g_pack_b", _I, [_P, _I, _I, _I, C.POINTER(Blocking), _I, C.POINTER(_P)]),
    ("q8g_pack_b_device", _I, [_P, _I, _I, _I, C.POINTER(Blocking), _I, _P, C.POINTER(_P)]),
    ("q8g_packed_b_replicate", _I, [_P, _I, C.POINTER(_P)]),
    ("q8g_packed_b_info", _I, [_P, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
    ("q8g_packed_b_blocking", _I, [_P, C.POINTER(Blocking)]),
    ("q8g_packed_b_col_offsets", _I, [_P, _P]),
    ("q8g_unpack_b", _I, [_P, _P, _I]),
    ("q8g_free_packed_b", _I, [_P]),
    ("q8g_epilogue_create", _I, [_P, C.POINTER(RequantParamsC), _P, C.POINTER(_P)]),
    ("q8g_epilogue_free", _I, [_P]),
    ("q8g_kernel_cache_create", _I, [_I, C.POINTER(_P)]),
    ("q8g_kernel_cache_free", _I, [_P]),
    ("q8g_kernel_cache_build_count", C.c_uint64, [_P]),
    ("q8g_kernel_cache_tile", _I, [_P, _I, _I, _I, _I, C.POINTER(_I)]),
    ("q8g_gemm_u8s8_requant", _I, [_P, _I, _I, _I, _P, _P, _P, _I, _I, _I, _P, _P]),
    ("q8g_gemm_u8s8_requant_peers", _I, [_P, _I, _I, _I, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P]),
    ("q8g_gemm_u8s8_raw_i32", _I, [_P, _I, _I, _I, _P, _P, _P, _I, _I, _I, _P, _P]),
    ("q8g_gemm_u8s8_requant_host", _I, [_P, _I, _I, _I, _P, _P, _P, _I, _I, _I, _P]),
    ("q8g_gemm_u8s8_raw_i32_host", _I, [_P, _I, _I, _I, _P, _P, _I, _I, _I, _P]),
    ("q8g_conv3x3_u8s8_nhwc", _I, [_P, _I, _I, _I, _I, _P, _P, _P, _I, _I, _P]),
    ("q8g_conv3x3_u8s8_nhwc_raw_i32", _I, [_P, _I, _I, _I, _I, C.c_int32, _P, _P, _I, _I, _P]),
    ("q8g_conv3x3_prepare", _I, [_P, _I, _P]),
    ("q8g_conv3x3_u8s8_nhwc_host", _I, [_P, _I, _I, _I, _I, _P, _P, _P, _I, _I, _P]),
    ("q8g_dw_filter_create", _I, [_P, _I, C.POINTER(RequantParamsC), _I, C.POINTER(_P)]),
    ("q8g_dw_filter_free", _I, [_P]),
    ("q8g_dwconv3x3_u8s8_nhwc", _I, [_P, _I, _I, _I, _I, _P, _P, _I, _I, _P]),
    ("q8g_dwconv3x3_u8s8_nhwc_host", _I, [_P, _I, _I, _I, _I, _P, _P, _I, _I, _P]),
    ("q8g_split_outliers", _I, [_P, _I, _I, _I, _I, _P, _I, _P, _P, _P, _I, C.POINTER(_I)]),
    ("q8g_sparse_csc_create", _I, [_P, _P, _P, _I, _I, _I, _I, C.POINTER(_P)]),
    ("q8g_sparse_csc_free", _I, [_P]),
    ("q8g_gemm_u8s8_pipeline", _I, [_P, _I, _I, _I, _P, C.POINTER(PipelineArgsC), _P, _I, _I, _I, _P, _P]),
    ("q8g_gemm_u8s8_pipeline_host", _I, [_P, _I, _I, _I, _P, C.POINTER(PipelineArgsC), _P, _P, _I, _I, _I, _P]),
]

EXPORTED = [s[0] for s in _SIGS]

_lib = None


def load() -> C.CDLL:
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, res, args in _SIGS:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    return load().q8g_last_error().decode(errors="replace")


def check(rc: int) -> None:
    if rc == Q8G_OK:
        return
    msg = last_error()
    if rc == Q8G_EINVAL:
        raise InvalidArgument(rc, msg)
    raise Q8GError(rc, msg)


def launch_count() -> int:
    return int(load().q8g_launch_count())


FAMILIES = ("pack", "gemm_simt", "gemm_tc_small_m", "gemm_tc_large_m", "conv_simt", "conv_tc", "dw_simt",
            "dw_tc", "post", "conv_im2col", "dw_fma", "peer_copy")


def launch_stats() -> dict:
    """Launch counts per kernel family (evidence of which kernel ran)."""
    arr = (C.c_uint64 * len(FAMILIES))()
    check(load().q8g_launch_stats(arr, len(FAMILIES)))
    return {f: int(v) for f, v in zip(FAMILIES, arr)}
