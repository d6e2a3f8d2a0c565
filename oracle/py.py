"""ctypes access to the CPU checkers (TEST INFRASTRUCTURE ONLY).

  Oracle  - liboracle.so, the C restatement (oracle.c)
  RefLib  - _ref/libq8ref*.so, the unmodified reference headers behind
            ref_shim.cpp
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libq8ref.so"
REF_RELEASE_SO = HERE / "_ref" / "libq8ref_release.so"
REF_V4_SO = HERE / "_ref" / "libq8ref_v4.so"


def host_has_avx512() -> bool:
    try:
        flags = Path("/proc/cpuinfo").read_text().split("flags")[1].split("\n")[0].split()
    except (OSError, IndexError):
        return False
    return all(f in flags for f in ("avx512f", "avx512bw", "avx512vl", "avx512dq", "avx512cd"))


def best_ref_so() -> Path:
    """The fastest reference build this host can run: -march=x86-64-v4 on
    AVX-512 hosts (BASELINE.md §3 asks for -march=native), else x86-64-v3."""
    return REF_V4_SO if REF_V4_SO.exists() and host_has_avx512() else REF_SO
REF_INCLUDE = Path("/root/reference/proj/include")

_P, _I, _D, _F = C.c_void_p, C.c_int, C.c_double, C.c_float
I32P = C.POINTER(C.c_int32)


def build(quiet: bool = True) -> None:
    """Compile the oracle (and, when the reference headers are present, the
    reference shim) with oracle/Makefile."""
    targets = [str(ORACLE_SO)]
    if REF_INCLUDE.exists():
        targets.append("ref")
    r = subprocess.run(["make", "-C", str(HERE), *targets], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")
    if not quiet:
        print(r.stdout)


def _p(a: np.ndarray):
    return None if a is None else a.ctypes.data


class Oracle:
    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            build()
        L = self.L = C.CDLL(str(path))
        sig = {
            "orc_rng_new": (_P, [C.c_uint64]),
            "orc_rng_free": (None, [_P]),
            "orc_rng_next": (C.c_uint64, [_P]),
            "orc_rng_u8": (None, [_P, _P, C.c_int64]),
            "orc_rng_i8": (None, [_P, _P, C.c_int64]),
            "orc_rng_int": (C.c_int32, [_P, C.c_int32, C.c_int32]),
            "orc_rng_int_fill": (None, [_P, C.c_int32, C.c_int32, _P, C.c_int64]),
            "orc_rng_real": (_D, [_P, _D, _D]),
            "orc_rng_real_fill": (None, [_P, _D, _D, _P, C.c_int64]),
            "orc_naive_gemm_i32": (None, [_P, _I, _I, _I, _P, _I, _I, _P, _I, _I]),
            "orc_col_offsets": (None, [_P, _I, _I, _I, _P]),
            "orc_row_offsets": (None, [_P, _I, _I, _I, _P]),
            "orc_requant_adjust": (C.c_int64, [C.c_int32] * 7),
            "orc_round_half_away": (C.c_longlong, [_D]),
            "orc_requant_scalar_ref": (C.c_uint8, [C.c_int32, C.c_int32, C.c_int32, _D] + [C.c_int32] * 5),
            "orc_requant_scalar_f32": (C.c_uint8, [C.c_int32, C.c_int32, C.c_int32, _F] + [C.c_int32] * 5),
            "orc_relu_quantized": (C.c_uint8, [C.c_uint8, C.c_int32]),
            "orc_requant_matrix": (None, [_P, _I, _I, _I, _P, _P, C.c_int32, _P, _I, C.c_int32, _P, _I, _P, _P,
                                          C.c_int32, _I, _P, _I]),
            "orc_prepack_ref_size": (C.c_int64, [_I, _I, _I, _I]),
            "orc_prepack_ref": (None, [_P, _I, _I, _I, _I, _I, _I, _P]),
            "orc_im2col3x3": (None, [_P, _I, _I, _I, _I, C.c_uint8, _P, _I]),
            "orc_conv3x3_i32": (None, [_P, _I, _I, _I, _I, C.c_uint8, _P, _I, _P, _I]),
            "orc_dwconv3x3": (None, [_P, _I, _I, _I, _I, C.c_int32, _P, _P, _P, _P, C.c_int32, _I, _P, _P, _I]),
            "orc_split_outliers": (_I, [_P, _I, _I, _I, _I, _P, _I, _P, _P, _P, _I]),
            "orc_spmdm_add": (None, [_P, _I, _I, _I, _P, _P, _P, _I, _P, _I]),
            "orc_dequant_f32": (None, [_P, _I, _I, _I, _D, C.c_int32, _P, _I]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args

    # ---- seeded std::mt19937_64 fixtures (test_util.hpp:10-54)
    def rng(self, seed: int) -> "Rng":
        return Rng(self, seed)

    # ---- GEMM core
    def naive_gemm_i32(self, a: np.ndarray, b: np.ndarray, threads: int = 0) -> np.ndarray:
        threads = threads or os.cpu_count() or 1
        a = np.ascontiguousarray(a, dtype=np.uint8)
        b = np.ascontiguousarray(b, dtype=np.int8)
        m, k = a.shape
        n = b.shape[1]
        c = np.zeros((m, n), dtype=np.int32)
        self.L.orc_naive_gemm_i32(_p(a), m, k, k, _p(b), n, n, _p(c), n, threads)
        return c

    def col_offsets(self, b: np.ndarray) -> np.ndarray:
        b = np.ascontiguousarray(b, dtype=np.int8)
        out = np.zeros(b.shape[1], dtype=np.int32)
        self.L.orc_col_offsets(_p(b), b.shape[0], b.shape[1], b.shape[1], _p(out))
        return out

    def row_offsets(self, a: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint8)
        out = np.zeros(a.shape[0], dtype=np.int32)
        self.L.orc_row_offsets(_p(a), a.shape[0], a.shape[1], a.shape[1], _p(out))
        return out

    def requant_matrix(self, acc, rowsum, colsum, zp_a, zp_b, k_total, bias, rounding, mult, zp_c, relu,
                       per_channel=None) -> np.ndarray:
        """pipeline.hpp:176-190 over a whole int32 accumulator matrix.
        zp_b / mult: scalar (per-tensor) or length-N arrays (per-channel)."""
        acc = np.ascontiguousarray(acc, dtype=np.int32)
        m, n = acc.shape
        pc = np.ndim(zp_b) > 0 or np.ndim(mult) > 0 if per_channel is None else per_channel
        zpb = np.ascontiguousarray(np.broadcast_to(np.asarray(zp_b, dtype=np.int32), (n,)) if pc
                                   else np.asarray([zp_b], dtype=np.int32))
        md = np.ascontiguousarray(np.broadcast_to(np.asarray(mult, dtype=np.float64), (n,)) if pc
                                  else np.asarray([mult], dtype=np.float64))
        mf = np.ascontiguousarray(np.broadcast_to(np.asarray(mult, dtype=np.float32), (n,)) if pc
                                  else np.asarray([mult], dtype=np.float32))
        rs = None if rowsum is None else np.ascontiguousarray(rowsum, dtype=np.int32)
        cs = np.ascontiguousarray(colsum, dtype=np.int32)
        bi = None if bias is None else np.ascontiguousarray(bias, dtype=np.int32)
        out = np.zeros((m, n), dtype=np.uint8)
        self.L.orc_requant_matrix(_p(acc), m, n, n, _p(rs), _p(cs), zp_a, _p(zpb), 1 if pc else 0, k_total,
                                  _p(bi), rounding, _p(md), _p(mf), zp_c, 1 if relu else 0, _p(out), n)
        return out

    # ---- outlier split / SpMDMAdd / WriteDequantF32 (sparse.hpp:33-80, pipeline.hpp:199-207)
    def split_outliers(self, b: np.ndarray, threshold: int):
        """-> (dense_small, col_ptr, row_idx, values)"""
        b = np.ascontiguousarray(b, dtype=np.int8)
        k, n = b.shape
        dense = np.zeros_like(b)
        cp = np.zeros(n + 1, dtype=np.int32)
        ri = np.zeros(k * n, dtype=np.int32)
        vals = np.zeros(k * n, dtype=np.int8)
        nnz = self.L.orc_split_outliers(_p(b), k, n, n, threshold, _p(dense), n, _p(cp), _p(ri), _p(vals), k * n)
        return dense, cp, ri[:nnz].copy(), vals[:nnz].copy()

    def spmdm_add(self, a, col_ptr, row_idx, values, acc):
        """acc (M x N int32, modified copy) += A x sparse"""
        a = np.ascontiguousarray(a, dtype=np.uint8)
        out = np.array(acc, dtype=np.int32, copy=True, order="C")
        cp = np.ascontiguousarray(col_ptr, dtype=np.int32)
        ri = np.ascontiguousarray(row_idx, dtype=np.int32)
        vals = np.ascontiguousarray(values, dtype=np.int8)
        self.L.orc_spmdm_add(_p(a), a.shape[0], a.shape[1], a.shape[1], _p(cp), _p(ri), _p(vals), out.shape[1],
                             _p(out), out.shape[1])
        return out

    def dequant_f32(self, acc, scale: float, zero_point: int):
        acc = np.ascontiguousarray(acc, dtype=np.int32)
        out = np.zeros(acc.shape, dtype=np.float32)
        self.L.orc_dequant_f32(_p(acc), acc.shape[0], acc.shape[1], acc.shape[1], scale, zero_point, _p(out),
                               acc.shape[1])
        return out

    def prepack_ref(self, b: np.ndarray, ncb: int, kcb: int, nr: int) -> np.ndarray:
        b = np.ascontiguousarray(b, dtype=np.int8)
        k, n = b.shape
        out = np.zeros(self.L.orc_prepack_ref_size(k, n, ncb, kcb), dtype=np.int8)
        self.L.orc_prepack_ref(_p(b), k, n, n, ncb, kcb, nr, _p(out))
        return out

    def im2col3x3(self, x: np.ndarray, zp_a: int, threads: int = 0) -> np.ndarray:
        threads = threads or os.cpu_count() or 1
        x = np.ascontiguousarray(x, dtype=np.uint8)
        nb, h, w, c = x.shape
        cols = np.zeros((nb * h * w, 9 * c), dtype=np.uint8)
        self.L.orc_im2col3x3(_p(x), nb, h, w, c, zp_a, _p(cols), threads)
        return cols

    def conv3x3_i32(self, x: np.ndarray, zp_a: int, wt: np.ndarray, threads: int = 0) -> np.ndarray:
        threads = threads or os.cpu_count() or 1
        x = np.ascontiguousarray(x, dtype=np.uint8)
        nb, h, w, c = x.shape
        wt = np.ascontiguousarray(wt, dtype=np.int8).reshape(9 * c, -1)
        oc = wt.shape[1]
        acc = np.zeros((nb * h * w, oc), dtype=np.int32)
        self.L.orc_conv3x3_i32(_p(x), nb, h, w, c, zp_a, _p(wt), oc, _p(acc), threads)
        return acc

    def dwconv3x3(self, x, zp_a, wt, zp_w, bias, mult, zp_c, relu, threads: int = 0):
        threads = threads or os.cpu_count() or 1
        x = np.ascontiguousarray(x, dtype=np.uint8)
        nb, h, w, c = x.shape
        wt = np.ascontiguousarray(wt, dtype=np.int8).reshape(9, c)
        zp_w = np.ascontiguousarray(zp_w, dtype=np.int32)
        bias = None if bias is None else np.ascontiguousarray(bias, dtype=np.int32)
        mult = np.ascontiguousarray(mult, dtype=np.float32)
        out = np.zeros_like(x)
        acc = np.zeros(x.shape, dtype=np.int32)
        self.L.orc_dwconv3x3(_p(x), nb, h, w, c, zp_a, _p(wt), _p(zp_w), _p(bias), _p(mult), zp_c,
                             1 if relu else 0, _p(out), _p(acc), threads)
        return out, acc


class Rng:
    """std::mt19937_64 with the reference fixture helpers (test_util.hpp)."""

    def __init__(self, orc: Oracle, seed: int):
        self.o = orc
        self.h = C.c_void_p(orc.L.orc_rng_new(seed))

    def __del__(self):
        try:
            self.o.L.orc_rng_free(self.h)
        except Exception:
            pass

    def next(self) -> int:
        return int(self.o.L.orc_rng_next(self.h))

    def u8_matrix(self, rows: int, cols: int) -> np.ndarray:
        a = np.empty((rows, cols), dtype=np.uint8)
        self.o.L.orc_rng_u8(self.h, _p(a), a.size)
        return a

    def i8_matrix(self, rows: int, cols: int) -> np.ndarray:
        a = np.empty((rows, cols), dtype=np.int8)
        self.o.L.orc_rng_i8(self.h, _p(a), a.size)
        return a

    def u8(self, shape) -> np.ndarray:
        a = np.empty(shape, dtype=np.uint8)
        self.o.L.orc_rng_u8(self.h, _p(a), a.size)
        return a

    def i8(self, shape) -> np.ndarray:
        a = np.empty(shape, dtype=np.int8)
        self.o.L.orc_rng_i8(self.h, _p(a), a.size)
        return a

    def int(self, lo: int, hi: int) -> int:
        return int(self.o.L.orc_rng_int(self.h, lo, hi))

    def ints(self, lo: int, hi: int, count: int) -> np.ndarray:
        a = np.empty(count, dtype=np.int32)
        self.o.L.orc_rng_int_fill(self.h, lo, hi, _p(a), count)
        return a

    def real(self, lo: float, hi: float) -> float:
        return float(self.o.L.orc_rng_real(self.h, lo, hi))

    def reals(self, lo: float, hi: float, count: int) -> np.ndarray:
        a = np.empty(count, dtype=np.float64)
        self.o.L.orc_rng_real_fill(self.h, lo, hi, _p(a), count)
        return a


class RefLib:
    """The unmodified reference (execute_gemm & co) through ref_shim.cpp."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (needs /root/reference at build time)")
        L = self.L = C.CDLL(str(path))
        sig = {
            "refx_last_error": (C.c_char_p, []),
            "refx_select_blocking": (_I, [_I, _I, _I, _P, _P]),
            "refx_prepack": (_P, [_P, _I, _I, _I, _P]),
            "refx_free": (None, [_P]),
            "refx_packed_size": (C.c_longlong, [_P]),
            "refx_packed_data": (None, [_P, _P]),
            "refx_col_offsets": (None, [_P, _P]),
            "refx_max_abs": (_I, [_P]),
            "refx_unpack": (_I, [_P, _P]),
            "refx_gemm_raw": (_I, [_P, _I, _I, _I, _P, _P, _I, _I]),
            "refx_gemm_requant": (_I, [_P, _I, _I, _I, _P, _D, _I, _I, _I, _P, _I, _P, _I, _I]),
            "refx_naive_gemm": (_I, [_P, _I, _I, _I, _P, _I, _I, _P]),
            "refx_requantize_scalar": (_I, [C.c_int32, C.c_int32, C.c_int32, _D, _I, _I, _I, _I, _P, _I, _I]),
            "refx_requantize_adjust": (C.c_longlong, [C.c_int32, C.c_int32, C.c_int32, _I, _I, _I, C.c_int32]),
            "refx_pipeline_validate": (_I, [_P, _I, C.c_char_p, _I]),
            "refx_split_outliers": (_I, [_P, _I, _I, _I, _I, _P, _P, _P, _P, _I, _P]),
            "refx_gemm_pipeline": (_I, [_P, _I, _I, _I, _P, _P, _P, _P, _I, _P, _I, _D, _I, _I, _I, _P, _I, _P, _D,
                                        _I, _P, _I, _I]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args

    def _chk(self, rc):
        if rc != 0:
            raise ValueError(self.L.refx_last_error().decode())

    def select_blocking(self, m, n, k, defaults=(56, 32, 256, 14, 32)):
        d = np.asarray(defaults, dtype=np.int32)
        out = np.zeros(5, dtype=np.int32)
        self._chk(self.L.refx_select_blocking(m, n, k, _p(d), _p(out)))
        return tuple(int(v) for v in out)

    def prepack(self, b: np.ndarray, bp=(56, 32, 256, 14, 32)):
        b = np.ascontiguousarray(b, dtype=np.int8)
        bpa = np.asarray(bp, dtype=np.int32)
        h = self.L.refx_prepack(_p(b), b.shape[0], b.shape[1], b.shape[1], _p(bpa))
        if not h:
            raise ValueError(self.L.refx_last_error().decode())
        return RefPacked(self, h, b.shape[0], b.shape[1])

    def naive_gemm(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.uint8)
        b = np.ascontiguousarray(b, dtype=np.int8)
        out = np.zeros((a.shape[0], b.shape[1]), dtype=np.int32)
        self._chk(self.L.refx_naive_gemm(_p(a), a.shape[0], a.shape[1], a.shape[1], _p(b), b.shape[1],
                                         b.shape[1], _p(out)))
        return out

    def requantize_scalar(self, acc, ro, co, mult, zp_a, zp_b, zp_c, k_total, bias=None, col=0):
        b = None if bias is None else np.ascontiguousarray(bias, dtype=np.int32)
        return int(self.L.refx_requantize_scalar(acc, ro, co, mult, zp_a, zp_b, zp_c, k_total, _p(b),
                                                 0 if b is None else len(b), col))

    def requantize_adjust(self, acc, ro, co, zp_a, zp_b, k_total, bias=0):
        return int(self.L.refx_requantize_adjust(acc, ro, co, zp_a, zp_b, k_total, bias))

    def split_outliers(self, b: np.ndarray, threshold: int):
        """the reference's split_outliers -> (dense_small, col_ptr, row_idx, values)"""
        b = np.ascontiguousarray(b, dtype=np.int8)
        k, n = b.shape
        dense = np.zeros_like(b)
        cp = np.zeros(n + 1, dtype=np.int32)
        ri = np.zeros(k * n, dtype=np.int32)
        vals = np.zeros(k * n, dtype=np.int8)
        nnz = C.c_int()
        self._chk(self.L.refx_split_outliers(_p(b), k, n, n, threshold, _p(dense), _p(cp), _p(ri), _p(vals), k * n,
                                             C.byref(nnz)))
        return dense, cp, ri[:nnz.value].copy(), vals[:nnz.value].copy()

    def pipeline_validate(self, kinds):
        k = np.asarray(kinds, dtype=np.int32)
        buf = C.create_string_buffer(512)
        rc = self.L.refx_pipeline_validate(_p(k), len(k), buf, 512)
        return None if rc == 0 else buf.value.decode()


class RefPacked:
    def __init__(self, lib: RefLib, h, k, n):
        self.lib, self.h, self.k, self.n = lib, C.c_void_p(h), k, n

    def __del__(self):
        try:
            self.lib.L.refx_free(self.h)
        except Exception:
            pass

    def data(self):
        out = np.zeros(self.lib.L.refx_packed_size(self.h), dtype=np.int8)
        self.lib.L.refx_packed_data(self.h, _p(out))
        return out

    def col_offsets(self):
        out = np.zeros(self.n, dtype=np.int32)
        self.lib.L.refx_col_offsets(self.h, _p(out))
        return out

    def max_abs(self):
        return int(self.lib.L.refx_max_abs(self.h))

    def gemm_raw(self, a, threads=1):
        a = np.ascontiguousarray(a, dtype=np.uint8)
        out = np.zeros((a.shape[0], self.n), dtype=np.int32)
        self.lib._chk(self.lib.L.refx_gemm_raw(_p(a), a.shape[0], a.shape[1], a.shape[1], self.h, _p(out), self.n,
                                               threads))
        return out

    def gemm_pipeline(self, a, writer, sparse=None, bias_add=None, mult=1.0, zp_a=0, zp_b=0, zp_c=0, rq_bias=None,
                      relu=False, col_offsets=None, dq_scale=1.0, dq_zero_point=0, threads=1):
        """execute_gemm with [SpMDMAdd] [BiasAdd] + writer: 'raw' | 'requant' | 'dequant'.
        sparse = (col_ptr, row_idx, values) of this packed (dense) weight's outliers."""
        a = np.ascontiguousarray(a, dtype=np.uint8)
        m, k = a.shape
        w = {"raw": 0, "requant": 1, "dequant": 2}[writer]
        out = np.zeros((m, self.n), dtype={0: np.int32, 1: np.uint8, 2: np.float32}[w])
        arrs = []

        def arr(x, dt):
            if x is None:
                return None
            v = np.ascontiguousarray(x, dtype=dt)
            arrs.append(v)
            return _p(v)
        cp, ri, vals = sparse if sparse is not None else (None, None, None)
        nnz = 0 if sparse is None else len(vals)
        self.lib._chk(self.lib.L.refx_gemm_pipeline(
            _p(a), m, k, k, self.h, arr(cp, np.int32), arr(ri, np.int32), arr(vals, np.int8), nnz,
            arr(bias_add, np.int32), w, mult, zp_a, zp_b, zp_c, arr(rq_bias, np.int32), 1 if relu else 0,
            arr(col_offsets, np.int32), dq_scale, dq_zero_point, out.ctypes.data, self.n, threads))
        return out

    def gemm_requant(self, a, mult, zp_a, zp_b, zp_c, bias=None, relu=False, threads=1, out=None):
        a = np.ascontiguousarray(a, dtype=np.uint8)
        if out is None:
            out = np.zeros((a.shape[0], self.n), dtype=np.uint8)
        b = None if bias is None else np.ascontiguousarray(bias, dtype=np.int32)
        self.lib._chk(self.lib.L.refx_gemm_requant(_p(a), a.shape[0], a.shape[1], a.shape[1], self.h, mult, zp_a,
                                                   zp_b, zp_c, _p(b), 1 if relu else 0, _p(out), self.n, threads))
        return out
