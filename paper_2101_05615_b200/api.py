"""Host-side mirror of the reference q8gemm API (proj/include/q8gemm/), on the
B200 C ABI.

Same names, argument meaning and error behaviour as the reference:
  BlockingParams / select_blocking         pack.hpp:15-38, dispatch.hpp:17-30
  prepack_weights -> PackedWeight          pack.hpp:63-79, 146-196
  OutputPipeline + stages                  pipeline.hpp:23-128
  execute_gemm(a, pw, out, pipeline, variant, thread_id, num_threads, cache)
                                           engine.hpp:59-169
  KernelCache(generic_only)                dispatch.hpp:92-146
plus the B200 extensions: per-channel zero points / fp32 multipliers and the
rounding mode on RequantParams, and conv3x3 / depthwise-3x3 entry points.

Matrices: a torch CUDA tensor is a device view (the timed path); a numpy array
is a host view (the reference calling convention: staged H2D/D2H).  Views may
be row slices / column windows with a leading dimension (MatrixView.ld).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import InvalidArgument, check, load

ROUND_REF = _lib.ROUND_REF
ROUND_F32_RNE = _lib.ROUND_F32_RNE
TILE_M = 128  # row granularity of a worker stripe on the GPU (one tcgen05 M tile)

try:  # torch is plumbing only (device memory / streams)
    import torch
except Exception:  # pragma: no cover
    torch = None


class KernelVariant(enum.IntEnum):
    """kernel.hpp:9-12.  kAccI16 is accepted when the reference would accept
    it (i16_accumulation_exact) and runs the exact int32 tensor-core path,
    which is bit-identical to the reference's exact int16 path."""
    kAccI32 = 0
    kAccI16 = 1


def i16_accumulation_exact(max_abs_b: int, kcb: int) -> bool:  # kernel.hpp:28-30
    return 255 * max_abs_b * kcb <= 32767


# ---------------------------------------------------------------- blocking

@dataclass
class BlockingParams:
    mcb: int = 56
    ncb: int = 32
    kcb: int = 256
    mr: int = 14
    nr: int = 32

    @staticmethod
    def defaults() -> "BlockingParams":
        return BlockingParams()

    def _c(self) -> _lib.Blocking:
        return _lib.Blocking(self.mcb, self.ncb, self.kcb, self.mr, self.nr)

    def validate(self) -> None:
        check(load().q8g_blocking_validate(C.byref(self._c())))


def select_blocking(m: int, n: int, k: int, defaults: BlockingParams) -> BlockingParams:
    out = _lib.Blocking()
    check(load().q8g_select_blocking(m, n, k, C.byref(defaults._c()), C.byref(out)))
    return BlockingParams(out.mcb, out.ncb, out.kcb, out.mr, out.nr)


def partition_stripes(num_blocks: int, thread_id: int, num_threads: int) -> tuple[int, int]:
    b, e = C.c_int(), C.c_int()
    check(load().q8g_partition_stripes(num_blocks, thread_id, num_threads, C.byref(b), C.byref(e)))
    return b.value, e.value


# ---------------------------------------------------------------- helpers

def stripe_rows(m: int, thread_id: int, num_threads: int) -> tuple[int, int]:
    """Rows [r0, r1) of worker `thread_id` of `num_threads`: the balanced,
    disjoint stripe of 128-row blocks of engine.hpp:40-47.  The same split
    shards a batch across ranks (one process per GPU, no collective)."""
    nblk = (m + TILE_M - 1) // TILE_M
    b0, b1 = partition_stripes(nblk, thread_id, num_threads)
    return min(b0 * TILE_M, m), min(b1 * TILE_M, m)


def _is_dev(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def _ld(x) -> int:
    if torch is not None and isinstance(x, torch.Tensor):
        if x.dim() != 2 or x.stride(1) != 1:
            raise InvalidArgument(_lib.Q8G_EINVAL, "matrix views must be row-major with unit column stride")
        return x.stride(0)
    if x.ndim != 2 or x.strides[1] != x.itemsize:
        raise InvalidArgument(_lib.Q8G_EINVAL, "matrix views must be row-major with unit column stride")
    return x.strides[0] // x.itemsize


def _ptr(x) -> int:
    return x.data_ptr() if torch is not None and isinstance(x, torch.Tensor) else x.ctypes.data


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream if torch is not None and torch.cuda.is_available() else None
    return getattr(stream, "cuda_stream", stream)


def _i32p(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int32))


# ---------------------------------------------------------------- packed weight

class PackedWeight:
    """pack.hpp:63-79.  Immutable after construction, device resident in the
    tcgen05 K-major 128B-swizzled layout, shareable across concurrent calls."""

    def __init__(self, handle: int, owner=True):
        self._h = C.c_void_p(handle)
        self._owner = owner
        k, n, mx, dev = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        check(load().q8g_packed_b_info(self._h, C.byref(k), C.byref(n), C.byref(mx), C.byref(dev)))
        self.k_total, self.n_total, self.max_abs, self.device = k.value, n.value, mx.value, dev.value
        b = _lib.Blocking()
        check(load().q8g_packed_b_blocking(self._h, C.byref(b)))
        self.blocking = BlockingParams(b.mcb, b.ncb, b.kcb, b.mr, b.nr)
        co = np.zeros(self.n_total, dtype=np.int32)
        check(load().q8g_packed_b_col_offsets(self._h, co.ctypes.data))
        self.col_offsets = co  # ColOffsets over full K (quant.hpp:31-34)

    @property
    def handle(self):
        return self._h

    def unpack(self) -> np.ndarray:
        """Test-only inverse (pack.hpp:199-225)."""
        out = np.zeros((self.k_total, self.n_total), dtype=np.int8)
        check(load().q8g_unpack_b(self._h, out.ctypes.data, self.n_total))
        return out

    def replicate(self, device: int) -> "PackedWeight":
        h = C.c_void_p()
        check(load().q8g_packed_b_replicate(self._h, device, C.byref(h)))
        return PackedWeight(h.value)

    def close(self):
        if self._owner and self._h:
            load().q8g_free_packed_b(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def prepack_weights(b, bp: Optional[BlockingParams] = None, device: int = 0) -> PackedWeight:
    """pack.hpp:146-196.  b: K x N int8 (numpy host array or CUDA tensor)."""
    bp = bp or BlockingParams.defaults()
    h = C.c_void_p()
    if _is_dev(b):
        if b.dtype != torch.int8:
            raise InvalidArgument(_lib.Q8G_EINVAL, "prepack_weights: B must be int8")
        check(load().q8g_pack_b_device(b.data_ptr(), b.shape[0], b.shape[1], _ld(b), C.byref(bp._c()),
                                       b.device.index, _stream_ptr(None), C.byref(h)))
    else:
        b = np.asarray(b)
        if b.dtype != np.int8:
            raise InvalidArgument(_lib.Q8G_EINVAL, "prepack_weights: B must be int8")
        if b.ndim != 2 or b.shape[0] < 1 or b.shape[1] < 1:
            raise InvalidArgument(_lib.Q8G_EINVAL, "prepack_weights: matrix must be non-empty")
        b = np.ascontiguousarray(b)
        check(load().q8g_pack_b(b.ctypes.data, b.shape[0], b.shape[1], b.shape[1], C.byref(bp._c()),
                                device, C.byref(h)))
    return PackedWeight(h.value)


# ---------------------------------------------------------------- pipeline

@dataclass
class RequantParams:
    """quant.hpp:36-43, extended: per-channel zp_b /
    multipliers and the rounding mode.  Default rounding is the reference's
    (fp64 multiply, round half away from zero)."""
    multiplier: float = 1.0
    zp_a: int = 0
    zp_b: int = 0
    zp_c: int = 0
    k_total: int = 1
    bias: Optional[Sequence[int]] = None
    zp_b_per_channel: Optional[Sequence[int]] = None
    multiplier_f32_per_channel: Optional[Sequence[float]] = None
    multiplier_per_channel: Optional[Sequence[float]] = None
    rounding: int = ROUND_REF


@dataclass
class QuantParams:  # quant.hpp:18-21
    scale: float = 1.0      # real units per quantum, > 0
    zero_point: int = 0


@dataclass
class SparseWeightCSC:
    """sparse.hpp:13-21: compressed-sparse-column store of the outlier weight
    entries.  Uploaded to a device on first use (one copy per device)."""
    col_ptr: np.ndarray          # n_total + 1, nondecreasing
    row_idx: np.ndarray          # strictly increasing within each column
    values: np.ndarray           # int8
    k_total: int = 0
    n_total: int = 0

    def nnz(self) -> int:
        return int(len(self.values))

    def _device(self, device: int) -> C.c_void_p:
        hs = self.__dict__.setdefault("_handles", {})
        if device not in hs:
            cp = np.ascontiguousarray(self.col_ptr, dtype=np.int32)
            ri = np.ascontiguousarray(self.row_idx, dtype=np.int32)
            va = np.ascontiguousarray(self.values, dtype=np.int8)
            h = C.c_void_p()
            check(load().q8g_sparse_csc_create(cp.ctypes.data, ri.ctypes.data if len(ri) else None,
                                               va.ctypes.data if len(va) else None, len(va), self.k_total,
                                               self.n_total, device, C.byref(h)))
            hs[device] = h
        return hs[device]

    def __del__(self):
        try:
            for h in self.__dict__.get("_handles", {}).values():
                load().q8g_sparse_csc_free(h)
        except Exception:
            pass


@dataclass
class SplitWeight:  # sparse.hpp:23-29
    dense_small: np.ndarray
    sparse: SparseWeightCSC
    threshold: int = 0


def split_outliers(b, threshold: int) -> SplitWeight:
    """sparse.hpp:33-58: B = dense_small + sparse, the outliers (|v| >=
    threshold) kept at full value in a CSC store.  Preprocessing only."""
    b = np.ascontiguousarray(np.asarray(b), dtype=np.int8)
    if b.ndim != 2:
        raise InvalidArgument(_lib.Q8G_EINVAL, "split_outliers: matrix must be non-empty")
    k, n = b.shape
    nnz = C.c_int()
    check(load().q8g_split_outliers(b.ctypes.data, k, n, n, int(threshold), None, n, None, None, None, 0,
                                    C.byref(nnz)))
    dense = np.zeros_like(b)
    cp = np.zeros(n + 1, dtype=np.int32)
    cap = max(1, nnz.value)
    ri = np.zeros(cap, dtype=np.int32)
    va = np.zeros(cap, dtype=np.int8)
    check(load().q8g_split_outliers(b.ctypes.data, k, n, n, int(threshold), dense.ctypes.data, n, cp.ctypes.data,
                                    ri.ctypes.data, va.ctypes.data, cap, C.byref(nnz)))
    sp = SparseWeightCSC(cp, ri[:nnz.value].copy(), va[:nnz.value].copy(), k, n)
    return SplitWeight(dense, sp, int(threshold))


@dataclass
class SpMDMAdd:  # pipeline.hpp:23-25 (general-pipeline path, post.cu)
    sparse: Optional[SparseWeightCSC] = None


@dataclass
class BiasAdd:  # pipeline.hpp:27-29
    bias: Sequence[int] = ()


@dataclass
class ReluQuantized:  # pipeline.hpp:31
    pass


@dataclass
class Requantize:  # pipeline.hpp:33-36
    params: RequantParams = field(default_factory=RequantParams)
    col_offsets: Optional[Sequence[int]] = None  # None -> the packed weight's own


@dataclass
class WriteRawI32:  # pipeline.hpp:38
    pass


@dataclass
class WriteDequantF32:  # pipeline.hpp:40-42: out = scale * (acc - zero_point)
    c_params: QuantParams = field(default_factory=QuantParams)


_WRITERS = (Requantize, WriteRawI32, WriteDequantF32)


class OutputPipeline:
    """pipeline.hpp:57-128: ordered stages ending in exactly one writer,
    validated at construction with the reference's messages."""

    def __init__(self, stages: Sequence[object]):
        self.stages = list(stages)
        err = OutputPipeline.validate(self.stages)
        if err is not None:
            raise InvalidArgument(_lib.Q8G_EINVAL, "OutputPipeline: " + err)

    @staticmethod
    def validate(stages) -> Optional[str]:
        if not stages:
            return "pipeline is empty; a terminal writer stage is required"
        for i in range(len(stages) - 1):
            if isinstance(stages[i], _WRITERS):
                return f"stage {i + 1} follows a writer; the writer must be the last stage"
        if not isinstance(stages[-1], _WRITERS):
            return "last stage must be a writer (Requantize, WriteRawI32, or WriteDequantF32)"
        for i, s in enumerate(stages):
            if isinstance(s, ReluQuantized):
                if not (i + 2 == len(stages) and isinstance(stages[-1], Requantize)):
                    return "ReluQuantized must immediately precede a Requantize writer"
            if isinstance(s, SpMDMAdd) and s.sparse is None:
                return "SpMDMAdd requires a sparse matrix"
            if isinstance(s, Requantize):
                p = s.params
                if not (p.multiplier > 0) and p.multiplier_f32_per_channel is None and p.multiplier_per_channel is None:
                    return "Requantize multiplier must be positive"
                if p.k_total < 1:
                    return "Requantize k_total must be >= 1"
        return None

    def writer(self):
        return type(self.stages[-1])

    def needs_row_offsets(self) -> bool:  # pipeline.hpp:114-119
        last = self.stages[-1]
        if isinstance(last, Requantize):
            p = last.params
            if p.zp_b_per_channel is not None:
                return bool(np.any(np.asarray(p.zp_b_per_channel) != 0))
            return p.zp_b != 0
        return False

    def has_relu(self) -> bool:
        return len(self.stages) >= 2 and isinstance(self.stages[-2], ReluQuantized)

    def bias_add(self) -> Optional[np.ndarray]:
        acc = None
        for s in self.stages:
            if isinstance(s, BiasAdd):
                b = np.asarray(s.bias, dtype=np.int64)
                acc = b if acc is None else acc + b
        return None if acc is None else acc.astype(np.int32)

    def bias_add_device(self, device):
        """The summed BiasAdd stages as a device tensor, cached on the pipeline
        so it outlives the (asynchronous) launches that read it -- a temporary
        freed at return could be recycled by the caching allocator while a
        kernel on another stream still reads it."""
        ba = self.bias_add()
        if ba is None:
            return None
        cache = self.__dict__.setdefault("_bias_dev", {})
        key = torch.device(device).index
        if key not in cache:
            cache[key] = torch.from_numpy(ba).to(device)
        return cache[key]

    def sparse(self) -> Optional[SparseWeightCSC]:
        for s in self.stages:
            if isinstance(s, SpMDMAdd):
                return s.sparse
        return None

    def general(self) -> bool:
        """True when the pipeline needs the general path (post.cu): an
        SpMDMAdd stage or the WriteDequantF32 writer."""
        return self.sparse() is not None or isinstance(self.stages[-1], WriteDequantF32)

    def epilogue(self, pw: PackedWeight) -> C.c_void_p:
        """Fold [BiasAdd]* [ReluQuantized] Requantize into the device table.
        Cached on this pipeline per packed weight (the pipeline holds a
        reference to the weight, so the key cannot be recycled)."""
        cache = self.__dict__.setdefault("_eps", {})
        hit = cache.get(id(pw))
        if hit is not None and hit[0] is pw:
            return hit[1]
        rq = self.stages[-1]
        assert isinstance(rq, Requantize)
        p = rq.params
        n = pw.n_total
        keep = []

        def arr(x, dt, name):
            if x is None:
                return None
            a = np.ascontiguousarray(np.asarray(x, dtype=dt))
            if a.shape != (n,):
                raise InvalidArgument(_lib.Q8G_EINVAL, f"Requantize: {name} must have N={n} entries")
            keep.append(a)
            return a.ctypes.data_as(C.POINTER({np.int32: C.c_int32, np.float32: C.c_float,
                                               np.float64: C.c_double}[dt]))

        cp = _lib.RequantParamsC()
        cp.multiplier = float(p.multiplier)
        cp.zp_a, cp.zp_b, cp.zp_c, cp.k_total = int(p.zp_a), int(p.zp_b), int(p.zp_c), int(p.k_total)
        cp.bias_host = arr(p.bias, np.int32, "bias") if p.bias is not None and len(p.bias) else None
        cp.zp_b_per_channel_host = arr(p.zp_b_per_channel, np.int32, "zp_b_per_channel")
        cp.multiplier_f32_per_channel_host = arr(p.multiplier_f32_per_channel, np.float32, "multiplier_f32")
        cp.multiplier_per_channel_host = arr(p.multiplier_per_channel, np.float64, "multiplier")
        cp.col_offsets_host = arr(rq.col_offsets, np.int32, "col_offsets")
        cp.rounding = int(p.rounding)
        cp.relu = 1 if self.has_relu() else 0
        ba = self.bias_add()
        if ba is not None:
            keep.append(ba)
        h = C.c_void_p()
        check(load().q8g_epilogue_create(pw.handle, C.byref(cp), None if ba is None else ba.ctypes.data,
                                         C.byref(h)))
        cache[id(pw)] = (pw, h)
        return h

    def __del__(self):
        try:
            for _, h in self.__dict__.get("_eps", {}).values():
                load().q8g_epilogue_free(h)
        except Exception:
            pass


# ---------------------------------------------------------------- dispatch cache

class KernelCache:
    """dispatch.hpp:92-146 analog: memoized shape class -> GPU tile kind."""

    def __init__(self, generic_only: bool = False):
        h = C.c_void_p()
        check(load().q8g_kernel_cache_create(1 if generic_only else 0, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def build_count(self) -> int:
        return int(load().q8g_kernel_cache_build_count(self._h))

    def tile(self, m: int, n: int, k: int, lda: int) -> int:
        t = C.c_int()
        check(load().q8g_kernel_cache_tile(self._h, m, n, k, lda, C.byref(t)))
        return t.value

    def __del__(self):
        try:
            load().q8g_kernel_cache_free(self._h)
        except Exception:
            pass


# ---------------------------------------------------------------- execute

def execute_gemm(a, pw: PackedWeight, out, pipeline: OutputPipeline,
                 variant: KernelVariant = KernelVariant.kAccI32, thread_id: int = 0, num_threads: int = 1,
                 cache: Optional[KernelCache] = None, stream=None) -> None:
    """engine.hpp:59-169.  Each (thread_id, num_threads) call computes a
    disjoint, balanced stripe of 128-row blocks; the union over workers is the
    whole output and is bit-identical to one call (test_engine.cpp:87-139)."""
    m, k = a.shape[0], a.shape[1]
    n = pw.n_total
    if k != pw.k_total:
        raise InvalidArgument(_lib.Q8G_EINVAL, "execute_gemm: A columns must equal the packed weight K")
    if out.shape[0] != m or out.shape[1] != n:
        raise InvalidArgument(_lib.Q8G_EINVAL, "execute_gemm: output must be M x N")
    if num_threads < 1 or thread_id < 0 or thread_id >= num_threads:
        raise InvalidArgument(_lib.Q8G_EINVAL, "execute_gemm: thread_id must be in [0, num_threads)")
    w = pipeline.writer()
    out_is_i32 = (out.dtype == torch.int32) if _is_dev(out) else (out.dtype == np.int32)
    out_is_u8 = (out.dtype == torch.uint8) if _is_dev(out) else (out.dtype == np.uint8)
    out_is_f32 = (out.dtype == torch.float32) if _is_dev(out) else (out.dtype == np.float32)
    if not ((w is WriteRawI32 and out_is_i32) or (w is Requantize and out_is_u8) or
            (w is WriteDequantF32 and out_is_f32)):
        raise InvalidArgument(_lib.Q8G_EINVAL, "pipeline writer does not match the output element type")
    if variant == KernelVariant.kAccI16 and not i16_accumulation_exact(pw.max_abs, pw.blocking.kcb):
        raise InvalidArgument(
            _lib.Q8G_EINVAL,
            f"execute_gemm: INT16 accumulation rejected: 255 * max|B| * kcb = {255 * pw.max_abs * pw.blocking.kcb} "
            "exceeds 32767; split outliers with a threshold satisfying 255 * (T - 1) * kcb <= 32767 "
            "(see max_i16_split_threshold)")
    r0, r1 = stripe_rows(m, thread_id, num_threads)
    if r0 >= r1:
        return
    if pipeline.general():
        _execute_general(a, pw, out, pipeline, r0, r1, cache, stream)
        return
    lib = load()
    cache_h = cache.handle if cache is not None else None
    dev = _is_dev(a)
    if dev != _is_dev(out):
        raise InvalidArgument(_lib.Q8G_EINVAL, "execute_gemm: A and out must both be device or both host views")
    lda, ldc = _ld(a), _ld(out)
    if w is WriteRawI32:
        ba = pipeline.bias_add()
        if dev:
            bdev = None
            if ba is not None:
                bdev = pipeline.bias_add_device(a.device)
            check(lib.q8g_gemm_u8s8_raw_i32(a.data_ptr(), m, k, lda, pw.handle,
                                            None if bdev is None else bdev.data_ptr(), out.data_ptr(), ldc,
                                            r0, r1, cache_h, _stream_ptr(stream)))
        else:
            if ba is not None:
                raise _lib.Q8GError(_lib.Q8G_ENOTSUP, "BiasAdd with WriteRawI32 needs device views")
            check(lib.q8g_gemm_u8s8_raw_i32_host(_ptr(a), m, k, lda, pw.handle, _ptr(out), ldc, r0, r1, None))
    else:
        ep = pipeline.epilogue(pw)
        if dev:
            check(lib.q8g_gemm_u8s8_requant(a.data_ptr(), m, k, lda, pw.handle, ep, out.data_ptr(), ldc, r0, r1,
                                            cache_h, _stream_ptr(stream)))
        else:
            check(lib.q8g_gemm_u8s8_requant_host(_ptr(a), m, k, lda, pw.handle, ep, _ptr(out), ldc, r0, r1, None))


def _execute_general(a, pw: PackedWeight, out, pipeline: OutputPipeline, r0: int, r1: int,
                     cache: Optional[KernelCache], stream) -> None:
    """[SpMDMAdd] [BiasAdd]* [ReluQuantized] writer (pipeline.hpp:157-207)
    through q8g_gemm_u8s8_pipeline; host views are staged through the device
    (the reference's host-view convention, synchronous)."""
    host = not _is_dev(a)
    if host != (not _is_dev(out)):
        raise InvalidArgument(_lib.Q8G_EINVAL, "execute_gemm: A and out must both be device or both host views")
    dev_index = pw.device
    if host:
        a_d = torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{dev_index}")
        out_d = torch.empty(out.shape, dtype={np.dtype(np.int32): torch.int32, np.dtype(np.uint8): torch.uint8,
                                              np.dtype(np.float32): torch.float32}[np.dtype(out.dtype)],
                            device=f"cuda:{dev_index}")
    else:
        a_d, out_d = a, out
    m, k = a_d.shape
    n = pw.n_total
    sp = pipeline.sparse()
    if sp is not None and (sp.k_total != k or sp.n_total != n):
        raise InvalidArgument(_lib.Q8G_EINVAL, "spmdm_block: block extents out of bounds")
    w = pipeline.writer()
    pa = _lib.PipelineArgsC()
    pa.sparse = sp._device(dev_index) if sp is not None else None
    keep = []
    if w is Requantize:
        pa.writer = _lib.Q8G_WRITE_REQUANT_U8
        pa.ep = pipeline.epilogue(pw)  # folds BiasAdd into the table
    else:
        pa.writer = _lib.Q8G_WRITE_RAW_I32 if w is WriteRawI32 else _lib.Q8G_WRITE_DEQUANT_F32
        bdev = pipeline.bias_add_device(a_d.device)
        if bdev is not None:
            pa.bias_add_dev = bdev.data_ptr()
        if w is WriteDequantF32:
            cp = pipeline.stages[-1].c_params
            pa.dq_scale, pa.dq_zero_point = float(cp.scale), int(cp.zero_point)
    check(load().q8g_gemm_u8s8_pipeline(a_d.data_ptr(), m, k, _ld(a_d), pw.handle, C.byref(pa), out_d.data_ptr(),
                                        _ld(out_d), r0, r1, cache.handle if cache is not None else None,
                                        _stream_ptr(stream)))
    if host:
        torch.cuda.synchronize(dev_index)
        res = out_d[r0:r1].cpu().numpy()
        out[r0:r1] = res


# ---------------------------------------------------------------- conv 3x3

def _host_contig(*arrays) -> None:
    for a in arrays:
        contiguous = a.is_contiguous() if isinstance(a, torch.Tensor) else a.flags["C_CONTIGUOUS"]
        if not contiguous:
            raise InvalidArgument(_lib.Q8G_EINVAL, "host views of NHWC tensors must be contiguous")


def prepack_conv3x3_weights(w, device: int = 0) -> PackedWeight:
    """w: [3][3][C][OC] int8 -> packed K=9C x N=OC matrix,
    with the tensor-core operand image built eagerly (q8g_conv3x3_prepare) so
    the weight is immutable from here on."""
    if not _is_dev(w):
        w = np.asarray(w)
    pw = prepack_weights(w.reshape(-1, w.shape[-1]), device=device)
    check(load().q8g_conv3x3_prepare(pw.handle, int(w.shape[2]), None))
    return pw


def execute_conv3x3(x, pw: PackedWeight, out, pipeline: OutputPipeline, zp_a: Optional[int] = None,
                    image_begin: int = 0, image_end: Optional[int] = None, stream=None) -> None:
    """NHWC u8 x [nb,h,w,c] -> out [nb,h,w,oc] (u8 with Requantize, int32 with
    WriteRawI32), stride 1, pad 1 with the quantized zero: Requantize's zp_a,
    or the `zp_a` argument for the raw writer."""
    nb, h, w, c = x.shape
    if out.shape != (nb, h, w, pw.n_total):
        raise InvalidArgument(_lib.Q8G_EINVAL, "conv3x3: output must be [N,H,W,OC]")
    image_end = nb if image_end is None else image_end
    lib = load()
    if not _is_dev(x):
        # host views (the reference convention): chunked, copies overlapped with the convolution
        if _is_dev(out) or pipeline.writer() is not Requantize:
            raise InvalidArgument(_lib.Q8G_EINVAL, "conv3x3: host views need host x and out and the Requantize writer")
        _host_contig(x, out)
        check(lib.q8g_conv3x3_u8s8_nhwc_host(_ptr(x), nb, h, w, c, pw.handle, pipeline.epilogue(pw), _ptr(out),
                                             image_begin, image_end, _stream_ptr(stream)))
        return
    if pipeline.writer() is WriteRawI32:
        zp_a = 0 if zp_a is None else int(zp_a)
        check(lib.q8g_conv3x3_u8s8_nhwc_raw_i32(x.data_ptr(), nb, h, w, c, zp_a, pw.handle, out.data_ptr(),
                                                 image_begin, image_end, _stream_ptr(stream)))
    else:
        ep = pipeline.epilogue(pw)
        check(lib.q8g_conv3x3_u8s8_nhwc(x.data_ptr(), nb, h, w, c, pw.handle, ep, out.data_ptr(), image_begin,
                                        image_end, _stream_ptr(stream)))


# ---------------------------------------------------------------- depthwise 3x3

class DepthwiseFilter:
    """Prepacked depthwise 3x3 filter [3][3][C] int8 with its per-channel
    requantization."""

    def __init__(self, w: np.ndarray, params: RequantParams, relu: bool, device: int = 0):
        w = np.ascontiguousarray(np.asarray(w, dtype=np.int8))
        c = w.shape[-1]
        self.c = c
        keep = []

        def arr(x, dt, ct):
            if x is None:
                return None
            a = np.ascontiguousarray(np.asarray(x, dtype=dt))
            keep.append(a)
            return a.ctypes.data_as(C.POINTER(ct))

        cp = _lib.RequantParamsC()
        cp.multiplier = float(params.multiplier)
        cp.zp_a, cp.zp_b, cp.zp_c, cp.k_total = int(params.zp_a), int(params.zp_b), int(params.zp_c), 9
        cp.bias_host = arr(params.bias, np.int32, C.c_int32)
        cp.zp_b_per_channel_host = arr(params.zp_b_per_channel, np.int32, C.c_int32)
        cp.multiplier_f32_per_channel_host = arr(params.multiplier_f32_per_channel, np.float32, C.c_float)
        cp.rounding = int(params.rounding)
        cp.relu = 1 if relu else 0
        h = C.c_void_p()
        check(load().q8g_dw_filter_create(w.ctypes.data, c, C.byref(cp), device, C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            load().q8g_dw_filter_free(self._h)
        except Exception:
            pass


def execute_dwconv3x3(x, filt: DepthwiseFilter, out, image_begin: int = 0, image_end: Optional[int] = None,
                      stream=None) -> None:
    nb, h, w, c = x.shape
    if out.shape != x.shape:
        raise InvalidArgument(_lib.Q8G_EINVAL, "dwconv3x3: output must be [N,H,W,C]")
    image_end = nb if image_end is None else image_end
    if not _is_dev(x):
        if _is_dev(out):
            raise InvalidArgument(_lib.Q8G_EINVAL, "dwconv3x3: x and out must both be device or both host views")
        _host_contig(x, out)
        check(load().q8g_dwconv3x3_u8s8_nhwc_host(_ptr(x), nb, h, w, c, filt._h, _ptr(out), image_begin, image_end,
                                                  _stream_ptr(stream)))
        return
    check(load().q8g_dwconv3x3_u8s8_nhwc(x.data_ptr(), nb, h, w, c, filt._h, out.data_ptr(), image_begin,
                                         image_end, _stream_ptr(stream)))
