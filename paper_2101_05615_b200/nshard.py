"""N-sharded multi-GPU GEMM: SURVEY §8(e)'s optional N-sharding.

The reference splits a GEMM only by rows (`execute_gemm`'s worker stripes,
/root/reference/proj/include/q8gemm/engine.hpp:39-47,102-103), and row
sharding stays the default multi-GPU mode (bench.py --gpus N).  When the
weight is what has to be split -- B too large to replicate, or M too small to
shard by rows -- each GPU packs a contiguous column range of B and computes
those output columns for all M rows; every GPU then needs the whole M x N
output.

B200-native gather: no separate collective pass.  The output of every rank
is a symmetric-memory buffer (torch.distributed._symmetric_memory: one
allocation per rank, peers mapped over NVLink), and the GEMM's epilogue
writes each finished tile of its columns to the local output AND straight to
every peer's output at the same offset (`q8g_gemm_u8s8_requant_peers`: TMA
stores from the epilogue's staging tile in the CTA-pair kernel, so the NVLink
transfer of one tile overlaps the MMAs of the next).  A device-side barrier
over the symmetric buffer then orders the peers' stores before the result is
read.  Without symmetric memory (gloo / CPU, or a build without it) the same
split runs with `all_gather_into_tensor` into [world][M][w_max] and a column
relayout ("allgather" mode) -- the same partition and bit-identical output.

Column ranges come from the reference's own stripe formula applied to
16-column blocks (`column_shard`), so shard outputs start 16-byte aligned.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import replace
from typing import Callable, Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import InvalidArgument, check
from .api import (OutputPipeline, ReluQuantized, Requantize, RequantParams, _stream_ptr, partition_stripes,
                  prepack_weights)

COL_ALIGN = 16      # columns per block: shard outputs start 16-byte aligned (TMA stores)
MAX_PEERS = 7       # q8g_gemm_u8s8_requant_peers: peer outputs per call (8 GPUs of a node)


def column_shard(n: int, rank: int, world: int, align: int = COL_ALIGN) -> tuple[int, int]:
    """Columns [n0, n1) of rank `rank`: engine.hpp:40-47's balanced contiguous
    partition over ceil(n / align) column blocks (empty for ranks past the
    block count)."""
    if n < 1 or world < 1 or not 0 <= rank < world or align < 1:
        raise InvalidArgument(_lib.Q8G_EINVAL, "column_shard: need n >= 1, 0 <= rank < world, align >= 1")
    b0, b1 = partition_stripes((n + align - 1) // align, rank, world)
    return min(b0 * align, n), min(b1 * align, n)


def shard_requant_params(rp: RequantParams, n0: int, n1: int) -> RequantParams:
    """RequantParams of output columns [n0, n1): the per-column vectors sliced,
    the scalars unchanged (the shard's own packed B supplies its colsums)."""
    def cut(v):
        return None if v is None else np.asarray(v)[n0:n1].copy()

    return replace(rp, bias=cut(rp.bias), zp_b_per_channel=cut(rp.zp_b_per_channel),
                   multiplier_f32_per_channel=cut(rp.multiplier_f32_per_channel),
                   multiplier_per_channel=cut(rp.multiplier_per_channel))


def _addr(t, offset: int) -> int:
    return (t if isinstance(t, int) else t.data_ptr()) + offset


def execute_gemm_to_peers(a: torch.Tensor, pw, out: torch.Tensor, peers: Sequence, pipeline: OutputPipeline,
                          col0: int, cache=None, stream=None) -> None:
    """Columns [col0, col0 + pw.n_total) of C = requant(A x B) into `out` (this
    device's whole M x N output, u8) and into every peer output at the same
    offset.  `peers` holds the other ranks' outputs: device pointers (int) of
    buffers shaped like `out` (same leading dimension), or tensors.  The
    writes to the peers are ordered by `stream`; synchronise the ranks before
    reading them."""
    if not (isinstance(a, torch.Tensor) and a.is_cuda and out.is_cuda):
        raise InvalidArgument(_lib.Q8G_EINVAL, "execute_gemm_to_peers: A and out must be device views")
    if out.dtype != torch.uint8 or pipeline.writer() is not Requantize or pipeline.general():
        raise InvalidArgument(_lib.Q8G_EINVAL, "execute_gemm_to_peers: u8 output through [ReluQuantized] Requantize")
    m, k = a.shape
    n_shard = pw.n_total
    if out.shape[0] != m or col0 < 0 or col0 + n_shard > out.shape[1] or out.stride(1) != 1:
        raise InvalidArgument(_lib.Q8G_EINVAL, "execute_gemm_to_peers: shard columns must lie inside out")
    if len(peers) > MAX_PEERS:
        raise InvalidArgument(_lib.Q8G_EINVAL, "execute_gemm_to_peers: 0 to 7 peer outputs")
    if n_shard == 0:
        return
    lib = _lib.load()
    ep = pipeline.epilogue(pw)
    ldc = out.stride(0)
    plist = (C.c_void_p * max(1, len(peers)))(*[_addr(p, col0) for p in peers])
    check(lib.q8g_gemm_u8s8_requant_peers(a.data_ptr(), m, k, a.stride(0), pw.handle, ep, _addr(out, col0), plist,
                                          len(peers), ldc, 0, m, None if cache is None else cache.handle,
                                          _stream_ptr(stream)))


def assemble_columns(gathered: torch.Tensor, widths: Sequence[int], out: torch.Tensor) -> None:
    """allgather mode: gathered[r, :, :widths[r]] are rank r's columns, in rank
    order; lay them side by side into out (M x N)."""
    c0 = 0
    for r, w in enumerate(widths):
        if w:
            out[:, c0:c0 + w].copy_(gathered[r, :, :w])
        c0 += w


class NShardedGemm:
    """One rank's part of a column-sharded GEMM over a torch.distributed group.

    b: the whole K x N int8 weight (every rank passes the same); rp / relu:
    the whole layer's requant parameters.  Rank r packs columns
    column_shard(N, r, world) on `device`.  Calling it with this rank's copy of
    A (M x K, u8, on `device`) returns the whole M x N u8 output on every rank.

    mode "peers" (NCCL + symmetric memory): the output is a symmetric buffer
    of m_max rows and the epilogue stores into every rank's copy directly.
    mode "allgather": shard output + all_gather_into_tensor + relayout.
    `compute(a, n0, n1)` replaces the device GEMM of a shard in allgather mode
    (host-logic tests on gloo); by default the shard runs through
    execute_gemm.
    """

    def __init__(self, b: np.ndarray, rp: RequantParams, relu: bool, m_max: int, group=None,
                 device: Optional[torch.device] = None, mode: Optional[str] = None,
                 compute: Optional[Callable] = None):
        import torch.distributed as dist

        self.group = group if group is not None else dist.group.WORLD
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        k, n = b.shape
        self.k, self.n, self.m_max = k, n, m_max
        self.n0, self.n1 = column_shard(n, self.rank, self.world)
        self.widths = [column_shard(n, r, self.world)[1] - column_shard(n, r, self.world)[0]
                       for r in range(self.world)]
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        self.compute = compute
        self.rp_shard = shard_requant_params(rp, self.n0, self.n1)
        stages = ([ReluQuantized()] if relu else []) + [Requantize(self.rp_shard)]
        self.pipeline = OutputPipeline(stages)
        self.pw = None
        if compute is None and self.n1 > self.n0:
            self.pw = prepack_weights(np.ascontiguousarray(b[:, self.n0:self.n1]), device=self.device.index or 0)
        if mode is None:
            mode = "peers" if (self.device.type == "cuda" and dist.get_backend(self.group) == "nccl") else "allgather"
        if mode not in ("peers", "allgather"):
            raise InvalidArgument(_lib.Q8G_EINVAL, "NShardedGemm: mode must be 'peers' or 'allgather'")
        if mode == "peers" and self.world - 1 > MAX_PEERS:
            raise InvalidArgument(_lib.Q8G_EINVAL, "NShardedGemm: peers mode serves up to 8 ranks")
        self.mode = mode
        if mode == "peers":
            import torch.distributed._symmetric_memory as symm_mem

            self.out = symm_mem.empty((m_max, n), dtype=torch.uint8, device=self.device)
            self.handle = symm_mem.rendezvous(self.out, self.group)
            self.peer_ptrs = [int(self.handle.buffer_ptrs[r]) for r in range(self.world) if r != self.rank]
        else:
            self.out = torch.empty((m_max, n), dtype=torch.uint8, device=self.device)

    def __call__(self, a, stream=None) -> torch.Tensor:
        import torch.distributed as dist

        m = a.shape[0]
        if m > self.m_max or a.shape[1] != self.k:
            raise InvalidArgument(_lib.Q8G_EINVAL, "NShardedGemm: A must be M x K with M <= m_max")
        out = self.out[:m]
        if self.mode == "peers":
            if self.pw is not None:
                # the peers' outputs share this buffer's leading dimension (n)
                execute_gemm_to_peers(a, self.pw, out, self.peer_ptrs, self.pipeline, self.n0, stream=stream)
            # every rank's peer stores have landed: the symmetric-memory barrier
            # runs on the GEMM's stream, after this rank's stores
            if stream is None:
                self.handle.barrier()
            else:
                with torch.cuda.stream(stream):
                    self.handle.barrier()
            return out
        wmax = max(self.widths)
        shard = torch.zeros((m, wmax), dtype=torch.uint8, device=self.device)
        if self.n1 > self.n0:
            if self.compute is not None:
                shard[:, :self.n1 - self.n0] = torch.as_tensor(self.compute(a, self.n0, self.n1))
            else:
                from .api import execute_gemm
                view = torch.empty((m, self.n1 - self.n0), dtype=torch.uint8, device=self.device)
                execute_gemm(a, self.pw, view, self.pipeline, stream=stream)
                shard[:, :self.n1 - self.n0] = view
        gathered = torch.empty((self.world * m, wmax), dtype=torch.uint8, device=self.device)
        dist.all_gather_into_tensor(gathered, shard, group=self.group)  # rank-major along dim 0
        assemble_columns(gathered.view(self.world, m, wmax), self.widths, out)
        return out
