"""Multi-rank host logic on CPU: two processes over torch.distributed (gloo,
127.0.0.1), the way bench.py runs one process per GPU.

- row sharding: each rank computes the stripe stripe_rows(m, rank, world)
  gives it (engine.hpp:40-47 partition over 128-row blocks; here the oracle
  stands in for the GPU kernel), the stripes are gathered and must equal the
  single-process result bit for bit, ragged last stripe and empty ranks
  included -- the path shards with no data-path collective;
- strong scaling (bench.py --gpus N): the C2 row stripes and the C3 / C4
  image ranges of the ranks cover the whole configuration exactly once, and
  the headline value is the configuration's total ops over the
  max-over-ranks step time;
- timing: bench.max_over_ranks takes the element-wise max over ranks.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(m, n, k):
    from oracle.py import Oracle
    orc = Oracle()
    rng = orc.rng(77)
    a = rng.u8_matrix(m, k)
    b = rng.i8_matrix(k, n)
    bias = rng.ints(-1000, 1000, n).astype(np.int32)
    zp_b = rng.ints(-10, 10, n).astype(np.int32)
    mult = (rng.reals(0.0005, 0.002, n)).astype(np.float32)
    return orc, a, b, bias, zp_b, mult


def _requant_rows(orc, a, b, bias, zp_b, mult):
    acc = orc.naive_gemm_i32(a, b)
    return orc.requant_matrix(acc, orc.row_offsets(a), orc.col_offsets(b), 128, zp_b, a.shape[1], bias,
                              1, mult, 5, True)  # 1 = F32_RNE


def _worker(rank, world, port, m, n, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2101_05615_b200 import api
        orc, a, b, bias, zp_b, mult = _problem(m, n, k)
        r0, r1 = api.stripe_rows(m, rank, world)
        part = _requant_rows(orc, a[r0:r1], b, bias, zp_b, mult) if r1 > r0 else np.zeros((0, n), np.uint8)
        parts = [None] * world
        dist.all_gather_object(parts, (r0, r1, part))
        # timing reduction: the slowest rank sets every timing
        t = bench.max_over_ranks([1.0 + rank, 10.0 - rank, 0.5 * (rank + 1)], torch.device("cpu"), world)
        if rank == 0:
            q.put((parts, t))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,world", [(300, 2), (100, 2), (640, 2)])
def test_row_sharding_two_ranks_matches_single_process(m, world):
    n, k = 48, 72
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts, t = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # disjoint, ordered, covering stripes
    bounds = [(r0, r1) for r0, r1, _ in parts]
    assert bounds[0][0] == 0 and bounds[-1][1] == m
    for (a0, a1), (b0, b1) in zip(bounds, bounds[1:]):
        assert a1 == b0
    got = np.concatenate([p for _, _, p in parts], axis=0)
    orc, a, b, bias, zp_b, mult = _problem(m, n, k)
    np.testing.assert_array_equal(got, _requant_rows(orc, a, b, bias, zp_b, mult))
    assert t == [float(world), 10.0, 0.5 * world]


def test_strong_scaling_partitions_cover_each_config_once():
    import bench
    for world in (1, 2, 4, 8, 3):
        m = bench.GEMM_CONFIGS["C2"][0]
        stripes = [bench.gemm_rows(m, r, world) for r in range(world)]
        assert stripes[0][0] == 0 and stripes[-1][1] == m
        assert all(a[1] == b[0] for a, b in zip(stripes, stripes[1:]))
        assert max(b - a for a, b in stripes) - min(b - a for a, b in stripes) <= 128  # balanced 128-row blocks
        for cfg in ("C3", "C4"):
            nb = bench.CONV_CONFIGS[cfg][0]
            imgs = [bench.image_range(nb, r, world) for r in range(world)]
            assert imgs[0][0] == 0 and imgs[-1][1] == nb
            assert all(a[1] == b[0] for a, b in zip(imgs, imgs[1:]))
    # value = the whole configuration's ops over the slowest rank's step time
    ops = bench.gemm_ops("C2")
    assert ops == 2.0 * 16384 * 4096 * 4096
    assert bench.whole_job_tops(ops, 0.2) == pytest.approx(ops / 0.2e-3 / 1e12)
