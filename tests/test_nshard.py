"""N-sharded multi-GPU GEMM (optional N-sharding;
paper_2101_05615_b200/nshard.py).

CPU (gloo, world 2 / 3, 127.0.0.1): NShardedGemm in allgather mode with the
oracle standing in for the shard GEMM -- column partition, per-column
parameter slicing, gather and relayout must give the single-process output
bit for bit, ragged last shard and empty ranks included.

GPU (one B200): the peer-store path.  Every "rank" of an N-way split runs on
the one GPU, each with its own M x N output buffer standing in for a peer's;
rank r's call writes its columns into its own buffer and, through
q8g_gemm_u8s8_requant_peers, into all the others.  After all ranks have run,
every buffer must equal the oracle's whole output.  The large-M shapes take
the CTA-pair kernel's TMA peer stores; small M, and a leading dimension that
is not a multiple of 16, take the copy-engine path.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(m, n, k, seed=91):
    from oracle.py import Oracle
    orc = Oracle()
    rng = orc.rng(seed)
    a = rng.u8_matrix(m, k)
    b = rng.i8_matrix(k, n)
    bias = rng.ints(-1000, 1000, n).astype(np.int32)
    zp_b = rng.ints(-10, 10, n).astype(np.int32)
    mult = (rng.reals(0.0005, 0.002, n)).astype(np.float32)
    return orc, a, b, bias, zp_b, mult


def _expected(orc, a, b, bias, zp_b, mult, relu=True):
    acc = orc.naive_gemm_i32(a, b)
    return orc.requant_matrix(acc, orc.row_offsets(a), orc.col_offsets(b), 128, zp_b, a.shape[1], bias,
                              1, mult, 5, relu)  # 1 = F32_RNE


def _rp(q8, k, bias, zp_b, mult):
    return q8.RequantParams(zp_a=128, zp_c=5, k_total=k, bias=bias, zp_b_per_channel=zp_b,
                            multiplier_f32_per_channel=mult, rounding=q8.ROUND_F32_RNE)


def test_column_shard_partition():
    from paper_2101_05615_b200.nshard import COL_ALIGN, column_shard
    for n in (1, 15, 16, 17, 100, 800, 1000, 4096):
        for world in (1, 2, 3, 4, 7, 8):
            sh = [column_shard(n, r, world) for r in range(world)]
            assert sh[0][0] == 0 and sh[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
            assert all(a0 % COL_ALIGN == 0 or a0 == a1 for a0, a1 in sh)  # aligned starts (or empty)
            widths = [b - a for a, b in sh]
            full = [w for w in widths if w]
            assert max(widths) - min(full) <= 2 * COL_ALIGN  # balanced blocks, ragged tail


def test_shard_requant_params_slices_columns():
    import paper_2101_05615_b200 as q8
    from paper_2101_05615_b200.nshard import shard_requant_params
    n = 40
    rp = _rp(q8, 64, np.arange(n, dtype=np.int32), np.arange(n, dtype=np.int32) % 7,
             np.linspace(0.001, 0.002, n).astype(np.float32))
    s = shard_requant_params(rp, 16, 32)
    np.testing.assert_array_equal(s.bias, np.arange(16, 32))
    np.testing.assert_array_equal(s.zp_b_per_channel, np.arange(16, 32) % 7)
    assert s.multiplier_f32_per_channel.shape == (16,) and s.zp_a == 128 and s.zp_c == 5 and s.k_total == 64


def _worker(rank, world, port, m, n, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2101_05615_b200 as q8
        orc, a, b, bias, zp_b, mult = _problem(m, n, k)

        def shard(a_t, n0, n1):  # the oracle stands in for this rank's device GEMM
            return _expected(orc, a_t.numpy(), b[:, n0:n1], bias[n0:n1], zp_b[n0:n1], mult[n0:n1])

        g = q8.NShardedGemm(b, _rp(q8, k, bias, zp_b, mult), relu=True, m_max=m, device="cpu",
                            mode="allgather", compute=shard)
        out = g(torch.from_numpy(a))
        q.put((rank, (g.n0, g.n1), out.numpy().copy()))
    except Exception:  # fail the test at once instead of at the queue timeout
        import traceback
        q.put((rank, None, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,world", [(37, 100, 2), (64, 48, 3), (20, 16, 3)])
def test_nsharded_gemm_allgather_matches_single_process(m, n, world):
    k = 72
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda t: t[0])
    errs = [r[2] for r in res if r[1] is None]
    assert not errs, errs[0]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc, a, b, bias, zp_b, mult = _problem(m, n, k)
    want = _expected(orc, a, b, bias, zp_b, mult)
    for _, _, out in res:  # every rank holds the whole output
        np.testing.assert_array_equal(out, want)


# ---------------------------------------------------------------- GPU: peer stores


def _peer_split(q8, orc, m, n, k, world, ldc=None, seed=91):
    """All `world` ranks of an N-split on one GPU; returns every rank's buffer
    and the oracle's whole output."""
    from paper_2101_05615_b200.nshard import column_shard, execute_gemm_to_peers, shard_requant_params
    _, a, b, bias, zp_b, mult = _problem(m, n, k, seed)
    ldc = ldc or n
    rp = _rp(q8, k, bias, zp_b, mult)
    ad = torch.from_numpy(a).cuda()
    bufs = [torch.full((m, ldc), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(world)]
    views = [t[:, :n] for t in bufs]
    before = q8.launch_stats()
    for r in range(world):
        n0, n1 = column_shard(n, r, world)
        if n1 == n0:
            continue
        pw = q8.prepack_weights(np.ascontiguousarray(b[:, n0:n1]))
        pipe = q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(shard_requant_params(rp, n0, n1))])
        execute_gemm_to_peers(ad, pw, views[r], [views[d] for d in range(world) if d != r], pipe, n0)
    torch.cuda.synchronize()
    after = q8.launch_stats()
    return bufs, _expected(orc, a, b, bias, zp_b, mult), {f: after[f] - before[f] for f in after}


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k,world,tma_peers", [
    (4864, 2048, 256, 2, True),    # CTA-pair kernel: TMA stores to the peer
    (9472, 4096, 128, 4, True),    # CTA-pair kernel, 3 peers
    (9472, 1600, 128, 3, True),    # CTA-pair kernel, 544 / 528 / 528-column shards (partial 512-column tiles)
    (128, 1024, 512, 2, False),    # split-K: copy-engine peer copies
    (300, 1000, 96, 3, False),     # 128-column tiles, ragged N
])
def test_gemm_to_peers_every_rank_holds_the_whole_output(cuda, orc, m, n, k, world, tma_peers):
    import paper_2101_05615_b200 as q8
    bufs, want, launched = _peer_split(q8, orc, m, n, k, world)
    assert launched["gemm_simt"] == 0
    if tma_peers:  # every rank's tiles went to its peers from the epilogue, no copies
        assert launched["gemm_tc_large_m"] == world and launched["peer_copy"] == 0
    else:
        assert launched["peer_copy"] == world * (world - 1)
    for r, t in enumerate(bufs):
        np.testing.assert_array_equal(t.cpu().numpy(), want, err_msg=f"rank {r}'s output")


@pytest.mark.gpu
def test_gemm_to_peers_wide_ldc_leaves_padding_untouched(cuda, orc):
    """ldc = N + 40 (not a multiple of 16: the CTA-pair kernel's TMA path
    declines, the copy engines carry the stripe): columns >= N of every
    buffer keep their canary."""
    import paper_2101_05615_b200 as q8
    m, n, k, world = 4864, 2048, 128, 2
    bufs, want, launched = _peer_split(q8, orc, m, n, k, world, ldc=n + 40)
    assert launched["peer_copy"] == world * (world - 1)
    for t in bufs:
        h = t.cpu().numpy()
        np.testing.assert_array_equal(h[:, :n], want)
        assert (h[:, n:] == 0xA5).all()


@pytest.mark.gpu
def test_gemm_to_peers_argument_errors(cuda):
    import paper_2101_05615_b200 as q8
    from paper_2101_05615_b200.nshard import execute_gemm_to_peers
    pw = q8.prepack_weights(np.ones((32, 32), np.int8))
    pipe = q8.OutputPipeline([q8.Requantize(q8.RequantParams(multiplier=0.01, k_total=32))])
    a = torch.zeros((16, 32), dtype=torch.uint8, device="cuda")
    out = torch.zeros((16, 64), dtype=torch.uint8, device="cuda")
    with pytest.raises(q8.InvalidArgument):
        execute_gemm_to_peers(a, pw, out, [out] * 8, pipe, 0)  # more than 7 peers
    with pytest.raises(q8.InvalidArgument):
        execute_gemm_to_peers(a, pw, out, [], pipe, 48)  # shard past the output
    lib = q8._lib.load()
    import ctypes as C
    rc = lib.q8g_gemm_u8s8_requant_peers(a.data_ptr(), 16, 32, 32, pw.handle, pipe.epilogue(pw), out.data_ptr(),
                                         None, 1, 64, 0, 16, None, None)
    assert rc == q8._lib.Q8G_EINVAL and b"peer output list" in lib.q8g_last_error()
    host = (C.c_uint8 * 64)()
    plist = (C.c_void_p * 1)(C.addressof(host))
    rc = lib.q8g_gemm_u8s8_requant_peers(a.data_ptr(), 16, 32, 32, pw.handle, pipe.epilogue(pw), out.data_ptr(),
                                         plist, 1, 64, 0, 16, None, None)
    assert rc == q8._lib.Q8G_EINVAL and b"device memory" in lib.q8g_last_error()


def _nccl_one_rank(mode, q):
    """world 1 over NCCL on cuda:0: the symmetric-memory allocation,
    rendezvous and barrier of "peers" mode, or the NCCL all-gather of
    "allgather" mode, around the device GEMM."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(_free_port())
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        import paper_2101_05615_b200 as q8
        m, n, k = 2048, 1024, 256
        orc, a, b, bias, zp_b, mult = _problem(m, n, k, seed=5)
        g = q8.NShardedGemm(b, _rp(q8, k, bias, zp_b, mult), relu=True, m_max=m, mode=mode)
        out = g(torch.from_numpy(a).cuda())
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        want = _expected(orc, a, b, bias, zp_b, mult)
        q.put((g.mode, bool((got == want).all())))
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put(("error", traceback.format_exc()))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["peers", "allgather"])
def test_nsharded_gemm_nccl_world_one(cuda, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_one_rank, args=(mode, q))
    p.start()
    got_mode, ok = q.get(timeout=300)
    p.join(timeout=60)
    assert got_mode == mode, ok
    assert ok is True
