"""Outlier split + SpMDMAdd + BiasAdd + every writer.

CPU: the oracle restatement (oracle.c orc_split_outliers / orc_spmdm_add /
orc_dequant_f32) and the C-ABI split (q8g_split_outliers) against fixtures
produced by the UNMODIFIED reference (tests/golden/ref_sparse.npz,
make_golden.py --only-sparse: sparse.hpp:33-80 + execute_gemm with
[SpMDMAdd, BiasAdd] and WriteRawI32 / [ReluQuantized] Requantize /
WriteDequantF32).

GPU (-m gpu): q8g_gemm_u8s8_pipeline (tensor-core dense GEMM + post.cu)
bit-exact against the same fixtures, and at larger shapes against the
oracle (both GEMM tile kinds).
"""
from pathlib import Path

import numpy as np
import pytest

import paper_2101_05615_b200 as q8

GOLD = Path(__file__).resolve().parent / "golden" / "ref_sparse.npz"


def _cases():
    g = np.load(GOLD)
    out = []
    for i in range(int(g["count"])):
        c = {key.split("_", 1)[1]: g[key] for key in g.files if key.startswith(f"{i}_")}
        out.append(c)
    return out


CASES = _cases()


def _bias_add(c):
    return c["bias_add"] if "bias_add" in c else None


def _oracle_acc(orc, c):
    dense, cp, ri, vals = orc.split_outliers(c["b"], int(c["threshold"]))
    acc = orc.spmdm_add(c["a"], cp, ri, vals, orc.naive_gemm_i32(c["a"], dense))
    if _bias_add(c) is not None:
        acc = (acc.astype(np.int64) + _bias_add(c)).astype(np.int32)
    return acc


@pytest.mark.parametrize("i", range(len(CASES)))
def test_oracle_split_spmdm_dequant_vs_reference(orc, i):
    c = CASES[i]
    dense, cp, ri, vals = orc.split_outliers(c["b"], int(c["threshold"]))
    assert (cp == c["col_ptr"]).all() and (ri == c["row_idx"]).all() and (vals == c["values"]).all()
    assert ((dense == 0) | (np.abs(dense.astype(int)) < int(c["threshold"]))).all()
    acc = _oracle_acc(orc, c)
    assert (acc == c["raw"]).all()
    k = int(c["k"])
    rq = orc.requant_matrix(acc, orc.row_offsets(c["a"]), c["col_offsets"], int(c["zp_a"]), int(c["zp_b"]), k,
                            c["rq_bias"], 0, float(c["mult"]), int(c["zp_c"]), bool(c["relu"]))
    assert (rq == c["requant"]).all()
    assert np.array_equal(orc.dequant_f32(acc, float(c["dq_scale"]), int(c["dq_zp"])), c["dequant"])


@pytest.mark.parametrize("i", range(0, len(CASES), 3))
def test_abi_split_outliers_vs_reference(i):
    c = CASES[i]
    sw = q8.split_outliers(c["b"], int(c["threshold"]))
    assert (sw.sparse.col_ptr == c["col_ptr"]).all()
    assert (sw.sparse.row_idx == c["row_idx"]).all() and (sw.sparse.values == c["values"]).all()
    assert sw.sparse.k_total == int(c["k"]) and sw.sparse.n_total == int(c["n"])
    rebuilt = sw.dense_small.astype(np.int32)
    for j in range(sw.sparse.n_total):
        for p in range(sw.sparse.col_ptr[j], sw.sparse.col_ptr[j + 1]):
            rebuilt[sw.sparse.row_idx[p], j] += sw.sparse.values[p]
    assert (rebuilt == c["b"]).all()


def test_split_outliers_errors():
    with pytest.raises(q8.InvalidArgument, match="threshold must be >= 1"):
        q8.split_outliers(np.ones((2, 2), np.int8), 0)


def test_pipeline_validation_messages_for_new_stages():
    with pytest.raises(q8.InvalidArgument, match="SpMDMAdd requires a sparse matrix"):
        q8.OutputPipeline([q8.SpMDMAdd(None), q8.WriteRawI32()])
    with pytest.raises(q8.InvalidArgument, match="the writer must be the last stage"):
        q8.OutputPipeline([q8.WriteDequantF32(), q8.WriteRawI32()])
    with pytest.raises(q8.InvalidArgument, match="ReluQuantized must immediately precede a Requantize"):
        q8.OutputPipeline([q8.ReluQuantized(), q8.WriteDequantF32()])
    p = q8.OutputPipeline([q8.BiasAdd([1]), q8.WriteDequantF32(q8.QuantParams(0.5, 3))])
    assert p.general() and p.writer() is q8.WriteDequantF32


# ------------------------------------------------------------------ GPU


def _run_gpu(c, writer, device_views=True):
    import torch
    sw = q8.split_outliers(c["b"], int(c["threshold"]))
    pw = q8.prepack_weights(sw.dense_small)
    m, n, k = int(c["m"]), int(c["n"]), int(c["k"])
    stages = [q8.SpMDMAdd(sw.sparse)]
    if _bias_add(c) is not None:
        stages.append(q8.BiasAdd(_bias_add(c)))
    if writer == "raw":
        stages.append(q8.WriteRawI32())
        dt = np.int32
    elif writer == "dequant":
        stages.append(q8.WriteDequantF32(q8.QuantParams(float(c["dq_scale"]), int(c["dq_zp"]))))
        dt = np.float32
    else:
        if bool(c["relu"]):
            stages.append(q8.ReluQuantized())
        stages.append(q8.Requantize(q8.RequantParams(multiplier=float(c["mult"]), zp_a=int(c["zp_a"]),
                                                     zp_b=int(c["zp_b"]), zp_c=int(c["zp_c"]), k_total=k,
                                                     bias=c["rq_bias"]), col_offsets=c["col_offsets"]))
        dt = np.uint8
    pipe = q8.OutputPipeline(stages)
    if device_views:
        a = torch.from_numpy(c["a"]).cuda()
        out = torch.zeros((m, n), dtype={np.int32: torch.int32, np.float32: torch.float32,
                                         np.uint8: torch.uint8}[dt], device="cuda")
        q8.execute_gemm(a, pw, out, pipe)
        torch.cuda.synchronize()
        return out.cpu().numpy()
    out = np.zeros((m, n), dtype=dt)
    q8.execute_gemm(c["a"], pw, out, pipe)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(CASES)))
def test_gpu_pipeline_vs_reference_fixture(cuda, i):
    c = CASES[i]
    before = q8.launch_stats()["post"]
    assert (_run_gpu(c, "raw") == c["raw"]).all()
    assert (_run_gpu(c, "requant") == c["requant"]).all()
    assert np.array_equal(_run_gpu(c, "dequant", device_views=(i % 2 == 0)), c["dequant"])
    assert q8.launch_stats()["post"] == before + 3


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k,thr", [(128, 4096, 1024, 100), (300, 512, 640, 120), (1, 256, 4096, 127)])
def test_gpu_pipeline_large_vs_oracle(cuda, orc, m, n, k, thr):
    import torch
    import configs
    c = configs.gemm_case(orc, "C1", m, n, k, seed=m + n + k + thr)
    sw = q8.split_outliers(c.b, thr)
    pw = q8.prepack_weights(sw.dense_small)
    acc = orc.naive_gemm_i32(c.a, c.b)  # dense + outliers == the original B
    a = torch.from_numpy(c.a).cuda()
    # requant F32_RNE per-channel with the original B's column offsets, ReLU
    rp = q8.RequantParams(zp_a=c.zp_a, zp_c=c.zp_c, k_total=k, bias=c.bias, zp_b_per_channel=c.zp_b,
                          multiplier_f32_per_channel=c.mult_f32, rounding=q8.ROUND_F32_RNE)
    pipe = q8.OutputPipeline([q8.SpMDMAdd(sw.sparse), q8.ReluQuantized(),
                              q8.Requantize(rp, col_offsets=orc.col_offsets(c.b))])
    out = torch.zeros((m, n), dtype=torch.uint8, device="cuda")
    q8.execute_gemm(a, pw, out, pipe)
    exp = orc.requant_matrix(acc, orc.row_offsets(c.a), orc.col_offsets(c.b), c.zp_a, c.zp_b, k, c.bias, 1,
                             c.mult_f32, c.zp_c, True)
    assert (out.cpu().numpy() == exp).all()
    # dequant with a BiasAdd stage, two worker stripes
    ba = np.arange(n, dtype=np.int32) * 3 - 1000
    pipe = q8.OutputPipeline([q8.SpMDMAdd(sw.sparse), q8.BiasAdd(ba), q8.WriteDequantF32(q8.QuantParams(0.0021, 7))])
    outf = torch.zeros((m, n), dtype=torch.float32, device="cuda")
    for t in (1, 0):
        q8.execute_gemm(a, pw, outf, pipe, thread_id=t, num_threads=2)
    torch.cuda.synchronize()
    assert np.array_equal(outf.cpu().numpy(), orc.dequant_f32((acc.astype(np.int64) + ba).astype(np.int32), 0.0021, 7))


@pytest.mark.gpu
def test_gpu_pipeline_sparse_shape_mismatch(cuda, orc):
    import torch
    b = orc.rng(3).i8_matrix(64, 32)
    sw = q8.split_outliers(b, 100)
    pw = q8.prepack_weights(orc.rng(4).i8_matrix(64, 48))  # other N
    pipe = q8.OutputPipeline([q8.SpMDMAdd(sw.sparse), q8.WriteRawI32()])
    with pytest.raises(q8.InvalidArgument, match="block extents out of bounds"):
        q8.execute_gemm(torch.zeros((4, 64), dtype=torch.uint8, device="cuda"), pw,
                        torch.zeros((4, 48), dtype=torch.int32, device="cuda"), pipe)
