"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED
reference (oracle/_ref/libq8ref.so, built by oracle/Makefile from
/root/reference/proj/include).  Run here, where the reference exists:

    python tests/golden/make_golden.py                  # everything
    python tests/golden/make_golden.py --only-sparse    # 5. outlier split / SpMDMAdd / dequant

Inputs are regenerable from the seeds with std::mt19937_64 (the reference
fixture generator, restated in oracle.c and pinned by its published KAT), so
the fixtures store seeds + reference outputs + input digests only.
"""
from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle.py import Oracle, RefLib, build  # noqa: E402
import configs  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    build()
    orc, ref = Oracle(), RefLib()

    # 1. C0 exactly as BASELINE configs[0], REF rounding (the reference's own)
    c = configs.gemm_case(orc, "C0", *configs.CONFIG_SHAPES["C0"])
    pk = ref.prepack(c.b, ref.select_blocking(64, 800, 320))
    acc = pk.gemm_raw(c.a, threads=4)
    out = pk.gemm_requant(c.a, c.mult_f64, c.zp_a, int(c.zp_b), c.zp_c, bias=c.bias, relu=False, threads=4)
    out_relu = pk.gemm_requant(c.a, c.mult_f64, c.zp_a, int(c.zp_b), c.zp_c, bias=c.bias, relu=True, threads=4)
    np.savez_compressed(OUT / "c0_reference.npz", out=out, out_relu=out_relu, acc_sha=sha(acc),
                        a_sha=sha(c.a), b_sha=sha(c.b), bias_sha=sha(c.bias), col_offsets=pk.col_offsets(),
                        max_abs=pk.max_abs())

    # 2. random small shapes: raw accumulators + REF requant (test_engine.cpp:87-113, 199-233 style)
    rng = orc.rng(2024)
    cases = []
    for t in range(30):
        m, n, k = rng.int(1, 40), rng.int(1, 40), rng.int(1, 40)
        a = rng.u8_matrix(m, k)
        b = rng.i8_matrix(k, n)
        mult = rng.real(0.0001, 0.01)
        zp_a, zp_b, zp_c = rng.int(0, 255), rng.int(-128, 127), rng.int(0, 255)
        bias = rng.ints(-2000, 2000, n)
        relu = bool(t % 2)
        bp = ref.select_blocking(m, n, k, [(56, 32, 256, 14, 32), (8, 6, 4, 4, 3), (24, 16, 8, 6, 8)][t % 3])
        p = ref.prepack(b, bp)
        cases.append(dict(m=m, n=n, k=k, a=a, b=b, mult=mult, zp_a=zp_a, zp_b=zp_b, zp_c=zp_c, bias=bias,
                          relu=relu, acc=p.gemm_raw(a, threads=1 + t % 4),
                          out=p.gemm_requant(a, mult, zp_a, zp_b, zp_c, bias=bias, relu=relu, threads=1 + t % 3),
                          colsum=p.col_offsets(), max_abs=p.max_abs(), packed=p.data(), bp=np.array(bp)))
    flat = {}
    for i, cs in enumerate(cases):
        for key, v in cs.items():
            flat[f"{i}_{key}"] = np.asarray(v)
    np.savez_compressed(OUT / "ref_small.npz", count=len(cases), **flat)

    # 3. scalar requantize KATs incl. exact ties (quant.hpp:115-133)
    rng = orc.rng(77)
    rows = []
    for t in range(3000):
        if t < 500:  # ties: mult = 0.5 / 0.25, odd adj
            mult = [0.5, 0.25, 0.125][t % 3]
            acc = rng.int(-600, 600)
            ro, co, zp_a, zp_b, k = 0, 0, 0, 0, 1
        else:
            mult = rng.real(1e-5, 0.05)
            acc, ro, co = rng.int(-2_000_000, 2_000_000), rng.int(0, 255 * 4096), rng.int(-128 * 4096, 127 * 4096)
            zp_a, zp_b, k = rng.int(0, 255), rng.int(-128, 127), rng.int(1, 4096)
        zp_c, bias = rng.int(0, 255), rng.int(-1000, 1000)
        q = ref.requantize_scalar(acc, ro, co, mult, zp_a, zp_b, zp_c, k, np.array([bias], np.int32), 0)
        adj = ref.requantize_adjust(acc, ro, co, zp_a, zp_b, k, bias)
        rows.append((acc, ro, co, mult, zp_a, zp_b, zp_c, k, bias, q, adj))
    arr = np.array(rows, dtype=np.float64)
    np.savez_compressed(OUT / "ref_requant_kat.npz", rows=arr)

    # 4. pipeline validation messages (pipeline.hpp:66-102)
    kinds = {"raw": [3], "requant": [2], "relu_requant": [1, 2], "bias_requant": [0, 2], "empty": [],
             "relu_raw": [1, 3], "writer_first": [3, 2], "no_writer": [0], "relu_not_last": [1, 0, 2]}
    msgs = {name: (ref.pipeline_validate(k) or "") for name, k in kinds.items()}
    np.savez_compressed(OUT / "ref_pipeline_msgs.npz", **{k: np.array(v) for k, v in msgs.items()})
    print("golden fixtures written to", OUT)


def main_sparse():
    """5. outlier split + SpMDMAdd + BiasAdd with each writer (sparse.hpp:33-80,
    pipeline.hpp:157-207): the reference splits B, then runs execute_gemm on
    the dense part with [SpMDMAdd, BiasAdd] and WriteRawI32 / [ReluQuantized]
    Requantize (col_offsets of the original B) / WriteDequantF32."""
    build()
    orc, ref = Oracle(), RefLib()
    rng = orc.rng(4242)
    flat, count = {}, 0
    for t in range(12):
        m, n, k = rng.int(1, 100), rng.int(1, 64), rng.int(1, 200)
        a, b = rng.u8_matrix(m, k), rng.i8_matrix(k, n)
        threshold = [16, 48, 100, 128][t % 4]
        dense, cp, ri, vals = ref.split_outliers(b, threshold)
        pk = ref.prepack(dense, ref.select_blocking(m, n, k))
        bias_add = rng.ints(-5000, 5000, n) if t % 3 else None
        mult, zp_a, zp_b, zp_c = rng.real(0.0001, 0.005), rng.int(0, 255), rng.int(-20, 20), rng.int(0, 255)
        rq_bias = rng.ints(-1000, 1000, n)
        relu = bool(t % 2)
        dq_scale, dq_zp = rng.real(0.0001, 0.1), rng.int(-500, 500)
        sp = (cp, ri, vals)
        case = dict(m=m, n=n, k=k, a=a, b=b, threshold=threshold, col_ptr=cp, row_idx=ri, values=vals,
                    mult=mult, zp_a=zp_a, zp_b=zp_b, zp_c=zp_c, rq_bias=rq_bias, relu=relu, dq_scale=dq_scale,
                    dq_zp=dq_zp, col_offsets=orc.col_offsets(b),
                    raw=pk.gemm_pipeline(a, "raw", sparse=sp, bias_add=bias_add, threads=1 + t % 3),
                    requant=pk.gemm_pipeline(a, "requant", sparse=sp, bias_add=bias_add, mult=mult, zp_a=zp_a,
                                             zp_b=zp_b, zp_c=zp_c, rq_bias=rq_bias, relu=relu,
                                             col_offsets=orc.col_offsets(b), threads=1 + t % 2),
                    dequant=pk.gemm_pipeline(a, "dequant", sparse=sp, bias_add=bias_add, dq_scale=dq_scale,
                                             dq_zero_point=dq_zp, threads=2),
                    dequant_dense=pk.gemm_pipeline(a, "dequant", dq_scale=dq_scale, dq_zero_point=dq_zp))
        if bias_add is not None:
            case["bias_add"] = bias_add
        for key, v in case.items():
            flat[f"{t}_{key}"] = np.asarray(v)
        count += 1
    np.savez_compressed(OUT / "ref_sparse.npz", count=count, **flat)
    print("sparse / dequant fixtures written to", OUT)


if __name__ == "__main__":
    if "--only-sparse" in sys.argv:
        main_sparse()
    else:
        main()
        main_sparse()
