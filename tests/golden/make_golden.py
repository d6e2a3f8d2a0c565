"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED
reference (oracle/_ref/libq8ref.so, built by oracle/Makefile from
/root/reference/proj/include).  Run here, where the reference exists:

    python tests/golden/make_golden.py

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


if __name__ == "__main__":
    main()
