"""Pins the oracle restatement (oracle/oracle.c) before anything is checked
against it: the reference unit-test known answers (proj/tests/test_*.cpp) and
the golden fixtures produced by the unmodified reference (tests/golden/,
made by tests/golden/make_golden.py from oracle/_ref).  CPU only."""
from pathlib import Path

import numpy as np
import pytest

import configs

GOLD = Path(__file__).resolve().parent / "golden"


def test_mt19937_64_published_kat(orc):
    # std::mt19937_64 default seed 5489: the 10000th output is 9981545732273789042
    r = orc.rng(5489)
    for _ in range(9999):
        r.next()
    assert r.next() == 9981545732273789042


def test_fixture_helpers_semantics(orc):
    # test_util.hpp:12-26: byte = rng() & 0xFF, int = lo + rng() % span
    r1, r2 = orc.rng(123), orc.rng(123)
    raw = [r1.next() for _ in range(6)]
    u = r2.u8_matrix(1, 2)
    assert list(u[0]) == [raw[0] & 0xFF, raw[1] & 0xFF]
    assert r2.int(-5, 5) == -5 + raw[2] % 11
    assert r2.real(1.0, 3.0) == 1.0 + 2.0 * ((raw[3] % 10001) / 10000.0)


def test_naive_gemm_kats(orc):
    # test_engine.cpp:29-38: 1x1x1 -> 6
    assert orc.naive_gemm_i32(np.array([[2]], np.uint8), np.array([[3]], np.int8))[0, 0] == 6
    # test_oracle.cpp:66-77 with unit scales: [[1,2],[3,4]] x [[5,-6],[7,8]]
    c = orc.naive_gemm_i32(np.array([[1, 2], [3, 4]], np.uint8), np.array([[5, -6], [7, 8]], np.int8))
    assert c.tolist() == [[19, 10], [43, 14]]


def test_col_offsets_kats(orc):
    # test_quant.cpp:92-117
    assert orc.col_offsets(np.array([[1, 2], [3, 4]], np.int8)).tolist() == [4, 6]
    assert orc.col_offsets(np.zeros((100, 3), np.int8)).tolist() == [0, 0, 0]
    r = orc.rng(13)
    b = r.i8_matrix(64, 64)
    assert (orc.col_offsets(b) == b.astype(np.int32).sum(0)).all()


def test_requant_fixed_points(orc):
    # test_quant.cpp:119-148 (REF mode, the reference's own arithmetic)
    L = orc.L
    assert L.orc_requant_scalar_ref(0, 0, 0, 1.0, 0, 0, 7, 4, 0) == 7
    assert L.orc_requant_scalar_ref(42, 123, -55, 1.0, 0, 0, 0, 4, 0) == 42
    assert L.orc_requant_scalar_ref(100000, 0, 0, 1.0, 0, 0, 0, 1, 0) == 255
    assert L.orc_requant_scalar_ref(-100000, 0, 0, 1.0, 0, 0, 0, 1, 0) == 0
    assert L.orc_requant_scalar_ref(10, 0, 0, 0.5, 0, 0, 0, 1, 10) == 10
    assert L.orc_requant_scalar_ref(10, 0, 0, 0.5, 0, 0, 0, 1, -6) == 2
    # the F32_RNE restatement agrees on these (no ties)
    assert L.orc_requant_scalar_f32(10, 0, 0, 0.5, 0, 0, 0, 1, 10) == 10
    assert L.orc_requant_scalar_f32(42, 123, -55, 1.0, 0, 0, 0, 4, 0) == 42


def test_rounding_modes_on_ties(orc):
    L = orc.L
    # 5 * 0.5 = 2.5: REF (half away) -> 3, RNE -> 2; -2.5 -> -3 / -2
    assert L.orc_requant_scalar_ref(5, 0, 0, 0.5, 0, 0, 100, 1, 0) == 103
    assert L.orc_requant_scalar_f32(5, 0, 0, 0.5, 0, 0, 100, 1, 0) == 102
    assert L.orc_requant_scalar_ref(-5, 0, 0, 0.5, 0, 0, 100, 1, 0) == 97
    assert L.orc_requant_scalar_f32(-5, 0, 0, 0.5, 0, 0, 100, 1, 0) == 98
    assert L.orc_round_half_away(0.49999999999999994) == 0
    assert L.orc_relu_quantized(3, 9) == 9 and L.orc_relu_quantized(12, 9) == 12


def test_offset_correction_identity(orc):
    # test_quant.cpp:153-179
    r = orc.rng(17)
    for _ in range(100):
        k = r.int(1, 8)
        zp_a, zp_b = r.int(0, 255), r.int(-128, 127)
        acc = ro = co = 0
        real = 0.0
        for _ in range(k):
            aq, bq = r.int(0, 255), r.int(-128, 127)
            acc += aq * bq
            ro += aq
            co += bq
            real += 0.5 * (aq - zp_a) * 0.25 * (bq - zp_b)
        assert 0.5 * 0.25 * orc.L.orc_requant_adjust(acc, ro, co, zp_a, zp_b, k, 0) == real


def test_ref_prepack_layout_kat(orc):
    # test_pack.cpp:97-111: K = kcb = 4, N = nr = 4, one block
    b = np.arange(1, 17, dtype=np.int8).reshape(4, 4)
    assert orc.prepack_ref(b, ncb=4, kcb=4, nr=4).tolist() == [1, 5, 2, 6, 3, 7, 4, 8, 9, 13, 10, 14, 11, 15, 12, 16]


def test_oracle_matches_reference_small_fixture(orc):
    g = np.load(GOLD / "ref_small.npz")
    for i in range(int(g["count"])):
        a, b = g[f"{i}_a"], g[f"{i}_b"]
        acc = orc.naive_gemm_i32(a, b)
        assert (acc == g[f"{i}_acc"]).all()
        cs = orc.col_offsets(b)
        assert (cs == g[f"{i}_colsum"]).all()
        assert int(np.abs(b.astype(np.int32)).max()) == int(g[f"{i}_max_abs"])
        rs = orc.row_offsets(a)
        out = orc.requant_matrix(acc, rs, cs, int(g[f"{i}_zp_a"]), int(g[f"{i}_zp_b"]), a.shape[1],
                                 g[f"{i}_bias"], 0, float(g[f"{i}_mult"]), int(g[f"{i}_zp_c"]),
                                 bool(g[f"{i}_relu"]), per_channel=False)
        assert (out == g[f"{i}_out"]).all(), f"case {i}"
        bp = g[f"{i}_bp"]
        assert (orc.prepack_ref(b, int(bp[1]), int(bp[2]), int(bp[4])) == g[f"{i}_packed"]).all()


def test_oracle_matches_reference_requant_kats(orc):
    rows = np.load(GOLD / "ref_requant_kat.npz")["rows"]
    L = orc.L
    for acc, ro, co, mult, zp_a, zp_b, zp_c, k, bias, q, adj in rows:
        args = (int(acc), int(ro), int(co))
        assert L.orc_requant_adjust(*args, int(zp_a), int(zp_b), int(k), int(bias)) == int(adj)
        assert L.orc_requant_scalar_ref(*args, float(mult), int(zp_a), int(zp_b), int(zp_c), int(k),
                                        int(bias)) == int(q)


def test_oracle_matches_reference_c0(orc):
    g = np.load(GOLD / "c0_reference.npz")
    c = configs.gemm_case(orc, "C0", *configs.CONFIG_SHAPES["C0"])
    import hashlib
    assert hashlib.sha256(c.a.tobytes()).hexdigest() == str(g["a_sha"])
    assert hashlib.sha256(c.b.tobytes()).hexdigest() == str(g["b_sha"])
    acc = orc.naive_gemm_i32(c.a, c.b)
    assert hashlib.sha256(acc.tobytes()).hexdigest() == str(g["acc_sha"])
    cs = orc.col_offsets(c.b)
    assert (cs == g["col_offsets"]).all()
    rs = orc.row_offsets(c.a)
    for relu, key in ((False, "out"), (True, "out_relu")):
        out = orc.requant_matrix(acc, rs, cs, c.zp_a, int(c.zp_b), 320, c.bias, 0, c.mult_f64, c.zp_c, relu,
                                 per_channel=False)
        assert (out == g[key]).all()
    # F32_RNE differs from REF only where the product sits on a .5 tie
    # (SURVEY probe: 2 of 51,200 at C0)
    f32 = orc.requant_matrix(acc, rs, cs, c.zp_a, int(c.zp_b), 320, c.bias, 1, np.float32(c.mult_f64), c.zp_c,
                             False, per_channel=False)
    diff = np.argwhere(f32 != g["out"])
    assert len(diff) <= 8


def test_oracle_matches_live_reference(orc, ref):
    """When oracle/_ref is built here, compare against it directly too."""
    r = orc.rng(99)
    for t in range(20):
        m, n, k = r.int(1, 96), r.int(1, 96), r.int(1, 200)
        a, b = r.u8_matrix(m, k), r.i8_matrix(k, n)
        pk = ref.prepack(b, ref.select_blocking(m, n, k))
        acc = pk.gemm_raw(a, threads=1 + t % 4)
        assert (orc.naive_gemm_i32(a, b) == acc).all()
        assert (ref.naive_gemm(a, b) == acc).all()
        mult = r.real(0.0001, 0.01)
        zp_a, zp_b, zp_c = r.int(0, 255), r.int(-128, 127), r.int(0, 255)
        bias = r.ints(-1000, 1000, n)
        out = pk.gemm_requant(a, mult, zp_a, zp_b, zp_c, bias=bias, relu=bool(t % 2), threads=2)
        mine = orc.requant_matrix(acc, orc.row_offsets(a), orc.col_offsets(b), zp_a, zp_b, k, bias, 0, mult, zp_c,
                                  bool(t % 2), per_channel=False)
        assert (mine == out).all()


def test_conv_oracle_im2col_semantics(orc):
    # App. A D2: padded taps read zp_a; k = (kh*3+kw)*C + c
    x = np.arange(2 * 3 * 3 * 2, dtype=np.uint8).reshape(2, 3, 3, 2)
    cols = orc.im2col3x3(x, 200)
    assert cols.shape == (18, 18)
    # pixel (0,0,0): taps (-1,-1),(-1,0),(-1,1),(0,-1) padded, (0,0) = x[0,0,0]
    assert cols[0, :8].tolist() == [200] * 8
    assert cols[0, 8:10].tolist() == x[0, 0, 0].tolist()
    assert cols[4, 8:10].tolist() == x[0, 1, 1].tolist()  # centre tap of the centre pixel


def test_dw_oracle_matches_conv_formulation(orc):
    # depthwise == per-channel conv with a diagonal filter (identity check)
    r = orc.rng(5)
    nb, h, w, c = 2, 5, 4, 3
    x = r.u8((nb, h, w, c))
    wt = r.i8((3, 3, c))
    zp_w = r.ints(-10, 10, c)
    mult = np.full(c, 0.01, np.float32)
    out, acc = orc.dwconv3x3(x, 17, wt, zp_w, None, mult, 5, False)
    full = np.zeros((3, 3, c, c), np.int8)
    for ch in range(c):
        full[:, :, ch, ch] = wt[:, :, ch]
    acc2 = orc.conv3x3_i32(x, 17, full)
    assert (acc.reshape(-1, c) == acc2).all()
