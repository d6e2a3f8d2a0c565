"""The C++ drop-in API (include/q8gemm_b200/q8gemm.hpp) through the reference
acceptance criteria (tests/cpp/acceptance_b200.cpp)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BIN = ROOT / "tests" / "cpp" / "acceptance_b200"


@pytest.fixture(scope="module")
def runner():
    import __graft_entry__ as g

    g.build_cpp_tests()
    assert BIN.exists()
    return BIN


def test_cpp_host_logic(runner):
    r = subprocess.run([str(runner), "host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all gating criteria passed" in r.stdout


@pytest.mark.gpu
def test_cpp_acceptance_on_gpu(runner, cuda):
    from paper_2101_05615_b200 import build as b

    cli = b.build_cli()
    r = subprocess.run([str(runner), "gpu", str(cli)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") == 10  # 0 host + 1, 2, 3 (outliers), 5, 6, 7, 8, 8 (CLI leg), 9 (N-sharded)
