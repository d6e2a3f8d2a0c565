"""The command-line harness (paper_2101_05615_b200/cli/q8gemm_cli.cpp): the
reference CLI's subcommands, flags, output lines, CSV header and exit codes
(proj/tools/q8gemm_cli.cpp, SPEC.md "[MODULE] cli": 0 success, 1 verification
failure, 2 invalid input / config).

CPU: argument and shapes-file errors (all raised before any GPU work).
GPU: verify (both variants, worker threads, the i16 refusal without the
split), bench CSV, demo, and byte-identical reruns for a fixed seed.
"""
import subprocess

import pytest

from paper_2101_05615_b200 import build as b


@pytest.fixture(scope="module")
def cli():
    return str(b.build_cli())


def run(cli, *args, timeout=300):
    r = subprocess.run([cli, *args], capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout, r.stderr


def test_help_and_missing_subcommand(cli):
    rc, out, _ = run(cli, "--help")
    assert rc == 0 and "verify" in out and "bench" in out and "demo" in out
    rc, _, err = run(cli)
    assert rc == 2 and "subcommand is required" in err
    rc, _, err = run(cli, "frobnicate")
    assert rc == 2 and "unknown subcommand" in err
    assert run(cli, "bench", "--help")[0] == 0


@pytest.mark.parametrize("args,msg", [
    (["verify", "--variant", "i8"], "not in {i32,i16}"),
    (["verify", "--threads", "0"], "not a positive number"),
    (["bench", "--repeats", "-3"], "not a positive number"),
    (["verify", "--seed", "x"], "not an unsigned integer"),
    (["demo", "--density", "1.5"], "not in range"),
    (["demo", "--shapes", "f"], "not expected"),        # --shapes is verify/bench only
    (["verify", "--repeats", "3"], "not expected"),     # --repeats is bench only
    (["verify", "--compare-naive"], "not expected"),
    (["bench", "--no-split"], "not expected"),
    (["verify", "--threads"], "requires an argument"),
    (["verify", "--mcb", "0"], "BlockingParams"),        # engine validation -> 2
    (["verify", "--mr", "8", "--mcb", "12"], "BlockingParams"),
])
def test_invalid_arguments_exit_2(cli, args, msg):
    rc, _, err = run(cli, *args)
    assert rc == 2, err
    assert msg in err


def test_shapes_file_errors(cli, tmp_path):
    bad = tmp_path / "bad.txt"
    bad.write_text("# comment\n1 2 3\n\n4 5\n")
    rc, _, err = run(cli, "verify", "--shapes", str(bad))
    assert rc == 2 and f"{bad}:4: expected \"M N K\" with positive integers" in err
    bad.write_text("1 2 3 4\n")
    assert run(cli, "verify", "--shapes", str(bad))[0] == 2
    bad.write_text("0 2 3\n")
    assert run(cli, "bench", "--shapes", str(bad))[0] == 2
    bad.write_text("# only comments\n\n")
    rc, _, err = run(cli, "verify", "--shapes", str(bad))
    assert rc == 2 and "no shapes found" in err
    rc, _, err = run(cli, "verify", "--shapes", str(tmp_path / "missing.txt"))
    assert rc == 2 and "cannot open shapes file" in err


# ------------------------------------------------------------------ GPU


@pytest.mark.gpu
@pytest.mark.parametrize("variant,threads", [("i32", 1), ("i32", 3), ("i16", 1), ("i16", 4)])
def test_verify_default_shapes(cuda, cli, variant, threads):
    rc, out, err = run(cli, "verify", "--variant", variant, "--threads", str(threads))
    lines = out.strip().splitlines()
    assert rc == 0, out + err
    assert len(lines) == 9 and all(ln.endswith("PASS max_dev=0") for ln in lines)
    assert lines[0] == f"M=1 N=1 K=1 variant={variant} threads={threads} : PASS max_dev=0"


@pytest.mark.gpu
def test_verify_i16_without_split_is_refused(cuda, cli, tmp_path):
    shapes = tmp_path / "s.txt"
    shapes.write_text("64 64 256\n")
    rc, _, err = run(cli, "verify", "--variant", "i16", "--no-split", "--shapes", str(shapes))
    assert rc == 2 and "INT16 accumulation rejected" in err
    # the split variant at a small kcb (threshold 1 + 32767 / (255 * 2) = 65) is exact
    rc, out, err = run(cli, "verify", "--variant", "i16", "--kcb", "2", "--shapes", str(shapes))
    assert rc == 0 and out.strip().endswith("PASS max_dev=0"), out + err


@pytest.mark.gpu
def test_verify_custom_shapes_and_determinism(cuda, cli, tmp_path):
    shapes = tmp_path / "s.txt"
    shapes.write_text("# acceptance shapes\n1 1 1\n4 5 6\n1 16 16\n16 16 16\n33 7 129\n\n56 32 64\n300 200 640\n")
    a = run(cli, "verify", "--shapes", str(shapes), "--seed", "99")
    b_ = run(cli, "verify", "--shapes", str(shapes), "--seed", "99")
    assert a[0] == 0 and a[1] == b_[1] and a[1].count("PASS") == 7
    assert run(cli, "verify", "--shapes", str(shapes), "--seed", "99", "--threads", "4")[0] == 0


@pytest.mark.gpu
def test_bench_csv(cuda, cli, tmp_path):
    shapes = tmp_path / "s.txt"
    shapes.write_text("128 4096 4096\n64 800 320\n")
    rc, out, err = run(cli, "bench", "--shapes", str(shapes), "--repeats", "5", "--compare-naive")
    assert rc == 0, err
    lines = out.strip().splitlines()
    assert lines[0] == "M,N,K,variant,threads,ns_median,gops"
    rows = [ln.split(",") for ln in lines[1:]]
    assert [r[:5] for r in rows] == [["128", "4096", "4096", "i32", "1"], ["128", "4096", "4096", "naive", "1"],
                                     ["64", "800", "320", "i32", "1"], ["64", "800", "320", "naive", "1"]]
    for r in rows:
        ns, gops = int(r[5]), float(r[6])
        m, n, k = map(int, r[:3])
        assert ns > 0 and abs(gops - 2 * m * n * k / ns) <= 1e-4 * max(1.0, gops)
    assert float(rows[0][6]) > 10 * float(rows[1][6])  # the GPU call beats the naive loop by far
    rc, out, _ = run(cli, "bench", "--variant", "i16", "--threads", "2", "--repeats", "3")
    assert rc == 0 and len(out.strip().splitlines()) == 10


@pytest.mark.gpu
def test_demo(cuda, cli):
    args = ["demo", "--m", "32", "--n", "24", "--k", "48", "--density", "0.02", "--seed", "7"]
    rc, out, err = run(cli, *args)
    assert rc == 0, out + err
    assert "engine vs integer reference: max_dev=0 (exact expected)" in out
    assert out.strip().endswith("PASS")
    assert "split: T=5" in out and "blocking: mcb=" in out
    assert run(cli, *args)[1] == out
    rc, out, _ = run(cli, "demo", "--m", "200", "--n", "300", "--k", "512", "--threads", "3")
    assert rc == 0 and out.strip().endswith("PASS")
