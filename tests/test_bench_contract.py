"""bench.py's reference arm (CPU, no GPU needed): one JSON line with the
driver's contract keys for the GEMM headline and the conv / depthwise
workloads, and silent non-zero ranks under torchrun."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def run_bench(*args, env_extra=None, timeout=300):
    env = dict(os.environ)
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True, cwd=ROOT,
                       env=env, timeout=timeout)
    return r.returncode, r.stdout, r.stderr


@pytest.mark.parametrize("cfg", ["C2", "C1", "C3", "C4"])
def test_reference_arm_line(cfg):
    if not (ROOT / "oracle" / "_ref").exists() and cfg != "C4":
        pytest.skip("oracle/_ref not built")
    rc, out, err = run_bench("--impl", "reference", "--config", cfg, "--steps", "1", "--warmup", "3")
    assert rc == 0, err
    lines = [ln for ln in out.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "TOPS" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] == d["cpu_baseline"]["value"]
    assert d["cpu_baseline"]["kind"] == ("port" if cfg == "C4" else "reference")
    assert d["cpu_baseline"]["cores"] >= 1
    # the same workload identity as our arm's line (the driver compares them)
    sys.path.insert(0, str(ROOT))
    import bench
    assert d["config"] == bench.config_dict(cfg, 1)
    assert d["ms_per_step"] > 0


def test_default_config_is_the_c2_headline():
    sys.path.insert(0, str(ROOT))
    import bench
    assert bench.HEADLINE == "C2" and bench.BOUND["C2"] == "tensor"
    assert bench.config_dict("C2", 8)["M"] == 16384


def test_reference_arm_other_ranks_silent():
    rc, out, _ = run_bench("--impl", "reference", "--config", "C1", "--steps", "1", "--gpus", "2",
                           env_extra={"RANK": "1", "WORLD_SIZE": "2"})
    assert rc == 0 and out.strip() == ""


REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches")


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["C2", "C1", "C3", "C4"])
def test_our_arm_line_on_the_gpu(cfg):
    """bench.py's own arm on a B200: one JSON line with every contract key, the
    device value and an end-to-end value through the host-view ABI, our
    kernels counted in the timed region, and the same config dict the
    reference arm prints."""
    rc, out, err = run_bench("--config", cfg, "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-sub",
                             timeout=600)
    assert rc == 0, err
    lines = [ln for ln in out.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in REQUIRED:
        assert key in d, key
    assert d["unit"] == "TOPS" and d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3
    assert d["gpu_launches"] == 3  # one launch of our kernel per step
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] == ("tensor" if cfg == "C2" else "hbm") and 0 < r["frac"] < 1 and r["peak"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    sys.path.insert(0, str(ROOT))
    import bench
    assert d["config"] == bench.config_dict(cfg, 1)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["C2", "C3", "C4"])
def test_multirank_bench_path_on_one_gpu(cfg):
    """The N > 1 code path of bench.py (torchrun, 2 ranks, strong scaling:
    C2 row stripes, C3 / C4 image ranges, max-over-ranks timing) run with both
    ranks sharing cuda:0 over gloo (Q8G_BENCH_SHARED_GPU=1).  A smoke test of
    the launch, partition and reduction plumbing that the driver's scaling run
    uses -- the numbers of a shared GPU are not measurements."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, Q8G_BENCH_SHARED_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), "--gpus",
                        "2", "--config", cfg, "--steps", "2", "--warmup", "3", "--no-sub", "--no-cpu-baseline"],
                       capture_output=True, text=True, cwd=ROOT, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    sys.path.insert(0, str(ROOT))
    import bench
    assert d["n_gpus"] == 2 and d["config"] == bench.config_dict(cfg, 2) and d["scaling"] == "strong"
    assert d["value"] > 0 and d["gpu_launches"] == 2 and d["e2e"]["value"] > 0
    per_gpu = bench.int8_peaks()[0] if cfg == "C2" else bench.peaks()[0]
    assert d["roofline"]["peak"] == pytest.approx(2 * per_gpu)
