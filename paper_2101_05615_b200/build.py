"""In-tree build of the CUDA library (libq8g_b200.so) for sm_100a.

Compiles every csrc/*.cu with nvcc (-gencode arch=compute_100a,code=sm_100a,
-lineinfo, no fast-math) in parallel and links one shared library next to
this file, so it travels to the GPU box with the repo snapshot.  Objects are
rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
# Variants, each from its own object directory and linked to the same
# libq8g_b200.so name so the package and the tests load them unchanged:
#   Q8G_CHECKED=1  device-side bounds / layout assertions (Q8G_CHECK, ptx.cuh);
#   Q8G_TRACE=1    the phase-trace stamps the tools/*_trace.py probes read.
#                  The production build compiles them out: even disabled at
#                  run time their branches cost C4 ~9 %.
CHECKED = os.environ.get("Q8G_CHECKED") == "1"
TRACE = os.environ.get("Q8G_TRACE") == "1"
BUILD = PKG / ("_build" + ("_checked" if CHECKED else "") + ("_trace" if TRACE else ""))
LIB = PKG / "libq8g_b200.so"
ROOT = PKG.parent

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "-Xptxas", "-warn-spills",
    f"-I{ROOT / 'include'}",
] + (["-DQ8G_CHECKED=1"] if CHECKED else []) + (["-DQ8G_TRACE=1"] if TRACE else [])


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _headers_mtime():
    hs = list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: Path, verbose: bool) -> Path:
    obj = BUILD / (src.stem + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, _headers_mtime()):
        return obj
    cmd = [NVCC, *ARCH, *NVFLAGS, "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and verbose:
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False, jobs: int | None = None) -> Path:
    BUILD.mkdir(exist_ok=True)
    srcs = _sources()
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    stamp = BUILD / "linked"  # which object set the current library was linked from
    if LIB.exists() and LIB.stat().st_mtime >= newest and stamp.exists() and \
            stamp.read_text() == str(LIB.stat().st_mtime_ns):
        return LIB
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs),
           "-lcuda" if False else "-ldl"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    for d in set(PKG.glob("_build*")) - {BUILD}:  # the other object sets are stale now
        (d / "linked").unlink(missing_ok=True)
    stamp.write_text(str(LIB.stat().st_mtime_ns))
    return LIB


CLI_SRC = PKG / "cli" / "q8gemm_cli.cpp"
CLI = PKG / "q8gemm_b200_cli"


def build_cli(verbose: bool = False) -> Path:
    """The reference command-line harness (verify / bench / demo) on the C++
    drop-in API, linked against the in-tree library."""
    deps = [CLI_SRC, LIB, ROOT / "include" / "q8gemm_b200" / "q8gemm.hpp", ROOT / "include" / "q8g_b200.h"]
    if CLI.exists() and CLI.stat().st_mtime >= max(d.stat().st_mtime for d in deps):
        return CLI
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", f"-I{ROOT / 'include'}", str(CLI_SRC), "-o", str(CLI),
           f"-L{PKG}", "-lq8g_b200", "-Wl,-rpath,$ORIGIN", "-pthread"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"CLI build failed:\n{r.stderr}")
    return CLI


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
    print(build_cli(verbose="-v" in sys.argv))
