"""Benchmark of the B200 fused u8 x s8 -> s32 GEMM + requantization hot path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C0..C4] [--impl ours|reference]

One JSON line on rank 0.  The headline (default) is BASELINE configs[2],
"C2": the large-batch FC layer M=16384 N=4096 K=4096 with per-channel
zero points / scales, int32 bias and ReLU fused into the requantizing
epilogue -- the tensor-bound configuration north_star's ">= 70% of dense
INT8 tensor peak" target is quoted on.  A "step" is one pass of the hot path
over the whole batch: one fused GEMM + requant launch (B prepacked once;
packing not timed, BASELINE configs[1]).

Multi-GPU (torchrun, one process per GPU): strong scaling of the configs
BASELINE partitions.  C2: rank r computes the row stripe
stripe_rows(16384, r, N) -- the reference's own balanced partition of row
blocks over workers (engine.hpp:39-47, 102-103) -- with B replicated; C3 / C4:
rank r convolves its contiguous range of the 32 images.  No collective on the
data path; the only collective is the max-over-ranks timing reduction.
value = the configuration's total int8 ops per step / the max-over-ranks step
time; roofline peaks are N x the per-GPU peak.

value     : whole-job int8 TOPS (2*M*N*K per step / device time), inputs
            resident in HBM, the K steps replayed from one CUDA graph over
            rotating buffer sets whose footprint is > 2x the 126 MB L2.
e2e       : the same metric through the C-ABI host-buffer entry points
            (q8g_gemm_u8s8_requant_host, q8g_conv3x3_u8s8_nhwc_host,
            q8g_dwconv3x3_u8s8_nhwc_host), wall clock per synchronous call:
            pinned host inputs copied in and outputs copied out every step.
roofline  : the dominant kernel (the only one launched) -- algorithmic ops
            (tensor-bound C2) or bytes (HBM-bound C1, C3, C4) per launch over
            its average launch duration in the timed region, against the
            measured peaks (int8: profiles/int8_peak.json, HBM:
            MEASURED_PEAKS.json); traffic = ncu DRAM bytes of the same kernel
            (profiles/traffic.json) or null.
sub       : C1 (N=1 only: BASELINE does not partition it), C3 and C4 measured
            the same way, each with its own roofline (headline run only).
cpu_baseline / --impl reference : the reference's own CPU path
            (oracle/_ref: unmodified q8gemm execute_gemm on all host cores, +
            the restated per-channel fp32 requant) on a bounded row sample.
clocks    : NVML SM clock / throttle reasons polled every ~0.5 ms during the
            timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "int8 TOPS (fused GEMM+requant) and fraction of INT8 tensor peak / HBM BW"
HEADLINE = "C2"
GEMM_CONFIGS = {
    # name: (M total, N, K, alpha_C, description)
    "C0": (64, 800, 320, 0.5, "C0 single FC: M=64 N=800 K=320 (BASELINE configs[0])"),
    "C1": (128, 4096, 4096, 2.2, "C1 production FC: M=128 N=4096 K=4096, per-channel zp_b/alpha_B, int32 bias, "
                                 "ReLU, u8 out (BASELINE configs[1])"),
    "C2": (16384, 4096, 4096, 2.2, "C2 large-batch FC: M=16384 N=4096 K=4096, per-channel zp_b/alpha_B, int32 bias, "
                                   "ReLU, u8 out (BASELINE configs[2])"),
}
CONV_CONFIGS = {
    # name: (images, H, W, C, OC or 0 = depthwise, alpha_C, description)
    "C3": (32, 56, 56, 64, 64, 0.8, "C3 conv3x3 as implicit GEMM: NHWC 32x56x56x64 -> 64, pad 1 with zp_a, "
                                    "per-channel requant + ReLU (BASELINE configs[3])"),
    "C4": (32, 112, 112, 256, 0, 0.1, "C4 depthwise 3x3: NHWC 32x112x112x256, pad 1 with zp_a, per-channel "
                                      "requant + ReLU (BASELINE configs[4])"),
}
# roofline bound per config: C0 launch latency (reported
# against HBM), C1 HBM (intensity 240 < ridge), C2 tensor, C3 ~balanced
# (reported against HBM), C4 HBM
BOUND = {"C0": "hbm", "C1": "hbm", "C2": "tensor", "C3": "hbm", "C4": "hbm"}
L2_BYTES = 126e6


# ---------------------------------------------------------------- shared pieces

def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def int8_peaks():
    """Measured dense INT8 tensor peaks of this pool's B200 (tools/int8_peak.cu,
    profiles/int8_peak.json): burst (the denominator: a K-step graph of
    ~0.2 ms launches is a burst), sustained, and the burst with uniformly
    random operands when measured."""
    p = ROOT / "profiles" / "int8_peak.json"
    if p.exists():
        d = json.loads(p.read_text())
        return (float(d["int8_tops_burst"]), float(d["int8_tops_sustained"]),
                d.get("int8_tops_burst_random"), "measured (profiles/int8_peak.json, tools/int8_peak.cu)")
    return 4500.0, 4500.0, None, "fallback (B200 dense INT8 spec, SURVEY 8(d))"


def traffic_of(cfg):
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        return json.loads(tf.read_text()).get(cfg)
    return None


def image_range(nb, rank, world):
    """Contiguous balanced image range of rank (batch sharding, C3 / C4)."""
    return nb * rank // world, nb * (rank + 1) // world


def gemm_rows(m, rank, world):
    """Row stripe of rank: the reference partition of 128-row blocks
    (engine.hpp:40-47 via q8g_partition_stripes)."""
    from paper_2101_05615_b200 import api
    return api.stripe_rows(m, rank, world)


def gemm_ops(cfg):
    m, n, k = GEMM_CONFIGS[cfg][:3]
    return 2.0 * m * n * k


def gemm_bytes(m, n, k):
    # A + B + u8 out + 16-byte per-column epilogue record (c, zp_b, mult)
    return m * k + k * n + m * n + 16 * n


def conv_ops_bytes(cfg, nb):
    """Algorithmic int8 ops and bytes of one conv / depthwise launch over nb
    images (x + y + weights + per-channel tables)."""
    _, h, w, c, oc, _, _ = CONV_CONFIGS[cfg]
    if oc:
        return 2.0 * nb * h * w * oc * 9 * c, nb * h * w * (c + oc) + 9 * c * oc + 16 * oc
    return 2.0 * 9 * nb * h * w * c, 2 * nb * h * w * c + 9 * c + 16 * c


def config_dict(cfg, world):
    """The workload identity -- identical in both arms."""
    if cfg in GEMM_CONFIGS:
        m, n, k, _, desc = GEMM_CONFIGS[cfg]
        par = ("rows sharded over the GPUs (strong scaling, stripe_rows = engine.hpp:40-47), B replicated, "
               "no collective") if cfg == "C2" else "one GPU (BASELINE does not partition it); stripes of rank 0"
        return {"workload": desc, "M": m, "N": n, "K": k, "gpus": world, "parallelism": par}
    nb, h, w, c, oc, _, desc = CONV_CONFIGS[cfg]
    return {"workload": desc, "images": nb, "H": h, "W": w, "C": c, "OC": oc or c, "gpus": world,
            "parallelism": "images sharded over the GPUs (strong scaling), weights replicated, no collective"}


def max_over_ranks(vals, device, world):
    """Element-wise max of per-rank timings (the slowest rank sets the step)."""
    if world <= 1:
        return [float(v) for v in vals]
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "gloo":  # shared-GPU smoke mode (Q8G_BENCH_SHARED_GPU): host tensors
        device = "cpu"
    t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.cpu()]


def whole_job_tops(total_ops_per_step, ms_per_step):
    return total_ops_per_step / (ms_per_step * 1e-3) / 1e12


class ClockSampler:
    """SM clock, max clock and throttle reasons polled through NVML every
    ~0.5 ms while the timed region runs (nvidia-smi samples at >= 100 ms would
    miss a few-ms region); falls back to a single nvidia-smi query."""

    # nvmlClocksEventReason* bits
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.stop_flag = False
        self.thread = None
        self.nv = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:  # noqa: BLE001 - no NVML: report unavailable
            self.nv = None

    def _reasons(self):
        nv = self.nv
        try:
            return int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
        except Exception:  # noqa: BLE001 - older binding name
            return int(nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h))

    def _run(self):
        nv = self.nv
        while not self.stop_flag:
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)), self._reasons()))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.0005)

    def start(self):
        if self.nv is not None:
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()

    def stop(self):
        self.stop_flag = True
        if self.thread is not None:
            self.thread.join(timeout=2)
        if self.nv is None or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable or no sample"], "samples": 0}
        bits = 0
        for _, r in self.samples:
            bits |= r
        return {"sm_mhz": float(np.median([s for s, _ in self.samples])), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(v for k, v in self.REASONS.items() if bits & k), "samples": len(self.samples),
                "source": "NVML, polled every ~0.5 ms during the timed region"}


def idle_rank_barriers(world):
    """A rank with no rows / images still joins timed_graph's two barriers."""
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.barrier()


def graph_upload(graph, stream):
    """cuGraphUpload of a captured torch graph on `stream` (driver API; the
    executable graph is a driver object shared with torch's runtime)."""
    import ctypes
    cuda = ctypes.CDLL("libcuda.so.1")
    cuda.cuGraphUpload.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    rc = cuda.cuGraphUpload(ctypes.c_void_p(graph.raw_cuda_graph_exec()), ctypes.c_void_p(stream.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"cuGraphUpload failed: CUresult {rc}")


def timed_graph(run_step, steps, stream, dev, world, sampler_index):
    """Capture `steps` steps in one CUDA graph, with the start / end CUDA
    events recorded INSIDE the graph as its first and last nodes (on the
    launching stream), so the timed region is exactly the K steps -- not the
    host's graph-launch submission, which for a 20-step graph of ~10 us
    kernels would add ~4 us per step.  One replay, a barrier + synchronize on
    both sides, clocks sampled during it.  Returns (ms, clocks)."""
    import torch
    import torch.distributed as dist
    start = torch.cuda.Event(enable_timing=True, external=True)
    end = torch.cuda.Event(enable_timing=True, external=True)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        start.record(stream)
        for i in range(steps):
            run_step(i)
        end.record(stream)
    # upload the graph before the timed replay: the first launch of a fresh
    # executable graph uploads its nodes while it runs, ~3 us per node, which
    # short kernels (C1 / C3, ~7-9 us) cannot hide
    # and replay it once untimed (C2 163.7 vs 164.2 us, C3 9.43 vs 9.68 us)
    graph_upload(graph, stream)
    for _ in range(int(os.environ.get("BENCH_WARM_REPLAYS", "1"))):
        graph.replay()
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(sampler_index)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    graph.replay()
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()
    if world > 1:
        dist.barrier()
    return start.elapsed_time(end), clocks


# ---------------------------------------------------------------- reference arm

def cpu_reference_gemm(cfg, threads, budget_s=15.0, max_steps=20, rows=None, build=None):
    """The reference's CPU path on this host on a bounded row sample: unmodified
    q8gemm execute_gemm[WriteRawI32] (oracle/_ref) with `threads` caller-owned
    workers + the restated per-channel fp32 requant (the reference is
    per-tensor only).  TOPS of the sample.  build: None = the fastest build
    this host runs (-march=x86-64-v4 on AVX-512 hosts, BASELINE.md §3's
    -march=native), "release" = the reference's CMake Release flags."""
    from oracle.py import REF_RELEASE_SO, Oracle, RefLib, best_ref_so  # CPU baseline leg only
    m_all, n, k, alpha_c, _ = GEMM_CONFIGS[cfg]
    m = rows or min(m_all, 1024)
    so = REF_RELEASE_SO if build == "release" else best_ref_so()
    orc, ref = Oracle(), RefLib(so)
    r = orc.rng(42)
    a = r.u8_matrix(m, k)
    b = r.i8_matrix(k, n)
    bias = r.ints(-1000, 1000, n)
    zp_b = r.ints(-10, 10, n)
    mult = (0.02 * r.reals(0.005, 0.02, n) / alpha_c).astype(np.float32)
    pk = ref.prepack(b, ref.select_blocking(m, n, k))
    colsum = pk.col_offsets()

    def step():
        acc = pk.gemm_raw(a, threads=threads)
        return orc.requant_matrix(acc, orc.row_offsets(a), colsum, 128, zp_b, k, bias, 1, mult, 5, True,
                                  per_channel=True)

    step()
    times = []
    t_all = time.perf_counter()
    while not times or (time.perf_counter() - t_all < budget_s and len(times) < max_steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    sec = float(np.median(times))
    ops = 2.0 * m * n * k
    busy = max(1, min(threads, -(-m // 56)))
    return {"value": ops / sec / 1e12, "unit": "TOPS", "cores": threads, "kind": "reference",
            "sample": f"{m} of {cfg}'s {m_all} rows ({m}x{n}x{k}): reference execute_gemm[WriteRawI32] + restated "
                      f"per-channel F32_RNE requant, median of {len(times)}, {threads} std::threads "
                      f"({busy} row stripes busy); build {so.name}",
            "ms_per_sample": sec * 1e3}


def conv_inputs(cfg):
    """Weights and per-channel requant parameters (BASELINE distributions, App. A D4)."""
    _, h, w, c, oc, alpha_c, _ = CONV_CONFIGS[cfg]
    r = np.random.default_rng(11)
    nout = oc or c
    wt = r.integers(-128, 128, (3, 3, c, oc) if oc else (3, 3, c)).astype(np.int8)
    bias = r.integers(-1000, 1001, nout).astype(np.int32)
    zp_b = r.integers(-10, 11, nout).astype(np.int32)
    mult = (0.02 * r.uniform(0.005, 0.02, nout) / alpha_c).astype(np.float32)
    return wt, bias, zp_b, mult


def cpu_reference_conv(cfg, threads, budget_s=15.0, images=0):
    """C3: restated im2col + the reference execute_gemm (oracle/_ref) + restated
    per-channel requant; C4: the restated depthwise loop (no reference path),
    on a bounded sample of images of the workload."""
    from oracle.py import Oracle, RefLib, best_ref_so  # CPU baseline leg only
    _, h, w, c, oc, _, _ = CONV_CONFIGS[cfg]
    orc = Oracle()
    wt, bias, zp_b, mult = conv_inputs(cfg)
    nimg = images or (2 if oc else 1)
    x = np.random.default_rng(5).integers(0, 256, (nimg, h, w, c)).astype(np.uint8)
    if oc:
        ref = RefLib(best_ref_so())
        wk = wt.reshape(9 * c, oc)
        pk = ref.prepack(wk, ref.select_blocking(nimg * h * w, oc, 9 * c))
        colsum = pk.col_offsets()

        def step():
            cols = orc.im2col3x3(x, 128, threads=threads)
            acc = pk.gemm_raw(cols, threads=threads)
            return orc.requant_matrix(acc, orc.row_offsets(cols), colsum, 128, zp_b, 9 * c, bias, 1, mult, 5, True,
                                      per_channel=True)
        kind, what = "reference", "restated im2col + reference execute_gemm[WriteRawI32] + restated requant"
    else:
        def step():
            return orc.dwconv3x3(x, 128, wt, zp_b, bias, mult, 5, True, threads=threads)
        kind, what = "port", "restated depthwise loop (the reference has no depthwise path)"
    step()
    times = []
    t_all = time.perf_counter()
    while not times or (time.perf_counter() - t_all < budget_s and len(times) < 20):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    sec = float(np.median(times))
    ops, _ = conv_ops_bytes(cfg, nimg)
    return {"value": ops / sec / 1e12, "unit": "TOPS", "cores": threads, "kind": kind,
            "sample": f"{nimg} of the workload's {CONV_CONFIGS[cfg][0]} images, {what}, median of {len(times)}, "
                      f"{threads} threads",
            "ms_per_sample": sec * 1e3}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    budget = min(120.0, 5.0 + 2.0 * args.steps)
    if args.config in CONV_CONFIGS:
        res = cpu_reference_conv(args.config, threads, budget_s=budget)
    else:
        res = cpu_reference_gemm(args.config, threads, budget_s=budget, max_steps=max(1, args.steps))
    ops = gemm_ops(args.config) if args.config in GEMM_CONFIGS else \
        conv_ops_bytes(args.config, CONV_CONFIGS[args.config][0])[0]
    line = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": "TOPS", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ops / (res["value"] * 1e12) * 1e3,  # the whole workload at the sample's rate
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8xs8->s32",
            "data": "synthetic (seeded mt19937_64 / numpy RNG, BASELINE distributions)",
            "config": config_dict(args.config, args.gpus),
            "path": "CPU " + res["kind"] + " (oracle/_ref; the reference's own execute_gemm)",
            "cpu_baseline": {k2: res[k2] for k2 in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": res["value"], "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm

def bench_gemm(cfg, ctx, steps, warmup, want_e2e=True):
    """One GEMM configuration on this rank's row stripe."""
    import torch

    import paper_2101_05615_b200 as q8
    from paper_2101_05615_b200 import _lib
    dev, rank, world, stream, lib = ctx["dev"], ctx["rank"], ctx["world"], ctx["stream"], ctx["lib"]
    m_all, n, k, alpha_c, _ = GEMM_CONFIGS[cfg]
    if cfg != "C2" and world > 1:
        r0, r1 = (0, m_all) if rank == 0 else (0, 0)
    else:
        r0, r1 = gemm_rows(m_all, rank, world)
    m = r1 - r0
    # weights and epilogue parameters: the same seeded draws on every rank (B replicated)
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device=dev, generator=g)
    bias = np.random.default_rng(7).integers(-1000, 1001, n).astype(np.int32)
    zp_b = np.random.default_rng(8).integers(-10, 11, n).astype(np.int32)
    mult = (0.02 * np.random.default_rng(9).uniform(0.005, 0.02, n) / alpha_c).astype(np.float32)
    rp = q8.RequantParams(zp_a=128, zp_c=5, k_total=k, bias=bias, zp_b_per_channel=zp_b,
                          multiplier_f32_per_channel=mult, rounding=q8.ROUND_F32_RNE)
    pipe = q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(rp)])
    pw0 = q8.prepack_weights(b, device=dev.index)
    out = {"rows": [r0, r1]}
    if m == 0:  # an idle rank still takes part in the barriers / reductions
        idle_rank_barriers(world)
        out.update(ms=0.0, launches=0, e2e_ms=0.0, clocks=None, kern_ms_isolated=0.0, nsets=0)
        return out
    # rotating buffer sets > 2x L2; the weights rotate too where they dominate the bytes
    rotate_b = k * n > m * (k + n)
    set_bytes = m * (k + n) + (k * n if rotate_b else 0)
    nsets = max(2, min(64, int(np.ceil(2.2 * L2_BYTES / set_bytes))))
    pws = [pw0] + ([pw0.replicate(dev.index) for _ in range(nsets - 1)] if rotate_b else [pw0] * (nsets - 1))
    g.manual_seed(99 + rank)
    As = [torch.randint(0, 256, (m, k), dtype=torch.uint8, device=dev, generator=g) for _ in range(nsets)]
    Cs = [torch.empty((m, n), dtype=torch.uint8, device=dev) for _ in range(nsets)]
    eps = [pipe.epilogue(p) for p in pws]

    def launch(i):
        j = i % nsets
        _lib.check(lib.q8g_gemm_u8s8_requant(As[j].data_ptr(), m, k, k, pws[j].handle, eps[j], Cs[j].data_ptr(), n,
                                             0, m, None, stream.cuda_stream))

    with torch.cuda.stream(stream):
        for i in range(max(warmup, nsets)):
            launch(i)
    torch.cuda.synchronize(dev)
    c0 = _lib.launch_count()
    ms, clocks = timed_graph(launch, steps, stream, dev, world, dev.index)
    # the graph capture counted its launches once
    out.update(ms=ms, launches=_lib.launch_count() - c0, clocks=clocks, nsets=nsets, set_bytes=set_bytes)
    if cfg == "C2" and clocks is not None:
        # the SM clock the last timed launch actually ran at (CTA 0 clock64 /
        # globaltimer): NVML reports the clock target, not the power-limited clock
        import ctypes
        cyc, ns = ctypes.c_uint64(), ctypes.c_uint64()
        if lib.q8g_debug_kernel_clock(ctypes.byref(cyc), ctypes.byref(ns)) == 0 and ns.value > 0:
            clocks["sm_mhz_in_kernel"] = cyc.value / ns.value * 1e3
            clocks["sm_mhz_in_kernel_source"] = "clock64 / globaltimer of CTA 0 over the last timed launch"
    # a lone launch (per-launch event pairs; no overlap with a neighbour)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nsets)]
    iso = []
    for _ in range(2):
        for j in range(nsets):
            ev[j][0].record(stream)
            launch(j)
            ev[j][1].record(stream)
        torch.cuda.synchronize(dev)
        iso += [a.elapsed_time(bb) for a, bb in ev]
    out["kern_ms_isolated"] = float(np.median(iso))
    if want_e2e:
        a_host = torch.randint(0, 256, (m, k), dtype=torch.uint8, generator=torch.Generator().manual_seed(3))
        a_host = a_host.pin_memory()
        c_host = torch.empty((m, n), dtype=torch.uint8).pin_memory()

        def e2e_call(i):
            j = i % nsets
            _lib.check(lib.q8g_gemm_u8s8_requant_host(a_host.data_ptr(), m, k, k, pws[j].handle, eps[j],
                                                      c_host.data_ptr(), n, 0, m, stream.cuda_stream))

        for i in range(2):
            e2e_call(i)
        n_e2e = max(3, min(steps, 20))
        ts = []
        for i in range(n_e2e):
            t0 = time.perf_counter()
            e2e_call(i)
            ts.append(time.perf_counter() - t0)
        out["e2e_ms"] = float(np.median(ts)) * 1e3
        out["e2e_bytes"] = (m * k, m * n)
    return out


def bench_conv(cfg, ctx, steps, warmup, want_e2e=True):
    """C3 / C4 on this rank's image range."""
    import torch

    import paper_2101_05615_b200 as q8
    from paper_2101_05615_b200 import _lib
    dev, rank, world, stream, lib = ctx["dev"], ctx["rank"], ctx["world"], ctx["stream"], ctx["lib"]
    nb_all, h, w, c, oc, _, _ = CONV_CONFIGS[cfg]
    i0, i1 = image_range(nb_all, rank, world)
    nb = i1 - i0
    nout = oc or c
    wt, bias, zp_b, mult = conv_inputs(cfg)
    rp = q8.RequantParams(zp_a=128, zp_c=5, k_total=9 * c if oc else 9, bias=bias, zp_b_per_channel=zp_b,
                          multiplier_f32_per_channel=mult, rounding=q8.ROUND_F32_RNE)
    out = {"images": [i0, i1]}
    if nb == 0:
        idle_rank_barriers(world)
        out.update(ms=0.0, launches=0, e2e_ms=0.0, clocks=None, kern_ms_isolated=0.0, nsets=0)
        return out
    if oc:
        pw = q8.prepack_conv3x3_weights(wt, device=dev.index)
        pipe = q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(rp)])
        ep = pipe.epilogue(pw)

        def call(x, y):
            _lib.check(lib.q8g_conv3x3_u8s8_nhwc(x.data_ptr(), nb, h, w, c, pw.handle, ep, y.data_ptr(), 0, nb,
                                                 stream.cuda_stream))

        def call_host(x, y):
            _lib.check(lib.q8g_conv3x3_u8s8_nhwc_host(x.data_ptr(), nb, h, w, c, pw.handle, ep, y.data_ptr(), 0, nb,
                                                      stream.cuda_stream))
    else:
        filt = q8.DepthwiseFilter(wt, rp, relu=True, device=dev.index)

        def call(x, y):
            _lib.check(lib.q8g_dwconv3x3_u8s8_nhwc(x.data_ptr(), nb, h, w, c, filt._h, y.data_ptr(), 0, nb,
                                                   stream.cuda_stream))

        def call_host(x, y):
            _lib.check(lib.q8g_dwconv3x3_u8s8_nhwc_host(x.data_ptr(), nb, h, w, c, filt._h, y.data_ptr(), 0, nb,
                                                        stream.cuda_stream))
    set_bytes = nb * h * w * (c + nout)
    nsets = max(2, min(64, int(np.ceil(2.2 * L2_BYTES / set_bytes))))
    g = torch.Generator(device=dev)
    g.manual_seed(99 + rank)
    xs = [torch.randint(0, 256, (nb, h, w, c), dtype=torch.uint8, device=dev, generator=g) for _ in range(nsets)]
    ys = [torch.empty((nb, h, w, nout), dtype=torch.uint8, device=dev) for _ in range(nsets)]

    def launch(i):
        call(xs[i % nsets], ys[i % nsets])

    with torch.cuda.stream(stream):
        for i in range(max(warmup, nsets)):
            launch(i)
    torch.cuda.synchronize(dev)
    c0 = _lib.launch_count()
    ms, clocks = timed_graph(launch, steps, stream, dev, world, dev.index)
    out.update(ms=ms, launches=_lib.launch_count() - c0, clocks=clocks, nsets=nsets, set_bytes=set_bytes)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nsets)]
    iso = []
    for _ in range(2):
        for j in range(nsets):
            ev[j][0].record(stream)
            launch(j)
            ev[j][1].record(stream)
        torch.cuda.synchronize(dev)
        iso += [a.elapsed_time(bb) for a, bb in ev]
    out["kern_ms_isolated"] = float(np.median(iso))
    if want_e2e:
        x_host = torch.randint(0, 256, (nb, h, w, c), dtype=torch.uint8, generator=torch.Generator().manual_seed(4))
        x_host = x_host.pin_memory()
        y_host = torch.empty((nb, h, w, nout), dtype=torch.uint8).pin_memory()
        for _ in range(2):
            call_host(x_host, y_host)
        ts = []
        for _ in range(max(3, min(steps, 20))):
            t0 = time.perf_counter()
            call_host(x_host, y_host)
            ts.append(time.perf_counter() - t0)
        out["e2e_ms"] = float(np.median(ts)) * 1e3
        out["e2e_bytes"] = (nb * h * w * c, nb * h * w * nout)
    return out


def summarize(cfg, res_all, world, steps):
    """Rank-0 record of one configuration from the max-over-ranks timings."""
    ms, kern_iso, e2e_ms = res_all
    ms_step = ms / steps
    if cfg in GEMM_CONFIGS:
        m, n, k = GEMM_CONFIGS[cfg][:3]
        ops = gemm_ops(cfg)
        abytes = gemm_bytes(m, n, k)
    else:
        ops, abytes = conv_ops_bytes(cfg, CONV_CONFIGS[cfg][0])
    value = whole_job_tops(ops, ms_step)
    hbm, hsrc = peaks()
    if BOUND[cfg] == "tensor":
        burst, sust, rnd, isrc = int8_peaks()
        roof = {"bound": "tensor", "achieved": value, "peak": burst * world, "unit": "TFLOP/s",
                "unit_note": "dense int8 tera-ops/s (2*M*N*K per launch)", "frac": value / (burst * world),
                "peak_source": isrc + f", burst x {world} GPU(s)", "frac_of_sustained_peak": value / (sust * world),
                "hbm_achieved_gbs": abytes / (ms_step * 1e-3) / 1e9}
        if rnd:
            roof["frac_of_random_operand_peak"] = value / (float(rnd) * world)
    else:
        achieved = abytes / (ms_step * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm * world, "unit": "GB/s",
                "frac": achieved / (hbm * world), "peak_source": hsrc + f" x {world} GPU(s)"}
    roof.update(traffic=traffic_of(cfg), algorithmic_bytes_per_launch=abytes, algorithmic_ops_per_launch=ops,
                kernel_ms=ms_step, kernel_ms_isolated=kern_iso)
    return value, ms_step, roof


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2101_05615_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Q8G_BENCH_SHARED_GPU=1 (tests only, never a measurement): every rank on
    # cuda:0 with a gloo group, to exercise the N > 1 code path on a one-GPU box
    shared = world > 1 and os.environ.get("Q8G_BENCH_SHARED_GPU") == "1"
    gpu = 0 if (world == 1 or shared) else local
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(gpu)
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", gpu)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = {"dev": dev, "rank": rank, "world": world, "stream": stream, "lib": _lib.load()}

    def one(cfg, steps, warmup, e2e=True):
        fn = bench_gemm if cfg in GEMM_CONFIGS else bench_conv
        r = fn(cfg, ctx, steps, warmup, want_e2e=e2e)
        t = max_over_ranks([r["ms"], r["kern_ms_isolated"], r.get("e2e_ms", 0.0)], dev, world)
        launches = max_over_ranks([r["launches"]], dev, world)[0]
        return r, t, launches

    cfg = args.config
    r, t, launches = one(cfg, args.steps, args.warmup)
    subs = {}
    if not args.no_sub and cfg == HEADLINE:
        for sc in ("C1", "C3", "C4"):
            if sc == "C1" and world > 1:
                continue
            sr, st, sl = one(sc, 20, 5)
            subs[sc] = (sr, st, sl)
    if rank == 0:
        value, ms_step, roof = summarize(cfg, t, world, args.steps)
        e2e_ms = t[2]
        if cfg in GEMM_CONFIGS:
            m, n, k = GEMM_CONFIGS[cfg][:3]
            h2d, d2h = m * k, m * n
            e2e_path = "q8g_gemm_u8s8_requant_host (pinned host A and C; chunked, copies overlapped with the GEMM)"
        else:
            nb, h, w, c, oc = CONV_CONFIGS[cfg][:5]
            h2d, d2h = nb * h * w * c, nb * h * w * (oc or c)
            e2e_path = ("q8g_conv3x3_u8s8_nhwc_host" if CONV_CONFIGS[cfg][4] else "q8g_dwconv3x3_u8s8_nhwc_host") + \
                " (pinned host x and y; chunked, copies overlapped with the kernel)"
        ops = gemm_ops(cfg) if cfg in GEMM_CONFIGS else conv_ops_bytes(cfg, CONV_CONFIGS[cfg][0])[0]
        line = {
            "metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8xs8->s32",
            "data": "synthetic (seeded torch / numpy RNG, BASELINE distributions)",
            "config": config_dict(cfg, world),
            "timing": {"graph": "K steps captured in one CUDA graph, uploaded (cuGraphUpload) and replayed once untimed, then one replay timed with CUDA events recorded inside the graph",
                       "l2": f"{r.get('nsets', 0)} rotating buffer sets of {r.get('set_bytes', 0) / 1e6:.1f} MB "
                             f"per rank (> 2x the 126 MB L2)", "packing": "excluded (prepacked once)",
                       "rank0_rows_or_images": r.get("rows", r.get("images"))},
            "roofline": roof,
            "e2e": {"value": whole_job_tops(ops, e2e_ms), "unit": "TOPS", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "path": e2e_path,
                    "timing": "host wall clock per synchronous call, median, max over ranks"},
            "gpu_launches": int(round(launches)),
            "clocks": r["clocks"],
        }
        if subs:
            line["sub"] = {}
            for sc, (sr, st, sl) in subs.items():
                sv, sms, sroof = summarize(sc, st, world, 20)
                sops = gemm_ops(sc) if sc in GEMM_CONFIGS else conv_ops_bytes(sc, CONV_CONFIGS[sc][0])[0]
                line["sub"][sc] = {"value": sv, "unit": "TOPS", "ms_per_step": sms, "steps": 20, "warmup": 5,
                                   "config": config_dict(sc, world if sc != "C1" else 1), "roofline": sroof,
                                   "e2e": {"value": whole_job_tops(sops, st[2]), "unit": "TOPS",
                                           "ms_per_step": st[2]},
                                   "gpu_launches": int(round(sl)), "clocks": sr["clocks"]}
        if world == 1 and not args.no_cpu_baseline:
            try:
                cb = (cpu_reference_gemm(cfg, os.cpu_count() or 1) if cfg in GEMM_CONFIGS
                      else cpu_reference_conv(cfg, os.cpu_count() or 1))
                line["cpu_baseline"] = {k2: cb[k2] for k2 in ("value", "unit", "cores", "kind", "sample")}
                if cfg in GEMM_CONFIGS:  # the reference's own CMake Release flags, for comparison
                    rel = cpu_reference_gemm(cfg, os.cpu_count() or 1, budget_s=5.0, max_steps=5, build="release")
                    line["cpu_baseline"]["release_flags_value"] = rel["value"]
            except Exception as e:  # noqa: BLE001 - the baseline is reported, never the target
                line["cpu_baseline"] = {"value": None, "unit": "TOPS", "cores": 0, "kind": "reference",
                                        "sample": f"unavailable: {e}"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=HEADLINE, choices=sorted(GEMM_CONFIGS) + sorted(CONV_CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="headline only (no C1 / C3 / C4 sub-records)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
