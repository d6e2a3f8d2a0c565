"""Per-launch timing of the conv3x3 (C3) and depthwise-3x3 (C4) paths.

  python tools/conv_sweep.py [--which c3|c4|both]

Graph-captured launches with event pairs, rotating input/output sets whose
footprint exceeds the L2, BASELINE shapes and value distributions
(synthetic).  Prints us/launch, int8 TOPS and algorithmic GB/s.
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2101_05615_b200 as q8  # noqa: E402


def time_graph(launches, reps=5):
    stream = torch.cuda.current_stream()
    for f in launches:
        f()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
          for _ in launches]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for (a, b), f in zip(ev, launches):
            a.record(stream)
            f()
            b.record(stream)
    ts = []
    for _ in range(reps):
        g.replay()
        torch.cuda.synchronize()
        ts += [a.elapsed_time(b) * 1e3 for a, b in ev]
    return float(np.median(ts))


def time_graph_batched(launches, reps=5, rounds=8):
    """One event pair around rounds x len(launches) back-to-back launches in
    one graph: per-launch time including the inter-kernel gap but without
    per-launch event records."""
    stream = torch.cuda.current_stream()
    for f in launches:
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(rounds):
            for f in launches:
                f()
    ts = []
    for _ in range(reps):
        a.record(stream)
        g.replay()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / (rounds * len(launches)))
    return float(np.median(ts))


BATCHED = False


def timed(launches):
    return time_graph_batched(launches) if BATCHED else time_graph(launches)


def c3(nsets=4):
    nb, h, w, c, oc = 32, 56, 56, 64, 64
    rng = np.random.default_rng(0)
    wt = rng.integers(-128, 128, (3, 3, c, oc)).astype(np.int8)
    pw = q8.prepack_conv3x3_weights(wt)
    rp = q8.RequantParams(zp_a=128, zp_c=5, k_total=9 * c, bias=rng.integers(-1000, 1001, oc).astype(np.int32),
                          zp_b_per_channel=rng.integers(-10, 11, oc).astype(np.int32),
                          multiplier_f32_per_channel=(0.02 * rng.uniform(0.005, 0.02, oc) / 0.8).astype(np.float32),
                          rounding=q8.ROUND_F32_RNE)
    pipe = q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(rp)])
    xs = [torch.randint(0, 256, (nb, h, w, c), dtype=torch.uint8, device="cuda") for _ in range(nsets)]
    ys = [torch.empty((nb, h, w, oc), dtype=torch.uint8, device="cuda") for _ in range(nsets)]
    us = timed([lambda i=i: q8.execute_conv3x3(xs[i], pw, ys[i], pipe) for i in range(nsets)])
    ops = 2.0 * nb * h * w * oc * 9 * c
    byts = 2 * nb * h * w * c + 9 * c * oc + 16 * oc
    print(f"C3 conv3x3 32x56x56x64->64: {us:9.2f} us  {ops / us / 1e6:8.1f} TOPS  {byts / us / 1e3:8.1f} GB/s "
          f"stats={q8.launch_stats()}", flush=True)


def c4(nsets=3):
    nb, h, w, c = 32, 112, 112, 256
    rng = np.random.default_rng(1)
    wt = rng.integers(-128, 128, (3, 3, c)).astype(np.int8)
    rp = q8.RequantParams(zp_a=128, zp_c=5, k_total=9, bias=rng.integers(-1000, 1001, c).astype(np.int32),
                          zp_b_per_channel=rng.integers(-10, 11, c).astype(np.int32),
                          multiplier_f32_per_channel=(0.02 * rng.uniform(0.005, 0.02, c) / 0.1).astype(np.float32),
                          rounding=q8.ROUND_F32_RNE)
    f = q8.DepthwiseFilter(wt, rp, relu=True)
    xs = [torch.randint(0, 256, (nb, h, w, c), dtype=torch.uint8, device="cuda") for _ in range(nsets)]
    ys = [torch.empty((nb, h, w, c), dtype=torch.uint8, device="cuda") for _ in range(nsets)]
    us = timed([lambda i=i: q8.execute_dwconv3x3(xs[i], f, ys[i]) for i in range(nsets)])
    ops = 2.0 * 9 * nb * h * w * c
    byts = 2 * nb * h * w * c + 9 * c + 16 * c
    print(f"C4 dwconv3x3 32x112x112x256: {us:9.2f} us  {ops / us / 1e6:8.1f} TOPS  {byts / us / 1e3:8.1f} GB/s "
          f"stats={q8.launch_stats()}", flush=True)


if __name__ == "__main__":
    torch.cuda.set_stream(torch.cuda.Stream())
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="both")
    ap.add_argument("--batched", action="store_true", help="one event pair around many back-to-back launches")
    a = ap.parse_args()
    BATCHED = a.batched
    if a.which in ("c3", "both"):
        c3()
    if a.which in ("c4", "both"):
        c4()
