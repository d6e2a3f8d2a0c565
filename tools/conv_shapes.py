"""Per-launch timing of conv3x3 shapes outside C3 (ResNet-style 256 / 512
channels): the im2col + tensor-core GEMM path vs the CUDA-core kernel
(Q8G_CONV_SIMT=1).  Graph-captured back-to-back launches, one event pair."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2101_05615_b200 as q8  # noqa: E402


def run(nb, h, w, c, oc, reps=20):
    rng = np.random.default_rng(0)
    wt = rng.integers(-128, 128, (3, 3, c, oc)).astype(np.int8)
    pw = q8.prepack_conv3x3_weights(wt)
    rp = q8.RequantParams(zp_a=128, zp_c=5, k_total=9 * c, bias=rng.integers(-1000, 1001, oc).astype(np.int32),
                          zp_b_per_channel=rng.integers(-10, 11, oc).astype(np.int32),
                          multiplier_f32_per_channel=np.full(oc, 1e-4, np.float32), rounding=q8.ROUND_F32_RNE)
    pipe = q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(rp)])
    x = torch.randint(0, 256, (nb, h, w, c), dtype=torch.uint8, device="cuda")
    y = torch.empty((nb, h, w, oc), dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            q8.execute_conv3x3(x, pw, y, pipe)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                q8.execute_conv3x3(x, pw, y, pipe)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g.replay()
        torch.cuda.synchronize()
        a.record(st)
        g.replay()
        b.record(st)
        torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps
    ops = 2.0 * nb * h * w * oc * 9 * c
    path = "simt" if os.environ.get("Q8G_CONV_SIMT") else "auto"
    print(f"{path:4s} conv3x3 {nb}x{h}x{w}x{c}->{oc}: {us:9.1f} us  {ops / us / 1e6:8.1f} TOPS", flush=True)


if __name__ == "__main__":
    for s in [(32, 56, 56, 64, 64), (32, 28, 28, 128, 128), (32, 28, 28, 256, 256), (32, 14, 14, 256, 256),
              (32, 7, 7, 512, 512), (32, 56, 56, 3, 64)]:
        run(*s)
