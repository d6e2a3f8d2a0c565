"""Per-unit timeline of CTA 0 in the tensor-core depthwise kernel (debug;
Q8G_TC_TRACE=1): halo TMA issued / landed / MMAs issued / epilogue start /
epilogue done, in us from the first stamp."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch

os.environ.setdefault("Q8G_TC_TRACE", "1")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2101_05615_b200 as q8  # noqa: E402
from paper_2101_05615_b200 import _lib  # noqa: E402


def main():
    nb, h, w, c = 32, 112, 112, 256
    rng = np.random.default_rng(1)
    wt = rng.integers(-128, 128, (3, 3, c)).astype(np.int8)
    rp = q8.RequantParams(zp_a=128, zp_c=5, k_total=9, bias=rng.integers(-1000, 1001, c).astype(np.int32),
                          zp_b_per_channel=rng.integers(-10, 11, c).astype(np.int32),
                          multiplier_f32_per_channel=np.full(c, 0.0025, np.float32), rounding=q8.ROUND_F32_RNE)
    f = q8.DepthwiseFilter(wt, rp, relu=True)
    x = torch.randint(0, 256, (nb, h, w, c), dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        q8.execute_dwconv3x3(x, f, y)
    torch.cuda.synchronize()
    buf = (C.c_uint64 * (8 * 1024 + 2048))()
    _lib.load().q8g_debug_tc_trace(buf, 2048)
    a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)[8192:8192 + 320].reshape(5, 64)
    n = int((a[0] > 0).sum())
    t0 = a[0, 0]
    print("unit  tma_issue  landed  mma_issued  epi_start  epi_done   (us)")
    for i in range(n):
        print(f"{i:4d} " + " ".join(f"{(a[j, i] - t0) / 1e3:9.2f}" for j in range(5)))


if __name__ == "__main__":
    main()
