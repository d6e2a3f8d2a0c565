"""Per-tile timeline of CTA 0 (leader of pair 0) in the CTA-pair GEMM kernel
(gemm_tc2.cu; debug, Q8G_TC_TRACE=1), C2 shape: first / last MMA issue and
epilogue start / done per tile, us from the kernel's first stamp.  Shows the
tensor pipe's idle gaps between tiles and whether a tile's MMAs stretch while
the previous tile's epilogue runs."""
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
    m, n, k = 16384, 4096, 4096
    b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device="cuda")
    a = torch.randint(0, 256, (m, k), dtype=torch.uint8, device="cuda")
    pw = q8.prepack_weights(b)
    zpb = 0 if "--zpb0" in sys.argv else 3  # zp_b = 0: no row sums (RS warps idle)
    rp = q8.RequantParams(zp_a=128, zp_c=5, k_total=k, zp_b_per_channel=np.full(n, zpb, np.int32),
                          multiplier_f32_per_channel=np.full(n, 1e-4, np.float32), rounding=q8.ROUND_F32_RNE)
    pipe = q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(rp)])
    c = torch.empty((m, n), dtype=torch.uint8, device="cuda")
    if "--raw" in sys.argv:
        pipe = q8.OutputPipeline([q8.WriteRawI32()])
        c = torch.empty((m, n), dtype=torch.int32, device="cuda")
    for _ in range(3):
        q8.execute_gemm(a, pw, c, pipe)
    torch.cuda.synchronize()
    buf = (C.c_uint64 * (8 * 1024 + 2048))()
    _lib.load().q8g_debug_tc_trace(buf, 2048)
    w = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
    tiles = w[9216:9216 + 128].reshape(32, 4)
    tiles = tiles[tiles[:, 0] > 0]
    t0 = w[0]
    print("tile  mma_first  mma_last  epi_start  epi_done   (us)   mma span  gap before")
    prev = None
    for i, r in enumerate(tiles):
        span = (r[1] - r[0]) / 1e3
        gap = (r[0] - prev) / 1e3 if prev is not None else 0.0
        print(f"{i:4d} " + " ".join(f"{(x - t0) / 1e3:9.2f}" for x in r) + f"   {span:8.2f}  {gap:8.2f}")
        prev = r[1]


if __name__ == "__main__":
    main()
