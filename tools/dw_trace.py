"""Per-unit timeline of CTA 0 in the tensor-core depthwise kernel (debug;
Q8G_TC_TRACE=1), in us from the first stamp: halo TMA issued, halo landed
(an idle warp waits on its full barrier), accumulator free and both waits
passed (MMA warp), MMAs issued, epilogue start / done; then each epilogue
warp's accumulator release, and the MMA warp's clock64 cycles per wait and
per loop iteration (what paces the kernel: the MMA issue loop).
Needs the trace build of the library: Q8G_TRACE=1 python -c "from
paper_2101_05615_b200 import build as b; b.build()" (the production build
compiles the stamps out; rebuild without Q8G_TRACE afterwards).
"""
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
    a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)[8192:8192 + 448].reshape(7, 64)
    n = int((a[0] > 0).sum())
    t0 = a[0, 0]
    # halo_landed: the halo's full barrier (an otherwise idle warp waits on it);
    # acc_free: the MMA warp got a free accumulator; mma_go: both (halo + accumulator)
    cols = [0, 5, 6, 1, 2, 3, 4]
    print("unit  tma_issue  halo_landed  acc_free  mma_go  mma_issued  epi_start  epi_done   (us)")
    for i in range(n):
        print(f"{i:4d} " + " ".join(f"{(a[j, i] - t0) / 1e3:9.2f}" for j in cols))


    w = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)[8192 + 448:8192 + 448 + 16 * 64].reshape(16, 64)
    if (w[:, 1] > 0).all():
        print("per epilogue warp (warp = K-group row x lane quarter): accumulator released, us after the unit's MMAs issued")
        print("unit " + " ".join(f"w{q:<5d}" for q in range(16)))
        for i in range(min(n, 40)):
            print(f"{i:4d} " + " ".join(f"{(w[q, i] - a[2, i]) / 1e3:6.2f}" for q in range(16)))


    c = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)[8192 + 24 * 64:8192 + 27 * 64].reshape(3, 64)
    if (c[2, 1] > 0):
        print("MMA warp per unit, SM cycles: wait for a free accumulator, wait for the halo, loop period")
        for i in range(1, min(n, 40)):
            print(f"{i:4d} {c[0, i]:8d} {c[1, i]:8d} {c[2, i] - c[2, i - 1]:8d}")


if __name__ == "__main__":
    main()
