"""Per-tile timeline of CTA 0 (leader of pair 0) in the 256 x 512 CTA-pair
GEMM (gemm_tc2w.cu; debug, Q8G_TC_TRACE=1) at the C2 shape, us from the
first stamp: when the MMA issuer got each accumulator half back (tempty),
when it committed each half (tfull), when the epilogue saw each half full
and when it had drained it into registers.  --raw / --zpb0 select the
epilogue; the last launch of --reps back-to-back launches is shown.
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
    m, n, k = 16384, 4096, 4096
    b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device="cuda")
    a = torch.randint(0, 256, (m, k), dtype=torch.uint8, device="cuda")
    pw = q8.prepack_weights(b)
    zpb = 0 if "--zpb0" in sys.argv else 3
    rp = q8.RequantParams(zp_a=128, zp_c=5, k_total=k, zp_b_per_channel=np.full(n, zpb, np.int32),
                          multiplier_f32_per_channel=np.full(n, 1e-4, np.float32), rounding=q8.ROUND_F32_RNE)
    pipe = q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(rp)])
    c = torch.empty((m, n), dtype=torch.uint8, device="cuda")
    if "--raw" in sys.argv:
        pipe = q8.OutputPipeline([q8.WriteRawI32()])
        c = torch.empty((m, n), dtype=torch.int32, device="cuda")
    for _ in range(5):
        q8.execute_gemm(a, pw, c, pipe)
    torch.cuda.synchronize()
    buf = (C.c_uint64 * (8 * 1024 + 2048))()
    _lib.load().q8g_debug_tc_trace(buf, 2048)
    w = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
    tiles = w[9216:9216 + 128].reshape(16, 8)
    epi = w[9472:9472 + 128].reshape(16, 8)
    keep = tiles[:, 0] > 0
    tiles, epi = tiles[keep], epi[keep]
    t0 = tiles[0, 0]
    clk, ns = w[10201] - w[10200], w[10203] - w[10202]
    print(f"launch: {ns / 1e3:.1f} us at {clk / max(ns, 1) * 1e3:.0f} MHz")
    print("tile  mma:tempty0 tempty1  tfull0  tfull1 | epi:full0 drained0  full1 drained1   (us)  tile span")
    for i, r in enumerate(tiles):
        span = (tiles[i + 1, 0] - r[0]) / 1e3 if i + 1 < len(tiles) else float("nan")
        print(f"{i:4d} " + " ".join(f"{(x - t0) / 1e3:8.2f}" for x in r) + f"   {span:8.2f}")
    print("epilogue warp 4, per half: row sums in hand / round-0 requant done / round-1 staging free / "
          "round-1 requant done (us)")
    for i, e in enumerate(epi):
        print(f"{i:4d} " + " ".join(f"{(x - t0) / 1e3:8.2f}" for x in (e[6], *e[0:3], e[7], *e[3:6])))


if __name__ == "__main__":
    main()
