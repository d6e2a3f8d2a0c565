"""Effective SM clock of the C2 CTA-pair GEMM (debug, Q8G_TC_TRACE=1): for
graphs of N back-to-back launches, the mean per-launch time and the last
launch's clock64 / globaltimer ratio measured in CTA 0 -- how far the 1 kW
power cap pulls the clock down as a run of C2 launches lengthens."""
import ctypes as C
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

os.environ.setdefault("Q8G_TC_TRACE", "1")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2101_05615_b200 as q8  # noqa: E402
from paper_2101_05615_b200 import _lib  # noqa: E402


def main():
    m, n, k = 16384, 4096, 4096
    args = [x for x in sys.argv[1:] if not x.startswith("--")]
    counts = [int(x) for x in (args or ["1", "5", "25", "100", "1000", "25"])]
    b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device="cuda")
    if "--zeroB" in sys.argv:  # data-dependence of the MMA power: constant operands
        b.zero_()
    pw = q8.prepack_weights(b)
    zpb = np.random.default_rng(1).integers(-10, 11, n).astype(np.int32)
    rp = q8.RequantParams(zp_a=128, zp_c=5, k_total=k, zp_b_per_channel=zpb,
                          multiplier_f32_per_channel=np.full(n, 1e-4, np.float32), rounding=q8.ROUND_F32_RNE)
    pipe = q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(rp)])
    As = [torch.randint(0, 256, (m, k), dtype=torch.uint8, device="cuda") for _ in range(2)]
    if "--zeroA" in sys.argv:
        for x in As:
            x.zero_()
    Cs = [torch.empty((m, n), dtype=torch.uint8, device="cuda") for _ in range(2)]
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    for j in range(2):
        q8.execute_gemm(As[j], pw, Cs[j], pipe)
    torch.cuda.synchronize()
    lib = _lib.load()
    buf = (C.c_uint64 * (8 * 1024 + 2048))()
    for cnt in counts:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(cnt):
                q8.execute_gemm(As[i % 2], pw, Cs[i % 2], pipe)
        g.replay()  # the first replay of a fresh graph also uploads it
        torch.cuda.synchronize()
        time.sleep(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        lib.q8g_debug_tc_trace(buf, 2048)
        w = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
        clk, ns = w[10201] - w[10200], w[10203] - w[10202]
        print(f"N={cnt:5d}  {e0.elapsed_time(e1) * 1e3 / cnt:8.1f} us/launch  last launch CTA0 "
              f"{ns / 1e3:7.1f} us at {clk / max(ns, 1) * 1e3:7.0f} MHz", flush=True)


if __name__ == "__main__":
    main()
