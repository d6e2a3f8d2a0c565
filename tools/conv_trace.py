"""Per-unit timeline of CTA 0 in the tensor-core conv3x3 kernel (debug;
Q8G_TC_TRACE=1), C3 shape.  Columns: halo issued / MMA start / MMA committed
/ epilogue start / epilogue done, us from the first stamp; plus prologue end.
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
    nb, h, w, c, oc = 32, 56, 56, 64, 64
    rng = np.random.default_rng(0)
    wt = rng.integers(-128, 128, (3, 3, c, oc)).astype(np.int8)
    pw = q8.prepack_conv3x3_weights(wt)
    rp = q8.RequantParams(zp_a=128, zp_c=5, k_total=9 * c, bias=rng.integers(-1000, 1001, oc).astype(np.int32),
                          zp_b_per_channel=rng.integers(-10, 11, oc).astype(np.int32),
                          multiplier_f32_per_channel=np.full(oc, 0.0005, np.float32), rounding=q8.ROUND_F32_RNE)
    pipe = q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(rp)])
    # --graph N: the last of N back-to-back launches replayed from a CUDA graph
    # over 22 rotating buffer sets (> 2x L2, as bench.py) -- the steady state
    nsets = 22 if "--graph" in sys.argv else 1
    xs = [torch.randint(0, 256, (nb, h, w, c), dtype=torch.uint8, device="cuda") for _ in range(nsets)]
    ys = [torch.empty((nb, h, w, oc), dtype=torch.uint8, device="cuda") for _ in range(nsets)]
    x, y = xs[0], ys[0]
    for _ in range(3):
        q8.execute_conv3x3(x, pw, y, pipe)
    torch.cuda.synchronize()
    if "--graph" in sys.argv:
        steps = int(sys.argv[sys.argv.index("--graph") + 1])
        s = torch.cuda.Stream()
        torch.cuda.set_stream(s)
        for i in range(nsets):
            q8.execute_conv3x3(xs[i], pw, ys[i], pipe)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(steps):
                q8.execute_conv3x3(xs[i % nsets], pw, ys[i % nsets], pipe)
        g.replay()  # the first replay also uploads the graph; time / trace the second
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        print(f"graph of {steps}: {e0.elapsed_time(e1) * 1e3 / steps:.2f} us per launch")
    buf = (C.c_uint64 * (8 * 1024 + 2048))()
    _lib.load().q8g_debug_tc_trace(buf, 2048)
    a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
    units = a[8192:8192 + 320].reshape(5, 64)
    t0 = a[8192 + 321]
    ent, ext = a[8704:8704 + 148], a[8704 + 160:8704 + 160 + 148]
    print(f"grid span: first entry {(ent.min() - t0) / 1e3:.2f}  last entry {(ent.max() - t0) / 1e3:.2f}  "
          f"first exit {(ext.min() - t0) / 1e3:.2f}  last exit {(ext.max() - t0) / 1e3:.2f} us; "
          f"CTA0 exit {(ext[0] - t0) / 1e3:.2f}")
    ee, xx = (ent - t0) / 1e3, (ext - t0) / 1e3
    order = np.argsort(xx)
    print("exit percentiles (us):", " ".join(f"p{q}={np.percentile(xx, q):.2f}" for q in (0, 10, 50, 90, 100)))
    print("latest 12 exits (cta: entry -> exit):",
          "  ".join(f"{i}: {ee[i]:.2f}->{xx[i]:.2f}" for i in order[-12:]))
    print("corr(entry, exit) =", f"{np.corrcoef(ee, xx)[0, 1]:.2f}")
    print(f"kernel entry at 0; barriers+image issued {(a[9344] - t0) / 1e3:.2f}, guards zeroed {(a[9345] - t0) / 1e3:.2f}, "
          f"TMEM allocated {(a[9346] - t0) / 1e3:.2f}, guard stores done {(a[9347] - t0) / 1e3:.2f}, prologue done at {(a[8192 + 320] - t0) / 1e3:.2f} us")
    n = int((units[0] > 0).sum())
    tl = a[8192 + 384:8192 + 448]
    w5, w6 = a[9216:9216 + 64], a[9280:9280 + 64]
    print("unit  halo_issued  mma_start  mma_commit  epi_start  epi_done  tmem_landed  past_tempty  past_full (us)")
    for i in range(n):
        print(f"{i:4d} " + " ".join(f"{(units[j, i] - t0) / 1e3:9.2f}" for j in range(5)) +
              f" {(tl[i] - t0) / 1e3:9.2f} {(w5[i] - t0) / 1e3:9.2f} {(w6[i] - t0) / 1e3:9.2f}")




if __name__ == "__main__":
    main()

