"""Per-launch timing of the tensor-core GEMM variants (tuning tool).

  Q8G_TC_CFG=32x8 python tools/tc_sweep.py --m 128 --n 4096 --k 4096

Times one kernel per graph node with event pairs (graph-captured, rotating
buffers > L2) for three epilogues: raw int32, requant with row sums
(per-channel zp_b), requant without row sums (zp_b = 0).
"""
import argparse
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2101_05615_b200 as q8  # noqa: E402
from paper_2101_05615_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=128)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--nsets", type=int, default=0, help="buffer sets (0: enough to exceed 2x L2)")
    ap.add_argument("--only", default="", help="run only this epilogue")
    args = ap.parse_args()
    m, n, k = args.m, args.n, args.k
    dev = torch.device("cuda:0")
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    g = torch.Generator(device=dev).manual_seed(0)
    b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device=dev, generator=g)
    set_bytes = m * k + k * n + m * n * 4
    nsets = args.nsets or max(2, min(32, int(np.ceil(2.2 * 126e6 / set_bytes))))
    pw0 = q8.prepack_weights(b)
    pws = [pw0] + [pw0.replicate(0) for _ in range(nsets - 1)]
    As = [torch.randint(0, 256, (m, k), dtype=torch.uint8, device=dev, generator=g) for _ in range(nsets)]
    Cu = [torch.empty((m, n), dtype=torch.uint8, device=dev) for _ in range(nsets)]
    Ci = [torch.empty((m, n), dtype=torch.int32, device=dev) for _ in range(nsets)]
    lib = _lib.load()
    zp = np.random.default_rng(1).integers(-10, 11, n).astype(np.int32)
    mult = np.full(n, 1e-4, np.float32)
    pipes = {
        "requant+rowsum": q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(q8.RequantParams(
            zp_a=128, zp_c=5, k_total=k, zp_b_per_channel=zp, multiplier_f32_per_channel=mult,
            rounding=q8.ROUND_F32_RNE))]),
        "requant(zp_b=0)": q8.OutputPipeline([q8.Requantize(q8.RequantParams(
            zp_a=128, zp_c=5, k_total=k, zp_b=0, multiplier_f32_per_channel=mult, rounding=q8.ROUND_F32_RNE))]),
    }
    res = {}
    for name in ["raw", *pipes]:
        if args.only and name != args.only:
            continue
        if name == "raw":
            def launch(j):
                _lib.check(lib.q8g_gemm_u8s8_raw_i32(As[j].data_ptr(), m, k, k, pws[j].handle, None,
                                                     Ci[j].data_ptr(), n, 0, m, None, stream.cuda_stream))
        else:
            eps = [pipes[name].epilogue(p) for p in pws]

            def launch(j, eps=eps):
                _lib.check(lib.q8g_gemm_u8s8_requant(As[j].data_ptr(), m, k, k, pws[j].handle, eps[j],
                                                     Cu[j].data_ptr(), n, 0, m, None, stream.cuda_stream))
        for j in range(nsets):
            launch(j)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
              for _ in range(nsets)]
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=stream):
            for j in range(nsets):
                ev[j][0].record(stream)
                launch(j)
                ev[j][1].record(stream)
        ts = []
        for _ in range(args.reps):
            gr.replay()
            torch.cuda.synchronize()
            ts += [a.elapsed_time(bb) * 1e3 for a, bb in ev]
        us = float(np.median(ts))
        res[name] = us
        abytes = m * k + k * n + m * n
        print(f"cfg={os.environ.get('Q8G_TC_CFG', 'auto')} sets={nsets} {m}x{n}x{k} {name:18s} {us:9.2f} us  "
              f"{2 * m * n * k / us / 1e6:8.1f} TOPS  {abytes / us / 1e3:8.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
