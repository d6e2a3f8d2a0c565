"""Phase timeline of one tensor-core GEMM launch (debug; needs Q8G_TC_TRACE=1).

Stamps (globaltimer ns) per CTA: 0 entry, 1 prologue done, 2 first TMA
issued, 3 first stage landed (MMA), 4 last MMA commit, 5 epilogue start,
6 epilogue done, 7 exit.  Prints min/median/max of each relative to the
earliest entry over all CTAs.
Needs the trace build of the library: Q8G_TRACE=1 python -c "from
paper_2101_05615_b200 import build as b; b.build()" (the production build
compiles the stamps out; rebuild without Q8G_TRACE afterwards).
"""
import argparse
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

NAMES = ["entry", "prologue", "tma0", "stage0", "mma_done", "epi_start", "epi_done", "exit"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=128)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--requant", action="store_true", help="per-channel F32 requant + ReLU (the bench's pipeline)")
    ap.add_argument("--steady", type=int, default=0,
                    help="trace the last of this many back-to-back launches over rotating weights (> L2)")
    args = ap.parse_args()
    m, n, k = args.m, args.n, args.k
    b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device="cuda")
    a = torch.randint(0, 256, (m, k), dtype=torch.uint8, device="cuda")
    pw = q8.prepack_weights(b)
    if args.requant:
        rp = q8.RequantParams(zp_a=128, zp_c=5, k_total=k, zp_b_per_channel=np.full(n, 3, np.int32),
                              multiplier_f32_per_channel=np.full(n, 1e-4, np.float32), rounding=q8.ROUND_F32_RNE)
        pipe = q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(rp)])
        c = torch.empty((m, n), dtype=torch.uint8, device="cuda")
    else:
        pipe = q8.OutputPipeline([q8.WriteRawI32()])
        c = torch.empty((m, n), dtype=torch.int32, device="cuda")
    for _ in range(3):
        q8.execute_gemm(a, pw, c, pipe)
    torch.cuda.synchronize()
    if args.steady:
        # back-to-back launches over rotating weights (> L2), replayed from one
        # CUDA graph like bench.py, so the launch spacing is the device's
        pws = [pw] + [pw.replicate(0) for _ in range(max(1, int(2.2 * 126e6 / (k * n))))]
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):  # the split-K workspace is per stream: create it before capture
            for p_ in pws:
                q8.execute_gemm(a, p_, c, pipe)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=st):
            for i in range(args.steady):
                q8.execute_gemm(a, pws[i % len(pws)], c, pipe)
        graph.replay()  # the first replay also uploads the graph; trace the second
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
    else:
        # flush L2 between the warm-up and the traced launch
        junk = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        junk.fill_(1)
        torch.cuda.synchronize()
        q8.execute_gemm(a, pw, c, pipe)
        torch.cuda.synchronize()
    buf = (C.c_uint64 * (8 * 1024 + 2048))()
    nct = _lib.load().q8g_debug_tc_trace(buf, 2048)
    allw = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
    if args.steady:
        # split-K: successive launches stamp alternate halves -> show both
        def fresh(h):  # stamped rows of the latest launch in this half
            h = h[h[:, 0] > 0]
            return h[h[:, 0] > h[:, 0].max() - 50_000] if len(h) else h
        h0, h1 = fresh(allw[:4096].reshape(512, 8)), fresh(allw[4096:8192].reshape(512, 8))
        if len(h0) and len(h1) and abs(int(h0[:, 0].min()) - int(h1[:, 0].min())) < 100_000:
            first, second = (h0, h1) if h0[:, 0].min() < h1[:, 0].min() else (h1, h0)
            z = first[:, 0].min()
            print(f"two successive launches, us from the first one's earliest entry ({len(first)} CTAs each)")
            for nm_i, nm in enumerate(NAMES):
                for tag, arr in (("N", first), ("N+1", second)):
                    col = arr[:, nm_i]
                    col = col[col > 0] - z
                    if len(col):
                        print(f"  {tag:3s} {nm:10s} min {col.min()/1e3:8.2f} us  med {np.median(col)/1e3:8.2f}"
                              f"  max {col.max()/1e3:8.2f}")
            return
    t = allw[:8 * 1024].reshape(1024, 8)[:nct]
    kbs = allw[8192:8192 + 192].reshape(3, 64)
    used = t[:, 0] > 0
    t = t[used]
    t0 = t[:, 0].min()
    print(f"cfg={os.environ.get('Q8G_TC_CFG', 'auto')} {m}x{n}x{k}: {len(t)} CTAs traced")
    for i, nm in enumerate(NAMES):
        col = t[:, i]
        col = col[col > 0] - t0
        if len(col):
            print(f"  {nm:10s} min {col.min()/1e3:8.2f} us  med {np.median(col)/1e3:8.2f}  max {col.max()/1e3:8.2f}")
    c0 = t[0, 0]
    kb6 = allw[8192:8192 + 384].reshape(6, 64)
    if (kb6[3] > 0).any():  # CTA-pair kernel: 6 columns
        nk = int((kb6[0] > 0).sum())
        print("  pair 0 per k-block (us from CTA0 entry): leader issue / past full / past pfull / MMAs issued /"
              " follower issue / relay sent")
        for kb in range(nk):
            print(f"    kb {kb:2d}: " + " ".join(f"{(kb6[w, kb]-c0)/1e3:7.2f}" for w in range(6)))
        return
    nk = int((kbs[0] > 0).sum())
    print("  CTA0 per k-block (us from its entry): issue / landed / mma-issued")
    for kb in range(nk):
        print(f"    kb {kb:2d}: {(kbs[0, kb]-c0)/1e3:7.2f} {(kbs[1, kb]-c0)/1e3:7.2f} {(kbs[2, kb]-c0)/1e3:7.2f}")


if __name__ == "__main__":
    main()
