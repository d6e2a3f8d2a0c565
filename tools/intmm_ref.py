"""cuBLASLt int8 GEMM (torch._int_mm, s8 x s8 -> s32, no epilogue) at a given
shape, event-timed per launch over rotating buffers: a library yardstick for
the tensor-bound C2 shape, not part of the product path."""
import argparse

import numpy as np
import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16384)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    m, n, k = args.m, args.n, args.k
    dev = torch.device("cuda:0")
    nsets = 3
    As = [torch.randint(-128, 128, (m, k), dtype=torch.int8, device=dev) for _ in range(nsets)]
    Bs = [torch.randint(-128, 128, (n, k), dtype=torch.int8, device=dev).t() for _ in range(nsets)]
    for j in range(nsets):
        torch._int_mm(As[j], Bs[j])
    torch.cuda.synchronize()
    ts = []
    for i in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(As[i % nsets], Bs[i % nsets])
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    us = float(np.median(ts))
    print(f"torch._int_mm {m}x{n}x{k}: median {us:.1f} us  best {min(ts):.1f} us  "
          f"{2 * m * n * k / us / 1e6:.1f} TOPS (median)", flush=True)


if __name__ == "__main__":
    main()
