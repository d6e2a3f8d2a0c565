"""Host-view C2 call (q8g_gemm_u8s8_requant_host, pinned A and C) wall time:
the e2e leg of bench.py in isolation, for chunk-size A/B (Q8G_HOST_CHUNK)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2101_05615_b200 as q8  # noqa: E402
from paper_2101_05615_b200 import _lib  # noqa: E402


def main():
    m, n, k = 16384, 4096, 4096
    b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device="cuda")
    pw = q8.prepack_weights(b)
    rp = q8.RequantParams(zp_a=128, zp_c=5, k_total=k, zp_b_per_channel=np.full(n, 3, np.int32),
                          multiplier_f32_per_channel=np.full(n, 1e-4, np.float32), rounding=q8.ROUND_F32_RNE)
    pipe = q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(rp)])  # owns the epilogue table
    ep = pipe.epilogue(pw)
    a = torch.randint(0, 256, (m, k), dtype=torch.uint8).pin_memory()
    c = torch.empty((m, n), dtype=torch.uint8).pin_memory()
    lib = _lib.load()
    s = torch.cuda.Stream()
    for _ in range(3):
        _lib.check(lib.q8g_gemm_u8s8_requant_host(a.data_ptr(), m, k, k, pw.handle, ep, c.data_ptr(), n, 0, m,
                                                  s.cuda_stream))
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        _lib.check(lib.q8g_gemm_u8s8_requant_host(a.data_ptr(), m, k, k, pw.handle, ep, c.data_ptr(), n, 0, m,
                                                  s.cuda_stream))
        ts.append(time.perf_counter() - t0)
    print(f"host-view C2: median {np.median(ts) * 1e3:.3f} ms, best {min(ts) * 1e3:.3f} ms")


if __name__ == "__main__":
    main()
