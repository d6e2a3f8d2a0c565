"""Where an end-to-end (host-view) C1 step spends its time: pinned H2D of A,
the device-view GEMM call, D2H of C, and the whole synchronous
q8g_gemm_u8s8_requant_host call.  CUDA events on one stream, medians."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2101_05615_b200 as q8  # noqa: E402
from paper_2101_05615_b200 import _lib  # noqa: E402


def main():
    m, n, k = 128, 4096, 4096
    b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device="cuda")
    pw = q8.prepack_weights(b)
    rp = q8.RequantParams(zp_a=128, zp_c=5, k_total=k, zp_b_per_channel=np.zeros(n, np.int32) + 3,
                          multiplier_f32_per_channel=np.full(n, 1e-4, np.float32), rounding=q8.ROUND_F32_RNE)
    pipe = q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(rp)])
    ep = pipe.epilogue(pw)
    lib = _lib.load()
    s = torch.cuda.Stream()
    a_h = torch.randint(0, 256, (m, k), dtype=torch.uint8).pin_memory()
    c_h = torch.empty((m, n), dtype=torch.uint8).pin_memory()
    a_d = torch.empty((m, k), dtype=torch.uint8, device="cuda")
    c_d = torch.empty((m, n), dtype=torch.uint8, device="cuda")

    def timed(f, reps=50):
        ts = []
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            f()
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return float(np.median(ts))

    with torch.cuda.stream(s):
        h2d = timed(lambda: a_d.copy_(a_h, non_blocking=True))
        d2h = timed(lambda: c_h.copy_(c_d, non_blocking=True))
        gemm = timed(lambda: _lib.check(lib.q8g_gemm_u8s8_requant(a_d.data_ptr(), m, k, k, pw.handle, ep, c_d.data_ptr(),
                                                                   n, 0, m, None, s.cuda_stream)))
        full = timed(lambda: _lib.check(lib.q8g_gemm_u8s8_requant_host(a_h.data_ptr(), m, k, k, pw.handle, ep,
                                                                        c_h.data_ptr(), n, 0, m, s.cuda_stream)))
        # the GEMM epilogue storing straight into the pinned host buffer (UVA-mapped)
        zc = timed(lambda: _lib.check(lib.q8g_gemm_u8s8_requant(a_d.data_ptr(), m, k, k, pw.handle, ep, c_h.data_ptr(),
                                                                 n, 0, m, None, s.cuda_stream)))
        ok_zc = bool(torch.equal(c_h, c_d.cpu()))
        # H2D split in two halves on two streams (two copy engines?)
        s2 = torch.cuda.Stream()

        def h2d_split():
            ev = torch.cuda.Event()
            ev.record(s)
            s2.wait_event(ev)
            a_d[: m // 2].copy_(a_h[: m // 2], non_blocking=True)
            with torch.cuda.stream(s2):
                a_d[m // 2:].copy_(a_h[m // 2:], non_blocking=True)
            ev2 = torch.cuda.Event()
            ev2.record(s2)
            s.wait_event(ev2)
        h2d2 = timed(h2d_split)
        # overlap probe: H2D on s2 concurrent with the GEMM on s (stale A), then D2H on s
        a_d2 = torch.empty_like(a_d)

        def overlap():
            ev = torch.cuda.Event()
            ev.record(s)
            s2.wait_event(ev)
            with torch.cuda.stream(s2):
                a_d2.copy_(a_h, non_blocking=True)
            _lib.check(lib.q8g_gemm_u8s8_requant(a_d.data_ptr(), m, k, k, pw.handle, ep, c_d.data_ptr(), n, 0, m, None,
                                                 s.cuda_stream))
            ev2 = torch.cuda.Event()
            ev2.record(s2)
            s.wait_event(ev2)
            c_h.copy_(c_d, non_blocking=True)
        ovl = timed(overlap)
    print(f"overlap probe (H2D || GEMM, then D2H): {ovl:.1f} us")
    print(f"GEMM writing C into pinned host memory: {zc:.1f} us (matches device result: {ok_zc})")
    print(f"H2D split over two streams: {h2d2:.1f} us")
    t0 = time.perf_counter()
    for _ in range(200):
        _lib.check(lib.q8g_gemm_u8s8_requant_host(a_h.data_ptr(), m, k, k, pw.handle, ep, c_h.data_ptr(), n, 0, m,
                                                  s.cuda_stream))
    wall = (time.perf_counter() - t0) / 200 * 1e6
    print(f"H2D A {m}x{k} pinned: {h2d:.1f} us ({m * k / h2d / 1e3:.1f} GB/s)")
    print(f"D2H C {m}x{n} pinned: {d2h:.1f} us ({m * n / d2h / 1e3:.1f} GB/s)")
    print(f"GEMM device views (single launch, not graphed): {gemm:.1f} us")
    print(f"host-view call (event span): {full:.1f} us   wall clock per call: {wall:.1f} us")


if __name__ == "__main__" and "--timeline" not in sys.argv:
    main()


def overlap_timeline():
    """Events around an H2D on one stream and a GEMM on another, both issued
    right after a common start event: do they run concurrently?"""
    m, n, k = 128, 4096, 4096
    b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device="cuda")
    pw = q8.prepack_weights(b)
    rp = q8.RequantParams(zp_a=128, zp_c=5, k_total=k, zp_b_per_channel=np.zeros(n, np.int32) + 3,
                          multiplier_f32_per_channel=np.full(n, 1e-4, np.float32), rounding=q8.ROUND_F32_RNE)
    pipe = q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(rp)])  # owns the epilogue
    ep = pipe.epilogue(pw)
    lib = _lib.load()
    s, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    a_h = torch.randint(0, 256, (m, k), dtype=torch.uint8).pin_memory()
    a_d = torch.empty((m, k), dtype=torch.uint8, device="cuda")
    a_d2 = torch.empty((m, k), dtype=torch.uint8, device="cuda")
    c_d = torch.empty((m, n), dtype=torch.uint8, device="cuda")
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for it in range(6):
        ev0, c0, c1, g0, g1 = E(), E(), E(), E(), E()
        ev0.record(s)
        s2.wait_event(ev0)
        c0.record(s2)
        with torch.cuda.stream(s2):
            a_d2.copy_(a_h, non_blocking=True)
        c1.record(s2)
        g0.record(s)
        _lib.check(lib.q8g_gemm_u8s8_requant(a_d.data_ptr(), m, k, k, pw.handle, ep, c_d.data_ptr(), n, 0, m, None,
                                             s.cuda_stream))
        g1.record(s)
        torch.cuda.synchronize()
        if it >= 3:
            print(f"copy {ev0.elapsed_time(c0)*1e3:6.1f} -> {ev0.elapsed_time(c1)*1e3:6.1f} us   "
                  f"gemm {ev0.elapsed_time(g0)*1e3:6.1f} -> {ev0.elapsed_time(g1)*1e3:6.1f} us")


if __name__ == "__main__" and "--timeline" in sys.argv:
    overlap_timeline()
