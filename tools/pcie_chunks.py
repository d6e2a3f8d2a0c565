"""PCIe floor of the host-view C2 call (64 MB in, 64 MB out, pinned): the
same chunk schedule as the library's host pipeline (ramped 512, 1024, 2048,
..., 1024, 512 rows of 4096 B) with the GEMM left out -- each chunk's D2H
waits only for its own H2D -- against one 64 MB copy per direction issued at
once.  Wall clock per round, median of 20."""
import time

import torch


def chunks(rows, c):
    q, h = c // 4, c // 2
    b, u = [0], 0

    def push(n):
        nonlocal u
        u = min(rows, u + n)
        if u > b[-1]:
            b.append(u)
    push(q)
    push(h)
    while rows - u > c + h + q:
        push(c)
    push(rows - u - h - q)
    push(h)
    push(q)
    return list(zip(b[:-1], b[1:]))


def main():
    rows, width = 16384, 4096
    hin = torch.randint(0, 256, (rows, width), dtype=torch.uint8).pin_memory()
    hout = torch.empty((rows, width), dtype=torch.uint8).pin_memory()
    din = torch.empty((rows, width), dtype=torch.uint8, device="cuda")
    dout = torch.randint(0, 256, (rows, width), dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def whole():
        with torch.cuda.stream(s1):
            din.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(dout, non_blocking=True)
        torch.cuda.synchronize()

    def chunked(c):
        for r0, r1 in chunks(rows, c):
            with torch.cuda.stream(s1):
                din[r0:r1].copy_(hin[r0:r1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s1)
            s2.wait_event(ev)
            with torch.cuda.stream(s2):
                hout[r0:r1].copy_(dout[r0:r1], non_blocking=True)
        torch.cuda.synchronize()

    def h2d_only():
        with torch.cuda.stream(s1):
            din.copy_(hin, non_blocking=True)
        torch.cuda.synchronize()

    def d2h_only():
        with torch.cuda.stream(s2):
            hout.copy_(dout, non_blocking=True)
        torch.cuda.synchronize()

    for name, f in (("H2D 64 MB alone", h2d_only), ("D2H 64 MB alone", d2h_only),
                    ("both directions, one copy each", whole),
                    ("chunked 2048 (ramped), D2H after its H2D", lambda: chunked(2048)),
                    ("chunked 4096 (ramped), D2H after its H2D", lambda: chunked(4096))):
        for _ in range(3):
            f()
        ts = []
        for _ in range(20):
            t0 = time.perf_counter()
            f()
            ts.append(time.perf_counter() - t0)
        ts.sort()
        print(f"{name:44s} median {ts[len(ts) // 2] * 1e3:.3f} ms  best {ts[0] * 1e3:.3f} ms")


if __name__ == "__main__":
    main()
