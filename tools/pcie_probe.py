"""Pinned host<->device copy rates on this box: H2D on one and two streams,
D2H alone, and H2D (two streams) concurrent with D2H -- the link bound that
bench.py's e2e number sits under."""

import json
import time

import torch


def rate(fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t0) / 1e9


def main():
    n = 512 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2, s3 = (torch.cuda.Stream() for _ in range(3))

    def h2d1():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)

    def h2d2():
        half = n // 2
        with torch.cuda.stream(s1):
            d[:half].copy_(h[:half], non_blocking=True)
        with torch.cuda.stream(s2):
            d[half:].copy_(h[half:], non_blocking=True)

    def d2h():
        with torch.cuda.stream(s3):
            h2.copy_(d2, non_blocking=True)

    def duplex():
        h2d2()
        d2h()

    out = {"h2d_1stream_GBs": rate(h2d1, n), "h2d_2streams_GBs": rate(h2d2, n), "d2h_GBs": rate(d2h, n)}
    t = 2 * n * 5 / 1e9
    duplex()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        duplex()
    torch.cuda.synchronize()
    out["duplex_total_GBs"] = round(t / (time.perf_counter() - t0), 2)
    print(json.dumps({k: round(v, 2) for k, v in out.items()}))


if __name__ == "__main__":
    main()
