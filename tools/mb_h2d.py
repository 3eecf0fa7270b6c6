"""H2D bandwidth probe: pinned host -> device, one vs two copy streams, chunk sizes.

    python tools/mb_h2d.py
"""
import time

import torch


def run(total, chunk, nstreams):
    src = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(total, dtype=torch.uint8, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, c0 in enumerate(range(0, total, chunk)):
            s = streams[i % nstreams]
            with torch.cuda.stream(s):
                dst[c0:c0 + chunk].copy_(src[c0:c0 + chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    return total / dt / 1e9


if __name__ == "__main__":
    total = 544_000_000
    for chunk in (4 << 20, 16 << 20, 64 << 20, 544_000_000):
        for ns in (1, 2):
            print(f"chunk {chunk >> 20:4d} MiB streams {ns}: {run(total, chunk, ns):6.1f} GB/s")
