"""Latency of the public host API for small batches (serving): predict_batch
and predict on numpy input, vs the device-only kernel time.

    python tools/api_latency.py [--depth 8] [--trees 1000]
    python tools/api_latency.py --irregular [--trees 5000]    # config 3's ensemble (F = 700)
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1212_2287_b200 import build_gpu, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--depth", type=int, default=8)
    ap.add_argument("--trees", type=int, default=1000)
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--irregular", action="store_true")
    a = ap.parse_args()
    rng = np.random.default_rng(1)
    d, T, F = a.depth, a.trees, 136
    if a.irregular:
        w = synth.config3(n=1, trees=T)
        flat, F, d = w.flat, w.f, "irr"
    else:
        n_int = (1 << d) - 1
        flat = synth.complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                                   rng.standard_normal((T, 1 << d)))
    ev = build_gpu(flat)
    for n in (1, 10, 100, 1000, 10000):
        x = rng.random((n, F), dtype=np.float32)
        for _ in range(10):
            ev.predict_batch(x)
        t0 = time.perf_counter()
        for _ in range(a.reps):
            ev.predict_batch(x)
        us = (time.perf_counter() - t0) / a.reps * 1e6
        print(f"d={d} T={T} predict_batch n={n:6d}: {us:8.1f} us/call", flush=True)
    x1 = rng.random(F, dtype=np.float32)
    t0 = time.perf_counter()
    for _ in range(a.reps):
        ev.predict(x1)
    print(f"d={d} T={T} predict (1 row):     {(time.perf_counter() - t0) / a.reps * 1e6:8.1f} us/call")


if __name__ == "__main__":
    main()
