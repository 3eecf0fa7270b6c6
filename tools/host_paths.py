"""End-to-end host-buffer scoring through the public API: pinned vs pageable input.

    python tools/host_paths.py [--rows 1000000]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1212_2287_b200 import build_gpu, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    w = synth.config1(n=a.rows)
    ev = build_gpu(w.flat)
    pageable = np.ascontiguousarray(w.x)
    pinned_t = torch.empty(pageable.shape, dtype=torch.float32, pin_memory=True)
    pinned_t.numpy()[:] = pageable
    out = np.empty(a.rows, np.float64)
    for name, m in (("pinned", pinned_t.numpy()), ("pageable", pageable)):
        ev._predict_into(m, out)
        t0 = time.perf_counter()
        for _ in range(a.reps):
            ev._predict_into(m, out)
        dt = (time.perf_counter() - t0) / a.reps
        print(f"{name:9s}: {dt * 1e3:7.2f} ms/pass  {a.rows * 1000 / dt:.3g} tree-evals/s  "
              f"{pageable.nbytes / dt / 1e9:5.1f} GB/s of input")


if __name__ == "__main__":
    main()
