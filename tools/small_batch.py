"""Small-batch latency probe: one scoring launch per call for N rows.

    python tools/small_batch.py [--depth 6] [--trees 100] [--ns 1000,10000,100000]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1212_2287_b200 import build_gpu, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--depth", type=int, default=6)
    ap.add_argument("--trees", type=int, default=100)
    ap.add_argument("--ns", default="1000,10000,100000")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--graph", action="store_true", help="replay a captured CUDA graph")
    ap.add_argument("--per-graph", type=int, default=1,
                    help="launches captured per graph (>1 hides the host's launch cost)")
    a = ap.parse_args()
    rng = np.random.default_rng(5)
    d, T, F = a.depth, a.trees, 136
    n_int = (1 << d) - 1
    flat = synth.complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                               rng.standard_normal((T, 1 << d)))
    ev = build_gpu(flat)
    for n in [int(v) for v in a.ns.split(",")]:
        x = torch.from_numpy(rng.random((n, F), dtype=np.float32)).cuda()
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        for _ in range(5):
            ev.score_device(x, out)
        run = lambda: ev.score_device(x, out)  # noqa: E731
        if a.graph:
            st = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for _ in range(a.per_graph):
                    ev.score_device(x, out)
            run = g.replay
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(a.reps):
            run()
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) * 1e3 / a.reps / (a.per_graph if a.graph else 1)
        got = out.cpu().numpy()
        ref = oracle.COracle(flat.arrays()).score(x.cpu().numpy()[:256], threads=4)
        print(f"d={d} T={T} n={n}: {us:8.1f} us/launch  {n * T / us * 1e6:.3g} evals/s  "
              f"exact={np.array_equal(got[:256], ref)}")


if __name__ == "__main__":
    main()
