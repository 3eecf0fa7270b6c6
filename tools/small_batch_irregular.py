"""Small / medium-batch latency of the irregular-tree kernel (config 3's ensemble).

    python tools/small_batch_irregular.py [--trees 5000] [--ns 32,1000,4000,20000] [--per-graph 4]
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
    ap.add_argument("--trees", type=int, default=5000)
    ap.add_argument("--ns", default="32,1000,4000,20000")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--per-graph", type=int, default=4)
    a = ap.parse_args()
    w = synth.config3(n=1, trees=a.trees)
    ev = build_gpu(w.flat)
    ref = oracle.COracle(w.flat.arrays())
    for n in [int(v) for v in a.ns.split(",")]:
        xh = synth.hash_uniform(w.hash_seed, 0, n, w.f, w.zero_prob)
        x = torch.from_numpy(xh).cuda()
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        for _ in range(3):
            ev.score_device(x, out)
        st = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(a.per_graph):
                ev.score_device(x, out)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(a.reps):
            g.replay()
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) * 1e3 / a.reps / a.per_graph
        m = min(n, 256)
        exact = np.array_equal(out.cpu().numpy()[:m], ref.score(xh[:m], threads=4))
        print(f"cfg3 trees={a.trees} n={n}: {us:9.1f} us/launch  {n * a.trees / us * 1e6:.3g} evals/s  "
              f"exact={exact}")


if __name__ == "__main__":
    main()
