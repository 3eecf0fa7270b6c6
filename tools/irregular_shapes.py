"""Irregular-tree kernel shapes at a given feature width (planner A/B).

    python tools/irregular_shapes.py [--f 136] [--rows 500000] [--trees 2000]

Scores LambdaMART-shaped trees (64 leaves, depth <= 16, Zipf fids) under every
forced TS_CSTREAM_PLAN shape and the planner's own choice; one line each with
ms/pass and a bit-exact check on a row sample against the C oracle.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1212_2287_b200 import build_gpu, synth  # noqa: E402

PLANS = ["", "8,8,8,1", "4,8,8,1", "2,8,8,1", "1,8,8,1", "4,16,8,1", "4,16,4,1", "2,16,8,1",
         "2,16,4,1", "2,16,3,1", "1,16,8,1", "1,16,4,1", "1,16,3,1"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--f", type=int, default=136)
    ap.add_argument("--rows", type=int, default=500_000)
    ap.add_argument("--trees", type=int, default=2000)
    a = ap.parse_args()
    flat = synth.irregular_flat(7, a.trees, a.f)
    rng = np.random.default_rng(3)
    X = rng.random((a.rows, a.f), dtype=np.float32)
    X[rng.random(X.shape) < 0.4] = 0.0
    xd = torch.from_numpy(X).cuda()
    sample = np.linspace(0, a.rows - 1, 1024).astype(np.int64)
    ref = oracle.COracle(flat.arrays()).score(X[sample], threads=8)
    for plan in PLANS:
        if plan:
            os.environ["TS_CSTREAM_PLAN"] = plan
        else:
            os.environ.pop("TS_CSTREAM_PLAN", None)
        ev = build_gpu(flat)
        out = torch.empty(a.rows, dtype=torch.float64, device="cuda")
        ev.score_device(xd, out)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(3):
            ev.score_device(xd, out)
        e.record()
        torch.cuda.synchronize()
        ok = np.array_equal(out.cpu().numpy()[sample], ref)
        print(f"plan {plan or 'auto':10s} {s.elapsed_time(e) / 3:8.2f} ms  exact={ok}  "
              f"compact_trees={ev.model.info['compact_trees']}", flush=True)
        ev.close()


if __name__ == "__main__":
    main()
