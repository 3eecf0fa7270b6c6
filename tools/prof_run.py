"""Small profiling driver: score a BASELINE workload a few times on cuda:0.

    python tools/prof_run.py [--cfg 1] [--n 200000] [--reps 3] [--depth 8]

Used under ncu (one GPU).  Prints the per-launch time measured with CUDA
events when run without a profiler.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1212_2287_b200 import build_gpu, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="1")
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--trees", type=int, default=1000)
    ap.add_argument("--depth", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    if a.cfg == "1":
        w = synth.config1(n=a.n, trees=a.trees)
    elif a.cfg == "2":
        w = synth.config2(a.depth, n=a.n, trees=a.trees)
    elif a.cfg == "3":
        w = synth.config3(n=a.n, trees=a.trees)
    else:
        w = synth.config0(n=a.n)
    ev = build_gpu(w.flat)
    if w.x is not None:
        x = torch.from_numpy(w.x).cuda()
    else:
        x = torch.from_numpy(w.rows(0, w.n)).cuda()
    out = torch.empty(w.n, dtype=torch.float64, device="cuda")
    ev.score_device(x, out=out)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.reps):
        ev.score_device(x, out=out)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.reps
    evals = w.n * w.flat.num_trees
    print(f"{w.name}: {ms:.3f} ms/launch-set, {evals / ms / 1e6:.3e} evals/s, "
          f"info={ev.model.info}")


if __name__ == "__main__":
    main()
