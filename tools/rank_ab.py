"""A/B of the rank layout (kRank: ts_rank.cu) against the fp32 streaming
layout (k_stream) for complete trees: same model, same device-resident rows,
CUDA events over back-to-back launches; scores compared bit for bit.

    python tools/rank_ab.py [--depths 9,10,11,12] [--rows 1000000] [--trees 1000]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1212_2287_b200 import GpuModel, synth  # noqa: E402


def timed(m, x, out, reps):
    for _ in range(2):
        m.score(x, out=out)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        m.score(x, out=out)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--depths", default="9,10,11,12")
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--trees", type=int, default=1000)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    for d in [int(v) for v in a.depths.split(",")]:
        if d in (3, 4, 6, 8, 10, 12):
            w = synth.config2(d, n=a.rows, trees=a.trees)
            flat, x = w.flat, torch.from_numpy(w.x).cuda()
        else:
            rng = np.random.default_rng(d)
            n_int = (1 << d) - 1
            flat = synth.complete_flat(136, d, rng.integers(0, 136, (a.trees, n_int)),
                                       rng.random((a.trees, n_int)),
                                       rng.standard_normal((a.trees, 1 << d)))
            x = torch.rand((a.rows, 136), device="cuda")
        out_r = torch.empty(a.rows, dtype=torch.float64, device="cuda")
        out_f = torch.empty_like(out_r)
        os.environ["TS_RANK_MIN_DEPTH"] = "1"
        mr = GpuModel(flat, 0)
        mf = GpuModel(flat, 0, rank=False)
        t_r, t_f = timed(mr, x, out_r, a.reps), timed(mf, x, out_f, a.reps)
        print(json.dumps({"depth": d, "rows": a.rows, "trees": a.trees,
                          "rank_ms": t_r, "fp32_ms": t_f, "speedup": t_f / t_r,
                          "rank_segments_layout": mr.info.get("num_segments"),
                          "equal": bool(torch.equal(out_r, out_f))}), flush=True)
        mr.close()
        mf.close()


if __name__ == "__main__":
    main()
