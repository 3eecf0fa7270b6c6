"""Time traced prediction (ts_trace: per-row visited-feature bitsets, logical
leaf ordinals, scores) on config-1 and config-3 shaped work, checking it
against the oracle's restatement of the reference's traced walk.

    python tools/trace_bench.py            # TS_GPU_SO=... for another build
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1212_2287_b200 import GpuModel, synth  # noqa: E402


def main():
    for name, w, n in [("cfg1 shape (F=136, 1000 d=8 trees)", synth.config1(n=100_000), 100_000),
                       ("cfg3 shape (F=700, 5000 irregular trees)", synth.config3(n=20_000), 20_000)]:
        x = torch.from_numpy(w.rows(0, n)).cuda()
        m = GpuModel(w.flat, 0, trace=True)
        words = (w.f + 31) // 32
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        vis = torch.zeros((n, words), dtype=torch.int32, device="cuda")
        ords = torch.empty((w.flat.num_trees, n), dtype=torch.int16, device="cuda")
        run = lambda: m.trace(x, out=out, leaf_ord=ords, visited=vis)  # noqa: E731
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        k = 64
        ref_bits, ref_leaves = oracle.trace(w.flat.arrays(), w.rows(0, k))
        ref_s = oracle.COracle(w.flat.arrays()).score(w.rows(0, k))
        ok = (np.array_equal(out[:k].cpu().numpy(), ref_s)
              and np.array_equal(vis[:k].cpu().numpy().view(np.uint32), ref_bits)
              and np.array_equal(ords[:, :k].cpu().numpy().view(np.uint16).astype(np.int64),
                                 ref_leaves))
        print(json.dumps({"workload": name, "rows": n, "trees": w.flat.num_trees, "ms": ms,
                          "tree_evals_per_s": n * w.flat.num_trees / ms * 1e3,
                          "lib": os.environ.get("TS_GPU_SO", "in-tree"),
                          "matches_oracle_trace_64_rows": bool(ok)}), flush=True)
        m.close()


if __name__ == "__main__":
    main()
