"""Host-buffer scoring latency (ts_score_host through GpuEvaluator._predict_into)
by buffer kind -- pageable / pinned input and output -- for 1k-100k rows of
a 100-tree depth-6 model, next to a plain numpy copy into pinned memory (the
staging cost a pageable input pays).

    python tools/host_latency.py
"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1212_2287_b200 import build_gpu, synth
rng = np.random.default_rng(1)
d, T, F = 6, 100, 136
n_int = (1 << d) - 1
flat = synth.complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)), rng.standard_normal((T, 1 << d)))
ev = build_gpu(flat)
for n in (1000, 10000, 100000):
    x = rng.random((n, F), dtype=np.float32)
    xp = torch.empty((n, F), dtype=torch.float32, pin_memory=True).numpy(); xp[:] = x
    outp = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    out = np.empty(n, np.float64)
    for name, xx, oo in (("pageable x, pageable out", x, out), ("pinned x, pageable out", xp, out), ("pageable x, pinned out", x, outp), ("pinned x, pinned out", xp, outp)):
        for _ in range(5): ev._predict_into(xx, oo)
        t0 = time.perf_counter()
        for _ in range(50): ev._predict_into(xx, oo)
        print(f"n={n:6d} {name:26s} {(time.perf_counter()-t0)/50*1e6:8.1f} us")
    t0 = time.perf_counter()
    for _ in range(50): np.copyto(xp, x)
    print(f"n={n:6d} numpy copy into pinned       {(time.perf_counter()-t0)/50*1e6:8.1f} us")
