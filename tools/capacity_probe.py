import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1212_2287_b200 import build_gpu, synth
for d in (10, 12):
    for F in (136, 68, 34):
        rng = np.random.default_rng(1)
        n_int = (1 << d) - 1
        T, n = 1000, 600_000
        flat = synth.complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)), rng.standard_normal((T, 1 << d)))
        ev = build_gpu(flat)
        x = torch.rand((n, F), device="cuda")
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        for _ in range(2): ev.score_device(x, out)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5): ev.score_device(x, out)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        print(f"d={d} F={F}: {ms:.3f} ms  {n*T/ms/1e6:.3g} evals/s", flush=True)
        ev.close()
