import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1212_2287_b200 import GpuModel, synth
for d in (12, 13, 14):
  for rank in (False, True):
    rng = np.random.default_rng(d)
    n_int = (1 << d) - 1
    T, n = 200, 500_000
    flat = synth.complete_flat(136, d, rng.integers(0, 136, (T, n_int)), rng.random((T, n_int)), rng.standard_normal((T, 1 << d)))
    m = GpuModel(flat, 0, rank=rank)
    x = torch.rand((n, 136), device="cuda"); out = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(2): m.score(x, out=out)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3): m.score(x, out=out)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 3
    print(f"d={d} T={T} n={n} rank_trees={m.info['rank_trees']}: {ms:.2f} ms  {n*T*d/ms/1e6:.3g} visits/s", flush=True)
