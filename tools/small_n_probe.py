import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1212_2287_b200 import build_gpu, synth
rng = np.random.default_rng(1)
d, T, F = 8, 1000, 136
n_int = (1 << d) - 1
flat = synth.complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)), rng.standard_normal((T, 1 << d)))
ev = build_gpu(flat)
for n in (1, 32, 1000):
    x = torch.rand((n, F), device="cuda"); out = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3): ev.score_device(x, out)
    torch.cuda.synchronize()
