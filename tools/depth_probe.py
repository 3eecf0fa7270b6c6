"""Throughput of complete trees of one depth at a chosen row width:
1M uniform rows x F features, 1000 complete trees of depth d, 3 timed passes,
bit-exact check of 2000 rows against the C oracle (used to tune the
per-depth chain counts and the global-leaf mode).

    python tools/depth_probe.py F d
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1212_2287_b200 import build_gpu, synth
import oracle
F = int(sys.argv[1]); d = int(sys.argv[2]); T = 1000; n = 1_000_000
rng = np.random.default_rng(3)
n_int = (1 << d) - 1
flat = synth.complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)), rng.standard_normal((T, 1 << d)))
ev = build_gpu(flat)
x = torch.from_numpy(rng.random((n, F), dtype=np.float32)).cuda()
out = torch.empty(n, dtype=torch.float64, device="cuda")
ev.score_device(x, out); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3): ev.score_device(x, out)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 3
ref = oracle.COracle(flat.arrays()).score(x[:2000].cpu().numpy(), threads=8)
print(f"F={F} d={d}: {ms:.3f} ms  {n*T/ms*1e3:.3e} tree-evals/s  exact={np.array_equal(out[:2000].cpu().numpy(), ref)}", flush=True)
