"""Complete trees over rows too wide for the complete-tree kernel's tile
(F = 700): the packer routes them to the irregular-tree kernel.

    python tools/wide_complete_probe.py
"""
import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo") if os.path.exists("/root/repo") else None
sys.path.insert(0, os.getcwd())
import oracle
from paper_1212_2287_b200 import build_gpu
from paper_1212_2287_b200.synth import complete_flat
rng = np.random.default_rng(1)
F, d, T, n = 700, 8, 500, 200000
n_int = (1 << d) - 1
flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)), rng.standard_normal((T, 1 << d)))
X = rng.random((n, F), dtype=np.float32)
xd = torch.from_numpy(X).cuda()
ref = oracle.COracle(flat.arrays()).score(X[:512], threads=8)
for force in ("", "1"):
    if force: os.environ["TS_FORCE_CSTREAM"] = "1"
    ev = build_gpu(flat)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    ev.score_device(xd, out); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3): ev.score_device(xd, out)
    e.record(); torch.cuda.synchronize()
    print("force_cstream" if force else "default", s.elapsed_time(e)/3, "ms", np.array_equal(out.cpu().numpy()[:512], ref), ev.model.info["complete_trees"], ev.model.info["compact_trees"])
