"""Long randomized parity run (400 mixed models) on the GPU against the C oracle.

    python tools/fuzz_run.py        # on a GPU box; the suite runs 40 of these
    FUZZ_UNIT=1 ...                 # all tree weights 1.0 (the tree-split modes' exact-sum paths)
"""
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import oracle
from test_gpu_parity import _fuzz_case, _ev
bad = 0
import os
lo = int(os.environ.get("FUZZ_SEED0", "5000"))
for seed in range(lo, lo + int(os.environ.get("FUZZ_N", "400"))):
    rng = np.random.default_rng(seed)
    ens, X = _fuzz_case(rng)
    if os.environ.get("FUZZ_UNIT"):
        from paper_1212_2287_b200 import Ensemble
        ens = Ensemble(ens.num_features, [(t, 1.0) for t, _w in ens.trees])
    s, o = oracle.COracle(ens.flat().arrays()).score(X, threads=2, with_ordinals=True)
    ev = _ev(ens)
    ok = np.array_equal(ev.predict_batch(X), s) and np.array_equal(ev.leaf_indices(X), o.astype(np.int64))
    if not ok:
        bad += 1; print("MISMATCH seed", seed)
    ev.close()
print("fuzz done, mismatches:", bad)
