"""Both CPU baselines of SURVEY 8(d)(ii), side by side, on this host's cores.

    python tools/cpu_baselines.py [--configs 0,2:3,2:4,2:6,1] [--seconds 8]

* ``port``: the C restatement of the reference's VPred path
  (``oracle/ts_oracle.c``), lockstep batches of 64 rows, one pthread per core.
* ``generated``: the reference's CodeGen strategy -- the C text its
  ``emit_source`` produces (``oracle/codegen.py`` emits it byte-identically,
  ``tests/test_codegen_baseline.py``) compiled with its own flags
  (``-O3 -fomit-frame-pointer -pipe``), one thread per core over row shards
  through ``score_batch`` (ref ``GeneratedUnit.score_batch_into``).

Each is gated first as the reference harness gates its strategies
(``_correctness_gate``, ref bench.py:220-231: the 1,000-row prefix must equal
the reference traversal exactly; here the C oracle, itself pinned to the
reference's golden vectors), then timed over whole passes of a row prefix
for about ``--seconds`` seconds.  Prints one JSON line per config with both
rates and which is faster (the reported baseline).  Compiles that are not
cached under ``oracle/_gen/`` happen first and are reported (config 1's
1000 x 511-node source takes minutes; ``__graft_entry__.build`` prebuilds it).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from oracle import codegen  # noqa: E402
from paper_1212_2287_b200 import synth  # noqa: E402


def workload(key: str, rows: int):
    if key == "0":
        return synth.config0()
    if key == "1":
        return synth.config1(n=rows)
    if key.startswith("2:"):
        return synth.config2(int(key[2:]), n=rows)
    raise ValueError(key)


def timed(fn, x, target_s):
    """Whole passes over growing prefixes until ~target_s; evals counted by caller."""
    probe = min(len(x), 2000)
    t0 = time.perf_counter()
    fn(x[:probe])
    dt = time.perf_counter() - t0
    rows = int(min(len(x), max(probe, probe * target_s / 3 / max(dt, 1e-6))))
    passes, t0 = 0, time.perf_counter()
    while True:
        fn(x[:rows])
        passes += 1
        dt = time.perf_counter() - t0
        if dt >= target_s or passes >= 100:
            return rows * passes, dt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,2:3,2:4,2:6,1")
    ap.add_argument("--seconds", type=float, default=8.0)
    ap.add_argument("--rows", type=int, default=200_000)
    a = ap.parse_args()
    cores = len(os.sched_getaffinity(0))
    for key in a.configs.split(","):
        w = workload(key, a.rows)
        T = w.flat.num_trees
        t0 = time.time()
        unit = codegen.cached_unit(w.flat)
        compiled_here = unit is None
        if unit is None:
            unit = codegen.compile_unit(w.flat)
        compile_s = time.time() - t0
        c = oracle.COracle(w.flat.arrays())
        prefix = w.x[:1000]
        ref = c.score(prefix, threads=cores)
        gate = {"port": bool(np.array_equal(c.score(prefix, threads=1), ref)),
                "generated": bool(np.array_equal(unit.score(prefix, threads=cores), ref))}
        out = np.empty(len(w.x), np.float64)
        rows_p, dt_p = timed(lambda xx: c.score(xx, threads=cores), w.x, a.seconds)
        rows_g, dt_g = timed(lambda xx: unit.score_parallel(xx, out[:len(xx)], cores), w.x, a.seconds)
        port, gen = rows_p * T / dt_p, rows_g * T / dt_g
        print(json.dumps({
            "config": key, "workload": w.name, "cores": cores, "trees": T,
            "port_evals_per_s": port, "generated_evals_per_s": gen,
            "faster": "generated" if gen > port else "port",
            "generated_over_port": gen / port,
            "correctness_gate_1000_rows": gate,
            "generated_compile_s": round(compile_s, 1) if compiled_here else "prebuilt",
            "sample": {"port": f"{rows_p} row-evals in {dt_p:.1f} s",
                       "generated": f"{rows_g} row-evals in {dt_g:.1f} s"},
        }), flush=True)


if __name__ == "__main__":
    main()
