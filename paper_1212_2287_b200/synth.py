"""Seeded synthetic workloads for the five BASELINE.json configurations.

The paper's learning-to-rank data (MSLR-WEB10K, LETOR) and its trained
models are not available; these generators stand in for them with the shapes
and value distributions BASELINE.json names.
Ensembles are built directly as :class:`FlatModel` arrays (no per-node Python
objects), thresholds and leaves rounded to float32 like ``Node`` does.

Instances:
* configs 0-2 use numpy ``PCG64`` streams seeded ``SeedSequence([20261020,
  cfg, 1])`` (trees use stream 0);
* configs 3 and 4 (2M x 700 and 64M x 136 rows -- 5.6 and 34.8 GB) use a
  counter-based generator so that any row can be produced independently, on
  the GPU (``ts_synth_uniform`` in ``_ts_gpu.so``) or on the host
  (:func:`hash_uniform`, bit-identical): element ``e = row * f + col`` maps
  to ``u = splitmix64(seed + (e + 1) * golden) >> 40`` scaled by 2^-24, so
  ``u`` is an exact float32 in [0, 1); a second stream zeroes entries with
  probability ``zero_prob`` (config 3's sparse-feature zeros).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .model import FlatModel

SEED = 20261020
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
ZERO_STREAM = np.uint64(0xD1B54A32D192ED03)


def _rng(cfg: int, stream: int):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED, cfg, stream])))


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * M1
    z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def hash_uniform(seed: int, row0: int, rows: int, f: int, zero_prob: float = 0.0) -> np.ndarray:
    """Host reproduction of ``ts_synth_uniform`` for rows ``[row0, row0+rows)``."""
    with np.errstate(over="ignore"):
        e = np.arange(row0 * f, (row0 + rows) * f, dtype=np.uint64)
        s = np.uint64(seed)
        u = (_mix(s + (e + np.uint64(1)) * GOLDEN) >> np.uint64(40)).astype(np.float32)
        x = u * np.float32(2.0 ** -24)
        if zero_prob > 0:
            z = _mix((s ^ ZERO_STREAM) + (e + np.uint64(1)) * GOLDEN) >> np.uint64(40)
            x[z < np.uint64(int(zero_prob * (1 << 24)))] = 0.0
    return x.reshape(rows, f)


def complete_flat(num_features: int, depth: int, fids, thetas, leaves, weights=None) -> FlatModel:
    """FlatModel of T complete trees from heap tables ``[T, 2^d-1]`` / ``[T, 2^d]``."""
    fids = np.asarray(fids, np.int32)
    T = fids.shape[0]
    n_int = (1 << depth) - 1
    n = 2 * n_int + 1
    fid = np.full((T, n), -1, np.int32)
    val = np.empty((T, n), np.float32)
    left = np.full((T, n), -1, np.int32)
    right = np.full((T, n), -1, np.int32)
    fid[:, :n_int] = fids
    val[:, :n_int] = np.asarray(thetas, np.float32)
    val[:, n_int:] = np.asarray(leaves, np.float32)
    idx = np.arange(n_int, dtype=np.int32)
    left[:, :n_int] = 2 * idx + 1
    right[:, :n_int] = 2 * idx + 2
    off = np.arange(T + 1, dtype=np.int64) * n
    w = np.ones(T, np.float64) if weights is None else np.asarray(weights, np.float64)
    return FlatModel(num_features, off, w, fid.ravel(), val.ravel(), left.ravel(), right.ravel())


@dataclass
class Workload:
    name: str
    flat: FlatModel
    n: int
    f: int
    x: np.ndarray | None = None          # host instances when generated on the host
    hash_seed: int | None = None         # counter-based instances (configs 3/4)
    zero_prob: float = 0.0
    meta: dict = field(default_factory=dict)

    def rows(self, row0: int, rows: int) -> np.ndarray:
        """Host copy of instances ``[row0, row0+rows)`` (for oracle checks)."""
        if self.x is not None:
            return self.x[row0:row0 + rows]
        return hash_uniform(self.hash_seed, row0, rows, self.f, self.zero_prob)


def _uniform_complete(cfg: int, T: int, d: int, F: int, leaf_sigma: float, rng=None):
    rng = rng or _rng(cfg, 0)
    n_int = (1 << d) - 1
    fids = rng.integers(0, F, size=(T, n_int), dtype=np.int32)
    thetas = rng.random((T, n_int), dtype=np.float32)
    leaves = (leaf_sigma * rng.standard_normal((T, 1 << d))).astype(np.float32)
    return complete_flat(F, d, fids, thetas, leaves)


def config0(n: int = 10_000) -> Workload:
    """10k x 136 U[0,1); 100 complete depth-6 trees; thr U[0,1); leaf N(0,1)."""
    flat = _uniform_complete(0, 100, 6, 136, 1.0)
    x = _rng(0, 1).random((n, 136), dtype=np.float32)
    return Workload("cfg0: 10k x 136, T=100 d=6", flat, n, 136, x=x)


def _config1_columns(kinds, n, rng):
    x = np.empty((n, len(kinds)), np.float32)
    for c, k in enumerate(kinds):
        if k == 0:
            x[:, c] = rng.random(n, dtype=np.float32)
        elif k == 1:
            x[:, c] = rng.lognormal(0.0, 1.0, n).astype(np.float32)
        else:
            x[:, c] = rng.integers(0, 51, n).astype(np.float32)
    return x


def config1(n: int = 1_000_000, trees: int = 1000, shard: int = 0) -> Workload:
    """1M x 136 mixed columns (70% U[0,1), 20% lognormal(0,1), 10% integer
    counts in [0,50]); 1000 complete depth-8 trees; each threshold is the
    split column's value in a random row of a seeded 100k-row sample drawn
    from the same column distributions (so count thresholds are integers and
    exact ties occur); leaf N(0,0.1).  ``shard`` selects an independent row
    stream of the same distribution (one per GPU in the scaling runs); the
    ensemble does not depend on it."""
    F = 136
    kinds = np.array([0] * 95 + [1] * 27 + [2] * 14)
    kinds = kinds[_rng(1, 2).permutation(F)]
    rt = _rng(1, 0)
    sample = _config1_columns(kinds, 100_000, _rng(1, 3))
    d = 8
    n_int = (1 << d) - 1
    fids = rt.integers(0, F, size=(trees, n_int), dtype=np.int32)
    rows = rt.integers(0, sample.shape[0], size=(trees, n_int))
    thetas = sample[rows, fids]
    leaves = (0.1 * rt.standard_normal((trees, 1 << d))).astype(np.float32)
    flat = complete_flat(F, d, fids, thetas, leaves)
    rx = np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED, 1, 1, shard])))
    x = _config1_columns(kinds, n, rx)
    return Workload(f"cfg1: {n // 1000}k x 136 mixed, T={trees} d=8", flat, n, F, x=x,
                    meta={"column_kinds": kinds})


def config2(depth: int, n: int = 1_000_000, trees: int = 1000) -> Workload:
    """1M x 136 U[0,1); 1000 complete trees of the given depth."""
    if depth not in (3, 4, 6, 8, 10, 12):
        raise ValueError("config 2 depths are 3, 4, 6, 8, 10, 12")
    flat = _uniform_complete(200 + depth, trees, depth, 136, 1.0)
    x = _rng(2, 1).random((n, 136), dtype=np.float32)
    return Workload(f"cfg2: {n // 1000}k x 136, T={trees} d={depth}", flat, n, 136, x=x)


def irregular_flat(cfg: int, T: int, F: int, leaves: int = 64, max_depth: int = 16,
                   zipf_s: float = 1.1, leaf_sigma: float = 0.05) -> FlatModel:
    """Trees grown by splitting a uniformly chosen leaf of depth < max_depth
    until ``leaves`` leaves; split fids truncated Zipf(s) over F ids."""
    rng = _rng(cfg, 0)
    p = np.arange(1, F + 1, dtype=np.float64) ** -zipf_s
    p /= p.sum()
    n = 2 * leaves - 1
    fid = np.full((T, n), -1, np.int32)
    val = np.empty((T, n), np.float32)
    left = np.full((T, n), -1, np.int32)
    right = np.full((T, n), -1, np.int32)
    all_fids = rng.choice(F, size=(T, leaves - 1), p=p).astype(np.int32)
    all_thr = rng.random((T, leaves - 1), dtype=np.float32)
    all_leaf = (leaf_sigma * rng.standard_normal((T, n))).astype(np.float32)
    picks = rng.random((T, leaves - 1))
    for t in range(T):
        depth = [0]
        open_leaves = [0]          # splittable leaves (depth < max_depth)
        used = 1
        for s in range(leaves - 1):
            k = int(picks[t, s] * len(open_leaves))
            i = open_leaves[k]
            open_leaves[k] = open_leaves[-1]
            open_leaves.pop()
            fid[t, i] = all_fids[t, s]
            val[t, i] = all_thr[t, s]
            left[t, i] = used
            right[t, i] = used + 1
            for c in (used, used + 1):
                depth.append(depth[i] + 1)
                if depth[c] < max_depth:
                    open_leaves.append(c)
            used += 2
        leaf_ids = fid[t] < 0
        val[t, leaf_ids] = all_leaf[t, leaf_ids]
    off = np.arange(T + 1, dtype=np.int64) * n
    return FlatModel(F, off, np.ones(T), fid.ravel(), val.ravel(), left.ravel(), right.ravel())


def config3(n: int = 2_000_000, trees: int = 5000) -> Workload:
    """2M x 700 U[0,1) with 40% exact zeros; 5000 irregular 64-leaf trees of
    depth <= 16, Zipf(1.1) split features, leaf N(0,0.05)."""
    flat = irregular_flat(3, trees, 700)
    return Workload(f"cfg3: {n // 1000}k x 700 sparse, T={trees} irregular<=16", flat, n, 700,
                    hash_seed=SEED * 10 + 3, zero_prob=0.4)


def config4a(n: int = 64_000_000) -> Workload:
    """64M x 136 U[0,1) instance-sharded; config 2's depth-8 ensemble."""
    flat = _uniform_complete(208, 1000, 8, 136, 1.0)
    return Workload(f"cfg4a: {n // 1_000_000}M x 136, T=1000 d=8", flat, n, 136,
                    hash_seed=SEED * 10 + 4)


def config4b(n: int = 8_000_000, trees: int = 20_000) -> Workload:
    """8M x 136 U[0,1) tree-sharded; 20,000 complete depth-10 trees."""
    flat = _uniform_complete(41, trees, 10, 136, 1.0)
    return Workload(f"cfg4b: {n // 1_000_000}M x 136, T={trees} d=10", flat, n, 136,
                    hash_seed=SEED * 10 + 41)
