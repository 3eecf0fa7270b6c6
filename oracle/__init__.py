"""CPU oracle for the scoring path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (and ``bench.py --impl reference``) may import this package.  The product
package never imports, links or calls it; it is the checker, never the thing
measured as the GPU result.

Two independent restatements of the reference ``treescore`` arithmetic:

* ``numpy`` (this file): lockstep predicated traversal over complete tables,
  one numpy statement per level for all rows at once, exactly the reference's
  ``batch_kernel`` (``evaluators.py:90-99``) applied tree by tree with
  ``acc += w * leaf64[ord]`` (``evaluators.py:529-535``).  The complete tables
  come from a recursive ``expand`` restating ``expand_to_complete``
  (``model.py:315-349``).  A linked walk restates ``traverse_to_leaf`` /
  ``reference_predict`` (``model.py:251-271``).
* ``C`` (``ts_oracle.c``, built to ``_ts_oracle.so`` by ``make``): the same
  arithmetic, multi-threaded over row shards; fast enough for the parity
  checks at BASELINE sizes and used as the CPU baseline (kind ``"port"``).

Pinning: ``tests/test_oracle.py`` checks both against golden vectors that
``tests/golden/make_golden.py`` produced by running the reference package
itself (scores from ``reference_batch`` and ``VPredicatedEvaluator``, per-tree
ordinals from ``batch_kernel`` on ``expand_to_complete``), and against the
reference's own known-answer cases (tie goes right, dummy routing, unbalanced
3-leaf ordinals {0, 2, 3}).

Inputs are "flat trees": ``tree_off int64[T+1]``, ``weight f64[T]`` and per
node ``fid int32`` (-1 = leaf), ``value f32`` (threshold or leaf value),
``left/right int32`` tree-local ids with the root at 0.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

MAX_DEPTH = 16
_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_ts_oracle.so")


# ---------------------------------------------------------------------------
# numpy restatement
# ---------------------------------------------------------------------------

def _depth(fid, left, right, node):
    if fid[node] < 0:
        return 0
    return 1 + max(_depth(fid, left, right, left[node]), _depth(fid, left, right, right[node]))


def expand(flat):
    """Flat trees -> list of complete tables ``(depth, fids, thetas, leaves)``."""
    off, _w, fid, val, left, right = flat
    out = []
    for t in range(len(off) - 1):
        o = int(off[t])
        f = fid[o:int(off[t + 1])]
        v = val[o:int(off[t + 1])]
        lc = left[o:int(off[t + 1])]
        rc = right[o:int(off[t + 1])]
        d = _depth(f, lc, rc, 0)
        if d > MAX_DEPTH:
            raise ValueError(f"tree {t} depth {d} exceeds {MAX_DEPTH}")
        n_int = (1 << d) - 1
        cf = np.zeros(n_int, np.int32)
        ct = np.zeros(n_int, np.float32)
        cl = np.zeros(1 << d, np.float32)

        def fill(node, slot):
            if slot >= n_int:
                cl[slot - n_int] = v[node]
            elif f[node] < 0:
                cf[slot] = 0
                ct[slot] = np.inf
                fill(node, 2 * slot + 1)
                fill(node, 2 * slot + 2)
            else:
                cf[slot] = f[node]
                ct[slot] = v[node]
                fill(lc[node], 2 * slot + 1)
                fill(rc[node], 2 * slot + 2)

        fill(0, 0)
        out.append((d, cf, ct, cl))
    return out


def ordinals(tables, X) -> np.ndarray:
    """Per-tree predicated leaf ordinals, shape ``(T, n)``, int64."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    n = X.shape[0]
    rows = np.arange(n)
    res = np.empty((len(tables), n), dtype=np.int64)
    for t, (d, cf, ct, _cl) in enumerate(tables):
        i = np.zeros(n, dtype=np.int64)
        for _ in range(d):
            i = (i << 1) + 1 + (X[rows, cf[i]] >= ct[i])
        res[t] = i - ((1 << d) - 1)
    return res


def score(tables, weights, X, ords=None, init=None) -> np.ndarray:
    """f64 tree-order sum ``acc += w * leaf64[ord]`` (starts at +0.0, or at
    ``init`` -- the running sums of the trees before these, for tree shards)."""
    if ords is None:
        ords = ordinals(tables, X)
    acc = np.zeros(ords.shape[1], dtype=np.float64) if init is None \
        else np.array(init, dtype=np.float64, copy=True)
    for t, (_d, _cf, _ct, cl) in enumerate(tables):
        acc += float(weights[t]) * cl.astype(np.float64)[ords[t]]
    return acc


def score_linked(flat, X) -> np.ndarray:
    """Row-by-row linked walk, strict ``<`` goes left (the reference oracle)."""
    off, w, fid, val, left, right = flat
    X = np.asarray(X, dtype=np.float32)
    out = np.empty(X.shape[0], dtype=np.float64)
    for r in range(X.shape[0]):
        acc = 0.0
        for t in range(len(off) - 1):
            o = int(off[t])
            i = 0
            while fid[o + i] >= 0:
                i = left[o + i] if float(X[r, fid[o + i]]) < float(val[o + i]) else right[o + i]
            acc += float(w[t]) * float(val[o + i])
        out[r] = acc
    return out


def trace(flat, X):
    """Restates predict_ensemble_traced (ref evaluators.py:599-620) per row:
    visited-feature bitsets ``uint32 [n, ceil(f/32)]`` (real splits only) and
    logical left-to-right leaf ordinals ``[T, n]``."""
    off, _w, fid, val, left, right = flat
    X = np.asarray(X, dtype=np.float32)
    n, f = X.shape
    T = len(off) - 1
    bits = np.zeros((n, (f + 31) // 32), np.uint32)
    leaves = np.empty((T, n), np.int64)
    for t in range(T):
        o = int(off[t])
        # left-to-right leaf numbering: depth-first, left child first
        ordinal = {}
        stack = [0]
        while stack:
            i = stack.pop()
            if fid[o + i] < 0:
                ordinal[i] = len(ordinal)
            else:
                stack.append(int(right[o + i]))
                stack.append(int(left[o + i]))
        for r in range(n):
            i = 0
            while fid[o + i] >= 0:
                k = int(fid[o + i])
                bits[r, k >> 5] |= np.uint32(1 << (k & 31))
                i = int(left[o + i]) if float(X[r, k]) < float(val[o + i]) else int(right[o + i])
            leaves[t, r] = ordinal[i]
    return bits, leaves


# ---------------------------------------------------------------------------
# C restatement (ctypes)
# ---------------------------------------------------------------------------

_lib = None


def build_c() -> str:
    """Compile ``_ts_oracle.so`` with the committed Makefile; return its path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build_c()
        lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        I32, I64 = ctypes.c_int32, ctypes.c_int64
        lib.orc_depths.argtypes = [I32, P, P, P, P, P]
        lib.orc_depths.restype = ctypes.c_int
        lib.orc_expand.argtypes = [I32, P, P, P, P, P, P, P, P, P, P, P]
        lib.orc_expand.restype = None
        lib.orc_score.argtypes = [I32, P, P, P, P, P, P, P, P, I64, I64, I64, P, P, I64,
                                  I64, ctypes.c_int]
        lib.orc_score.restype = None
        lib.orc_score_linked.argtypes = [I32, P, P, P, P, P, P, P, I64, I64, P]
        lib.orc_score_linked.restype = None
        _lib = lib
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


class COracle:
    """Expanded complete tables plus the threaded C scorer."""

    def __init__(self, flat):
        lib = _load()
        off, w, fid, val, left, right = [np.ascontiguousarray(a) for a in flat]
        self.flat = (off.astype(np.int64), w.astype(np.float64), fid.astype(np.int32),
                     val.astype(np.float32), left.astype(np.int32), right.astype(np.int32))
        off, w, fid, val, left, right = self.flat
        T = len(off) - 1
        self.num_trees = T
        self.depth = np.zeros(T, np.int32)
        if lib.orc_depths(T, _p(off), _p(fid), _p(left), _p(right), _p(self.depth)) != 0:
            raise ValueError(f"tree depth exceeds {MAX_DEPTH}")
        d = self.depth.astype(np.int64)
        self.int_off = np.zeros(T + 1, np.int64)
        self.leaf_off = np.zeros(T + 1, np.int64)
        np.cumsum((1 << d) - 1, out=self.int_off[1:])
        np.cumsum(1 << d, out=self.leaf_off[1:])
        self.cfid = np.zeros(max(1, self.int_off[-1]), np.int32)
        self.ctheta = np.zeros(max(1, self.int_off[-1]), np.float32)
        self.cleaf = np.zeros(self.leaf_off[-1], np.float32)
        lib.orc_expand(T, _p(off), _p(fid), _p(val), _p(left), _p(right), _p(self.depth),
                       _p(self.int_off), _p(self.leaf_off), _p(self.cfid), _p(self.ctheta),
                       _p(self.cleaf))
        self.weight = w

    def tables(self):
        """Complete tables in the numpy oracle's ``(d, fids, thetas, leaves)`` form."""
        out = []
        for t in range(self.num_trees):
            a, b = self.int_off[t], self.int_off[t + 1]
            c, e = self.leaf_off[t], self.leaf_off[t + 1]
            out.append((int(self.depth[t]), self.cfid[a:b], self.ctheta[a:b], self.cleaf[c:e]))
        return out

    def score(self, X, *, threads: int | None = None, with_ordinals: bool = False,
              v: int = 64):
        lib = _load()
        X = np.ascontiguousarray(X, dtype=np.float32)
        n, f = X.shape
        out = np.empty(n, np.float64)
        ords = np.empty((self.num_trees, n), np.uint16) if with_ordinals else None
        threads = threads or len(os.sched_getaffinity(0))
        lib.orc_score(self.num_trees, _p(self.depth), _p(self.int_off), _p(self.leaf_off),
                      _p(self.cfid), _p(self.ctheta), _p(self.cleaf), _p(self.weight),
                      _p(X), n, f, f, _p(out), _p(ords), n, v, threads)
        return (out, ords) if with_ordinals else out

    def score_linked(self, X):
        lib = _load()
        X = np.ascontiguousarray(X, dtype=np.float32)
        out = np.empty(X.shape[0], np.float64)
        off, w, fid, val, left, right = self.flat
        lib.orc_score_linked(self.num_trees, _p(off), _p(fid), _p(val), _p(left), _p(right),
                             _p(w), _p(X), X.shape[0], X.shape[1], _p(out))
        return out


# ---------------------------------------------------------------------------
# sampled parity at BASELINE sizes (SURVEY 8(c) sampling protocol)
# ---------------------------------------------------------------------------

def sample_rows(n: int, k: int, run: int = 32, seed: int = 0) -> np.ndarray:
    """Sorted row indices for a parity sample of about ``k`` rows spread over
    ``[0, n)``: the first and last ``run`` rows (the tail tile included) plus
    seeded random runs of ``run`` contiguous rows (whole 32-row warp blocks
    when ``run`` is 32), so every region of a multi-GB matrix is visited."""
    if n <= k:
        return np.arange(n, dtype=np.int64)
    rng = np.random.default_rng(seed)
    starts = [0, max(0, n - run)]
    starts += list(rng.integers(0, max(1, n - run), size=max(0, k // run - 2)))
    rows = np.unique(np.concatenate([np.arange(s, min(n, s + run)) for s in starts]))
    return rows.astype(np.int64)


def runs_of(rows: np.ndarray):
    """``[(start, length)]`` of the contiguous runs in sorted ``rows``."""
    if len(rows) == 0:
        return []
    cut = np.flatnonzero(np.diff(rows) != 1) + 1
    bounds = np.concatenate([[0], cut, [len(rows)]])
    return [(int(rows[a]), int(b - a)) for a, b in zip(bounds[:-1], bounds[1:])]


def score_tolerance(c: "COracle", X, ref) -> np.ndarray:
    """Per-row bound of the north star's 1e-5 relative check with the
    SURVEY 8(c) denominator guard: ``1e-5 * max(|s_ref|, sum_t |w_t leaf_t|)``."""
    _, ords = c.score(X, with_ordinals=True)
    mag = np.zeros(X.shape[0], np.float64)
    for t in range(c.num_trees):
        lv = c.cleaf[c.leaf_off[t]:c.leaf_off[t + 1]].astype(np.float64)
        mag += np.abs(c.weight[t] * lv[ords[t]])
    return 1e-5 * np.maximum(np.abs(ref), mag)
