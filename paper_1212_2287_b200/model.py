"""Logical tree ensembles, their validation, and the text model format.

This is the host-side mirror of the reference's model layer
(``treescore/model.py``) for the one hot path this package accelerates:
scoring dense fp32 instances against an ordered list of weighted regression
trees.  The public names and their meaning follow the reference so that code
written against it keeps working:

* ``Node.leaf`` / ``Node.internal`` narrow thresholds and leaf values to
  float32 and reject non-finite values (ref ``model.py:74-119``).
* ``Tree`` derives depth / leaf count / node count / max fid and rejects
  shared nodes (ref ``model.py:131-183``).
* ``Ensemble`` keeps trees in evaluation order with float64 weights
  (ref ``model.py:186-226``).
* ``CompleteTree`` / ``expand_to_complete`` give the breadth-first complete
  table with dummy ``(fid=0, theta=+inf)`` padding (ref ``model.py:278-349``).
* ``traverse_to_leaf`` / ``reference_predict`` are the scalar semantics
  (left iff ``x[fid] < threshold``; ties go right; f64 accumulation in tree
  order, ref ``model.py:251-271``).
* ``parse_model`` / ``serialize_model`` implement the line-oriented text
  format (ref ``model.py:356-535``, grammar in ``SPEC.md`` External Interfaces).

Unlike the reference, every tree is stored *flat*: four parallel arrays
(``fid``, ``value``, ``left``, ``right``) in breadth-first order with the
root at 0 and leaves marked by ``fid == -1``.  Flat trees are what the native
packer (``csrc/ts_pack.cpp``) consumes, so large ensembles (20,000 trees of
depth 10) never materialise Python node objects.  ``Tree.root`` still
rebuilds a ``Node`` graph on demand for callers that walk nodes.
"""

from __future__ import annotations

import math
from collections import deque
from typing import Iterable, NamedTuple

import numpy as np

MAX_DEPTH = 16
DUMMY_FID = 0
DUMMY_THETA = math.inf


class ModelError(Exception):
    """Base class for model construction and model-format errors."""


class ModelSyntaxError(ModelError):
    """Malformed model document; carries 1-based ``line`` and ``col``."""

    def __init__(self, message: str, line: int, col: int):
        super().__init__(f"line {line}, col {col}: {message}")
        self.line = line
        self.col = col


class ModelSemanticError(ModelError):
    """Well-formed document (or object graph) that is not a valid ensemble."""


class DepthLimitError(ModelError):
    """Tree deeper than MAX_DEPTH for a predicated (complete-table) layout."""


def _narrow(x) -> float:
    """Round to the nearest float32 and return it as an exact Python float."""
    with np.errstate(over="ignore"):
        return float(np.float32(x))


class Node:
    """One logical node: an internal split (fid, threshold) or a leaf (value)."""

    __slots__ = ("fid", "threshold", "value", "left", "right")

    def __init__(self, fid, threshold, value, left, right):
        self.fid = fid
        self.threshold = threshold
        self.value = value
        self.left = left
        self.right = right

    @classmethod
    def leaf(cls, value) -> "Node":
        v = _narrow(value)
        if not math.isfinite(v):
            raise ModelSemanticError(f"leaf value must be finite, got {v!r}")
        return cls(-1, 0.0, v, None, None)

    @classmethod
    def internal(cls, fid: int, threshold, left: "Node", right: "Node") -> "Node":
        fid = int(fid)
        if fid < 0:
            raise ModelSemanticError(f"feature id must be non-negative, got {fid}")
        thr = _narrow(threshold)
        if not math.isfinite(thr):
            raise ModelSemanticError(f"threshold must be finite, got {thr!r}")
        if not (isinstance(left, Node) and isinstance(right, Node)):
            raise ModelSemanticError("internal node requires exactly two child nodes")
        return cls(fid, thr, 0.0, left, right)

    @property
    def is_leaf(self) -> bool:
        return self.left is None

    def __repr__(self):
        if self.is_leaf:
            return f"Node.leaf({self.value!r})"
        return f"Node.internal(fid={self.fid}, threshold={self.threshold!r}, ...)"


def _is_foreign_node(obj) -> bool:
    # Duck-typed node from the reference package (treescore.model.Node).
    return all(hasattr(obj, a) for a in ("fid", "threshold", "value", "left", "right"))


class Tree:
    """A validated binary regression tree stored as flat BFS arrays.

    ``fid[i] == -1`` marks a leaf whose value is ``value[i]``; otherwise
    ``value[i]`` is the float32 threshold and ``left[i]``/``right[i]`` are the
    child ids.  Node 0 is the root.  ``depth`` is the longest root-to-leaf
    edge count (0 for a single leaf).
    """

    __slots__ = ("fid", "value", "left", "right", "depth", "leaf_count",
                 "node_count", "max_fid", "_root", "_leaf_ord")

    def __init__(self, root=None, *, _flat=None):
        if _flat is not None:
            fid, value, left, right = _flat
        else:
            if isinstance(root, Tree):
                fid, value, left, right = root.fid, root.value, root.left, root.right
            elif isinstance(root, Node) or (root is not None and _is_foreign_node(root)):
                fid, value, left, right = _flatten_graph(root)
                self._root = root if isinstance(root, Node) else None
            else:
                raise ModelSemanticError("tree root must be a Node")
        self.fid = np.ascontiguousarray(fid, dtype=np.int32)
        self.value = np.ascontiguousarray(value, dtype=np.float32)
        self.left = np.ascontiguousarray(left, dtype=np.int32)
        self.right = np.ascontiguousarray(right, dtype=np.int32)
        if _flat is not None or not hasattr(self, "_root"):
            self._root = None
        self._leaf_ord = None
        self._validate_and_measure()
        for a in (self.fid, self.value, self.left, self.right):
            a.flags.writeable = False

    # -- construction helpers --------------------------------------------------

    @classmethod
    def from_arrays(cls, fid, value, left, right) -> "Tree":
        """Build from flat arrays (any node order with root at id 0)."""
        fid = np.asarray(fid, dtype=np.int64)
        value = np.asarray(value, dtype=np.float64)
        left = np.asarray(left, dtype=np.int64)
        right = np.asarray(right, dtype=np.int64)
        with np.errstate(over="ignore"):
            value32 = value.astype(np.float32)
        return cls(_flat=(fid, value32, left, right))

    @classmethod
    def complete(cls, depth: int, fids, thetas, leaves) -> "Tree":
        """Build a complete tree directly from heap-ordered tables."""
        n_int = (1 << depth) - 1
        n = 2 * n_int + 1
        fid = np.full(n, -1, dtype=np.int32)
        value = np.empty(n, dtype=np.float32)
        left = np.full(n, -1, dtype=np.int32)
        right = np.full(n, -1, dtype=np.int32)
        fid[:n_int] = np.asarray(fids, dtype=np.int32)
        with np.errstate(over="ignore"):
            value[:n_int] = np.asarray(thetas, dtype=np.float32)
            value[n_int:] = np.asarray(leaves, dtype=np.float32)
        idx = np.arange(n_int, dtype=np.int32)
        left[:n_int] = 2 * idx + 1
        right[:n_int] = 2 * idx + 2
        return cls(_flat=(fid, value, left, right))

    def _validate_and_measure(self):
        n = self.fid.shape[0]
        if n == 0:
            raise ModelSemanticError("empty tree")
        if not (self.value.shape == self.left.shape == self.right.shape == (n,)):
            raise ModelSemanticError("flat tree arrays differ in length")
        internal = self.fid >= 0
        if np.any(self.fid < -1):
            raise ModelSemanticError("feature id must be non-negative")
        if not np.all(np.isfinite(self.value)):
            bad = int(np.flatnonzero(~np.isfinite(self.value))[0])
            what = "threshold" if internal[bad] else "leaf value"
            raise ModelSemanticError(f"{what} must be finite (node {bad})")
        kids = np.concatenate([self.left[internal], self.right[internal]])
        if kids.size and (kids.min() < 0 or kids.max() >= n):
            raise ModelSemanticError("child id out of range")
        if np.any(kids == 0):
            raise ModelSemanticError("root must not appear as a child")
        counts = np.bincount(kids, minlength=n) if kids.size else np.zeros(n, np.int64)
        if np.any(counts > 1):
            raise ModelSemanticError("node appears twice in the same tree")
        # Breadth-first depth labelling; with unique parents and a parentless
        # root, every node reached exactly once means no cycles.
        depth = np.full(n, -1, dtype=np.int64)
        depth[0] = 0
        frontier = np.array([0], dtype=np.int64)
        seen = 1
        level = 0
        while frontier.size:
            inner = frontier[internal[frontier]]
            nxt = np.concatenate([self.left[inner], self.right[inner]]).astype(np.int64)
            level += 1
            if nxt.size:
                if np.any(depth[nxt] >= 0):
                    raise ModelSemanticError("cycle in tree")
                depth[nxt] = level
                seen += nxt.size
            frontier = nxt
        if seen != n:
            raise ModelSemanticError("node unreachable from the root")
        leaves = ~internal
        self.depth = int(depth[leaves].max())
        self.leaf_count = int(leaves.sum())
        self.node_count = int(n)
        self.max_fid = int(self.fid.max()) if internal.any() else -1

    # -- reference-compatible views -----------------------------------------------

    @property
    def root(self) -> Node:
        if self._root is None:
            nodes = [None] * self.node_count
            order = _bfs_order(self.fid, self.left, self.right)
            for i in reversed(order):
                if self.fid[i] < 0:
                    nodes[i] = Node(-1, 0.0, float(self.value[i]), None, None)
                else:
                    nodes[i] = Node(int(self.fid[i]), float(self.value[i]), 0.0,
                                    nodes[self.left[i]], nodes[self.right[i]])
            self._root = nodes[0]
        return self._root

    def leaf_ordinals(self) -> np.ndarray:
        """Left-to-right ordinal of every leaf node id (-1 for internal ids)."""
        if self._leaf_ord is None:
            ords = np.full(self.node_count, -1, dtype=np.int64)
            k = 0
            stack = [0]
            while stack:
                i = stack.pop()
                if self.fid[i] < 0:
                    ords[i] = k
                    k += 1
                else:
                    stack.append(int(self.right[i]))
                    stack.append(int(self.left[i]))
            self._leaf_ord = ords
        return self._leaf_ord

    def leaf_ordinal(self, node) -> int:
        """Left-to-right index of a leaf (a node id or a Node of ``root``)."""
        if isinstance(node, (int, np.integer)):
            return int(self.leaf_ordinals()[int(node)])
        # Locate the Node object in the materialised graph.
        root = self.root
        k = 0
        stack = [root]
        while stack:
            cur = stack.pop()
            if cur.left is None:
                if cur is node:
                    return k
                k += 1
            else:
                stack.append(cur.right)
                stack.append(cur.left)
        raise KeyError("node is not a leaf of this tree")

    def __repr__(self):
        return (f"Tree(depth={self.depth}, leaves={self.leaf_count}, "
                f"nodes={self.node_count})")


def _bfs_order(fid, left, right):
    order = []
    q = deque([0])
    while q:
        i = q.popleft()
        order.append(i)
        if fid[i] >= 0:
            q.append(int(left[i]))
            q.append(int(right[i]))
    return order


def _flatten_graph(root):
    """Node graph (ours or the reference's) -> flat BFS arrays."""
    fid, value, left, right = [], [], [], []
    ids = {}
    q = deque([root])
    ids[id(root)] = 0
    order = []
    while q:
        node = q.popleft()
        order.append(node)
        if node.left is not None:
            for child in (node.left, node.right):
                if child is None:
                    raise ModelSemanticError("internal node requires exactly two child nodes")
                if id(child) in ids:
                    raise ModelSemanticError("node appears twice in the same tree")
                ids[id(child)] = len(ids)
                q.append(child)
    for node in order:
        if node.left is None:
            fid.append(-1)
            value.append(node.value)
            left.append(-1)
            right.append(-1)
        else:
            fid.append(int(node.fid))
            value.append(node.threshold)
            left.append(ids[id(node.left)])
            right.append(ids[id(node.right)])
    with np.errstate(over="ignore"):
        value32 = np.asarray(value, dtype=np.float64).astype(np.float32)
    return (np.asarray(fid, np.int32), value32,
            np.asarray(left, np.int32), np.asarray(right, np.int32))


class FlatModel(NamedTuple):
    """A whole ensemble as concatenated flat arrays (the C ABI's ts_model_desc).

    Nodes of tree ``t`` are ``[tree_off[t], tree_off[t+1])`` with tree-local
    ids, root at 0; ``fid == -1`` marks a leaf; ``value`` is the fp32
    threshold or leaf value.  Building one directly (see ``synth``) skips
    per-tree Python objects for very large ensembles; the native packer
    validates it exactly as ``Tree``/``Ensemble`` would.
    """

    num_features: int
    tree_off: np.ndarray   # int64 [T+1]
    weight: np.ndarray     # float64 [T]
    fid: np.ndarray        # int32 [n]
    value: np.ndarray      # float32 [n]
    left: np.ndarray       # int32 [n]
    right: np.ndarray      # int32 [n]

    @property
    def num_trees(self) -> int:
        return len(self.tree_off) - 1

    def arrays(self):
        """``(tree_off, weight, fid, value, left, right)``."""
        return tuple(self[1:])

    def subset(self, t0: int, t1: int) -> "FlatModel":
        """Trees ``[t0, t1)`` as their own FlatModel (a tree shard)."""
        if not 0 <= t0 < t1 <= self.num_trees:
            raise ValueError(f"bad tree range [{t0}, {t1}) of {self.num_trees}")
        a, b = int(self.tree_off[t0]), int(self.tree_off[t1])
        return FlatModel(self.num_features, self.tree_off[t0:t1 + 1] - a,
                         self.weight[t0:t1], self.fid[a:b], self.value[a:b], self.left[a:b],
                         self.right[a:b])

    def depths(self) -> np.ndarray:
        """Depth of every tree (longest root-to-leaf edge count)."""
        out = np.zeros(self.num_trees, np.int64)
        for t in range(self.num_trees):
            a, b = int(self.tree_off[t]), int(self.tree_off[t + 1])
            fid, lc, rc = self.fid[a:b], self.left[a:b], self.right[a:b]
            level = np.array([0])
            d = 0
            while True:
                inner = level[fid[level] >= 0]
                if inner.size == 0:
                    break
                level = np.concatenate([lc[inner], rc[inner]])
                d += 1
            out[t] = d
        return out

    def to_ensemble(self) -> "Ensemble":
        trees = []
        for t in range(self.num_trees):
            a, b = int(self.tree_off[t]), int(self.tree_off[t + 1])
            trees.append((Tree(_flat=(self.fid[a:b], self.value[a:b], self.left[a:b],
                                      self.right[a:b])), float(self.weight[t])))
        return Ensemble(self.num_features, trees)


class Ensemble:
    """Ordered weighted trees over ``num_features`` dense fp32 features.

    ``trees`` is a tuple of ``(Tree, weight)`` with float64 weights.  Entries
    may be given as ``Tree``, ``Node`` (root), ``(tree_or_root, weight)``, or
    reference ``treescore`` trees (duck-typed on ``.root``).
    """

    __slots__ = ("num_features", "trees", "_flat")

    def __init__(self, num_features: int, trees: Iterable):
        num_features = int(num_features)
        if num_features < 1:
            raise ModelSemanticError("num_features must be positive")
        out = []
        for entry in trees:
            if isinstance(entry, (tuple, list)):
                tree, weight = entry
            else:
                tree, weight = entry, 1.0
            tree = _as_tree(tree)
            weight = float(weight)
            if not math.isfinite(weight):
                raise ModelSemanticError(f"tree weight must be finite, got {weight!r}")
            if tree.max_fid >= num_features:
                raise ModelSemanticError(
                    f"feature id {tree.max_fid} out of range (num_features={num_features})")
            out.append((tree, weight))
        if not out:
            raise ModelSemanticError("ensemble must contain at least one tree")
        self.num_features = num_features
        self.trees = tuple(out)
        self._flat = None

    @classmethod
    def from_reference(cls, ref_ensemble) -> "Ensemble":
        """Adopt a reference ``treescore.Ensemble`` (same order and weights)."""
        return cls(ref_ensemble.num_features,
                   [(t.root, w) for t, w in ref_ensemble.trees])

    def flat(self) -> "FlatModel":
        """Concatenated flat arrays for the native packer (cached)."""
        if self._flat is None:
            sizes = np.array([t.node_count for t, _ in self.trees], dtype=np.int64)
            off = np.zeros(len(sizes) + 1, dtype=np.int64)
            np.cumsum(sizes, out=off[1:])
            w = np.array([w for _, w in self.trees], dtype=np.float64)
            cat = lambda name, dt: np.ascontiguousarray(
                np.concatenate([getattr(t, name) for t, _ in self.trees]), dtype=dt)
            self._flat = FlatModel(self.num_features, off, w, cat("fid", np.int32),
                                   cat("value", np.float32), cat("left", np.int32),
                                   cat("right", np.int32))
        return self._flat

    def __len__(self):
        return len(self.trees)

    def __repr__(self):
        return f"Ensemble(num_features={self.num_features}, trees={len(self.trees)})"


def _as_tree(obj) -> Tree:
    if isinstance(obj, Tree):
        return obj
    if isinstance(obj, Node) or _is_foreign_node(obj):
        return Tree(obj)
    if hasattr(obj, "root"):  # reference treescore.Tree
        return Tree(obj.root)
    raise ModelSemanticError("tree entry must be a Tree or a Node")


class TreeStats(NamedTuple):
    """Depth/leaf statistics of an ensemble (ref ``model.py:229-233``)."""

    avg_depth: float
    max_depth: int
    avg_leaves: float


def tree_stats(ensemble: Ensemble) -> TreeStats:
    """Averaged over the ensemble's trees, as ref ``model.py:236-244``."""
    depths = [t.depth for t, _ in ensemble.trees]
    leaves = [t.leaf_count for t, _ in ensemble.trees]
    return TreeStats(sum(depths) / len(depths), max(depths), sum(leaves) / len(leaves))


# ---------------------------------------------------------------------------
# Scalar semantics (the rule every path shares)
# ---------------------------------------------------------------------------

def traverse_to_leaf(root, x):
    """Walk a Node graph: left iff ``x[fid] < threshold``; ties go right."""
    node = root
    while node.left is not None:
        node = node.left if float(x[node.fid]) < node.threshold else node.right
    return node


def reference_predict(ensemble: Ensemble, x) -> float:
    """f64 ``acc += weight * leaf`` in tree order over flat trees."""
    acc = 0.0
    for tree, weight in ensemble.trees:
        i = 0
        fid, val, lft, rgt = tree.fid, tree.value, tree.left, tree.right
        while fid[i] >= 0:
            i = lft[i] if float(x[fid[i]]) < float(val[i]) else rgt[i]
        acc += weight * float(val[i])
    return acc


# ---------------------------------------------------------------------------
# Complete-table expansion (the packer's specification)
# ---------------------------------------------------------------------------

class CompleteTree:
    """Breadth-first complete tables: children of ``i`` at ``2i+1``/``2i+2``."""

    __slots__ = ("depth", "fids", "thetas", "leaf_values")

    def __init__(self, depth: int, fids, thetas, leaf_values):
        self.depth = int(depth)
        self.fids = np.ascontiguousarray(fids, dtype=np.int32)
        self.thetas = np.ascontiguousarray(thetas, dtype=np.float32)
        self.leaf_values = np.ascontiguousarray(leaf_values, dtype=np.float32)
        n_int = (1 << self.depth) - 1
        if self.fids.shape != (n_int,) or self.thetas.shape != (n_int,):
            raise ModelSemanticError("node table size does not match depth")
        if self.leaf_values.shape != (1 << self.depth,):
            raise ModelSemanticError("leaf table size does not match depth")
        for a in (self.fids, self.thetas, self.leaf_values):
            a.flags.writeable = False

    @property
    def internal_count(self) -> int:
        return (1 << self.depth) - 1

    @property
    def table_entries(self) -> int:
        return (1 << (self.depth + 1)) - 1

    def __repr__(self):
        return f"CompleteTree(depth={self.depth})"


def expand_to_complete(tree: Tree) -> CompleteTree:
    """Expand to a complete tree of the tree's own depth (level by level).

    An early leaf at depth ``k`` becomes a dummy subtree: internal slots get
    ``(DUMMY_FID, +inf)`` and all ``2^(d-k)`` leaves below repeat its value.
    """
    tree = _as_tree(tree)
    d = tree.depth
    if d > MAX_DEPTH:
        raise DepthLimitError(
            f"tree depth {d} exceeds MAX_DEPTH={MAX_DEPTH} for complete-table layouts")
    n_int = (1 << d) - 1
    fids = np.full(n_int, DUMMY_FID, dtype=np.int32)
    thetas = np.full(n_int, DUMMY_THETA, dtype=np.float32)
    # src[k] = logical node occupying heap slot k of the current level.
    src = np.zeros(1, dtype=np.int64)
    for level in range(d):
        base = (1 << level) - 1
        inner = tree.fid[src] >= 0
        slots = base + np.arange(src.size)
        fids[slots[inner]] = tree.fid[src[inner]]
        thetas[slots[inner]] = tree.value[src[inner]]
        nxt = np.empty(2 * src.size, dtype=np.int64)
        nxt[0::2] = np.where(inner, tree.left[src], src)
        nxt[1::2] = np.where(inner, tree.right[src], src)
        src = nxt
    leaves = tree.value[src].astype(np.float32)
    return CompleteTree(d, fids, thetas, leaves)


# ---------------------------------------------------------------------------
# Text model format
# ---------------------------------------------------------------------------

def _fmt(x: float) -> str:
    return repr(float(x))


def serialize_model(ensemble: Ensemble) -> str:
    """Canonical text: BFS node ids, shortest round-trip float literals."""
    out = [f"ensemble {ensemble.num_features} {len(ensemble.trees)}"]
    for tree, weight in ensemble.trees:
        out.append(f"tree {_fmt(weight)}")
        order = _bfs_order(tree.fid, tree.left, tree.right)
        new_id = {old: k for k, old in enumerate(order)}
        for k, i in enumerate(order):
            if tree.fid[i] < 0:
                out.append(f"leaf {k} {_fmt(tree.value[i])}")
            else:
                out.append(f"node {k} {int(tree.fid[i])} {_fmt(tree.value[i])} "
                           f"{new_id[int(tree.left[i])]} {new_id[int(tree.right[i])]}")
        out.append("end")
    return "\n".join(out) + "\n"


def _lines(text: str):
    for lineno, raw in enumerate(text.splitlines(), 1):
        body = raw.lstrip()
        if not body or body.startswith("#"):
            continue
        toks = []
        col = 0
        for part in raw.split():
            col = raw.index(part, col)
            toks.append((part, col + 1))
            col += len(part)
        yield lineno, toks


def _int(tok, what, line):
    try:
        return int(tok[0])
    except ValueError:
        raise ModelSyntaxError(f"expected integer {what}, got {tok[0]!r}", line, tok[1])


def _float(tok, what, line):
    try:
        return float(tok[0])
    except ValueError:
        raise ModelSyntaxError(f"expected float {what}, got {tok[0]!r}", line, tok[1])


def parse_model(text: str) -> Ensemble:
    """Parse the text format into a validated :class:`Ensemble`.

    Error classes and messages follow ref ``model.py:416-602``: syntax errors
    carry line/column, semantic errors name the tree and node id.
    """
    it = _lines(text)
    nxt = lambda: next(it, None)
    entry = nxt()
    if entry is None:
        raise ModelSyntaxError("empty document, expected 'ensemble' header", 1, 1)
    line, toks = entry
    if toks[0][0] != "ensemble" or len(toks) != 3:
        raise ModelSyntaxError("expected header 'ensemble <num_features> <num_trees>'",
                               line, toks[0][1])
    nf = _int(toks[1], "num_features", line)
    nt = _int(toks[2], "num_trees", line)
    if nf < 1:
        raise ModelSemanticError(f"num_features must be positive, got {nf}")
    if nt < 1:
        raise ModelSemanticError(f"num_trees must be positive, got {nt}")
    trees = []
    last = line
    for t in range(nt):
        entry = nxt()
        if entry is None:
            raise ModelSyntaxError(f"expected {nt} tree blocks, found {t}", last, 1)
        line, toks = entry
        last = line
        if toks[0][0] != "tree" or len(toks) != 2:
            raise ModelSyntaxError("expected 'tree <weight>'", line, toks[0][1])
        weight = _float(toks[1], "weight", line)
        defs = {}
        while True:
            entry = nxt()
            if entry is None:
                raise ModelSyntaxError(f"tree {t}: missing 'end'", last, 1)
            line, toks = entry
            last = line
            word, c0 = toks[0]
            if word == "end":
                if len(toks) != 1:
                    raise ModelSyntaxError("unexpected tokens after 'end'", line, toks[1][1])
                break
            if word == "node":
                if len(toks) != 6:
                    raise ModelSyntaxError(
                        "expected 'node <id> <fid> <theta> <left> <right>'", line, c0)
                nid = _int(toks[1], "node id", line)
                fid = _int(toks[2], "feature id", line)
                theta = _float(toks[3], "threshold", line)
                lc = _int(toks[4], "left child id", line)
                rc = _int(toks[5], "right child id", line)
                if fid < 0:
                    raise ModelSyntaxError("feature id must be non-negative", line, toks[2][1])
                if fid >= nf:
                    raise ModelSemanticError(
                        f"tree {t}, line {line}: feature id {fid} out of range "
                        f"(num_features={nf})")
                if not math.isfinite(_narrow(theta)):
                    raise ModelSemanticError(f"tree {t}, line {line}: threshold must be finite")
                payload = (fid, theta, lc, rc)
            elif word == "leaf":
                if len(toks) != 3:
                    raise ModelSyntaxError("expected 'leaf <id> <value>'", line, c0)
                nid = _int(toks[1], "node id", line)
                value = _float(toks[2], "leaf value", line)
                if not math.isfinite(_narrow(value)):
                    raise ModelSemanticError(f"tree {t}, line {line}: leaf value must be finite")
                payload = (-1, value, -1, -1)
            else:
                raise ModelSyntaxError(f"expected 'node', 'leaf' or 'end', got {word!r}",
                                       line, c0)
            if nid < 0:
                raise ModelSyntaxError("node id must be non-negative", line, toks[1][1])
            if nid in defs:
                raise ModelSemanticError(f"tree {t}: duplicate node id {nid}")
            defs[nid] = payload
        trees.append((_tree_from_defs(t, defs), weight))
    entry = nxt()
    if entry is not None:
        raise ModelSyntaxError("unexpected content after final tree", entry[0], entry[1][0][1])
    return Ensemble(nf, trees)


def _tree_from_defs(t: int, defs: dict) -> Tree:
    n = len(defs)
    if n == 0:
        raise ModelSemanticError(f"tree {t}: empty tree block")
    if set(defs) != set(range(n)):
        missing = min(set(range(n)) - set(defs))
        raise ModelSemanticError(
            f"tree {t}: node ids must be dense in [0, {n}), id {missing} is missing")
    refs = [0] * n
    for nid in range(n):
        fid, _, lc, rc = defs[nid]
        if fid < 0:
            continue
        for c in (lc, rc):
            if c not in defs:
                raise ModelSemanticError(
                    f"tree {t}: node {nid} references dangling child id {c}")
            refs[c] += 1
    if refs[0]:
        raise ModelSemanticError(f"tree {t}: root (id 0) must not appear as a child")
    for nid in range(1, n):
        if refs[nid] > 1:
            raise ModelSemanticError(f"tree {t}: node {nid} has multiple parents")
    seen = set()
    q = deque([0])
    while q:
        i = q.popleft()
        if i in seen:
            continue
        seen.add(i)
        fid, _, lc, rc = defs[i]
        if fid >= 0:
            q.append(lc)
            q.append(rc)
    if len(seen) != n:
        orphan = min(set(defs) - seen)
        raise ModelSemanticError(
            f"tree {t}: node {orphan} is unreachable from the root "
            "(disconnected or cyclic block)")
    arr = np.array([defs[i] for i in range(n)], dtype=object)
    return Tree.from_arrays(arr[:, 0].astype(np.int64), arr[:, 1].astype(np.float64),
                            arr[:, 2].astype(np.int64), arr[:, 3].astype(np.int64))


def parse_model_native(text) -> FlatModel:
    """Parse with the native parser (``ts_parse_model``) straight to a
    :class:`FlatModel` -- no per-node Python objects (config 4b's 20,000-tree
    files).  Same errors as :func:`parse_model`."""
    import ctypes
    from . import _lib
    lib = _lib.load()
    data = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    out = ctypes.POINTER(_lib.FlatModelC)()
    rc = lib.ts_parse_model(data, len(data), ctypes.byref(out))
    try:
        if rc == _lib.TS_ERR_SYNTAX:
            msg = _lib.last_error()
            msg = msg.split(": ", 1)[1] if msg.startswith("line ") else msg
            raise ModelSyntaxError(msg, out.contents.err_line, out.contents.err_col)
        if rc == _lib.TS_ERR_INVALID:
            raise ModelSemanticError(_lib.last_error())
        if rc != _lib.TS_OK:
            raise ModelError(f"ts_parse_model failed ({rc}): {_lib.last_error()}")
        m = out.contents
        T, n = m.num_trees, m.num_nodes
        arr = lambda p, k, dt: np.ctypeslib.as_array(p, shape=(max(k, 1),))[:k].astype(dt)
        return FlatModel(int(m.num_features), arr(m.tree_node_offset, T + 1, np.int64),
                         arr(m.tree_weight, T, np.float64), arr(m.node_fid, n, np.int32),
                         arr(m.node_value, n, np.float32), arr(m.node_left, n, np.int32),
                         arr(m.node_right, n, np.int32))
    finally:
        if out:
            lib.ts_flat_free(out)


def load_flat_model(path) -> FlatModel:
    """Read a model file with the native parser (see parse_model_native)."""
    with open(path, "rb") as fh:
        return parse_model_native(fh.read())


def load_model(path) -> Ensemble:
    with open(path, "r", encoding="utf-8") as fh:
        return parse_model(fh.read())


def save_model(ensemble: Ensemble, path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(serialize_model(ensemble))
