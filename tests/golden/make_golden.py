"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

For every case this writes ``<case>.model.txt`` (the reference's
``serialize_model`` output) and ``<case>.npz`` holding:

* ``X``            float32 [n, f] instances
* ``scores``       float64 [n]    ``treescore.reference_batch`` (linked walk,
                                  ``evaluators.py:623-629``)
* ``scores_vpred`` float64 [n]    ``build(ens, "vpredicated", 16).predict_batch``
                                  (``evaluators.py:479-550``)
* ``ordinals``     int32 [T, n]   per-tree predicated leaf ordinals:
                                  ``batch_kernel(d)`` on ``expand_to_complete``
                                  (``evaluators.py:90-99``, ``model.py:315-349``)
* ``depths``       int32 [T]
* ``trace_bits``   uint32 [n, ceil(f/32)]  ``predict_ensemble_traced`` visited
                                  feature ids as bitsets (``evaluators.py:599-620``)
* ``trace_leaves`` int32 [T, n]   its logical left-to-right leaf ordinals
* ``coverage``     float64 [2]    ``measure_feature_coverage`` mean, variance
                                  (``bench.py:412-427``)

The GPU parity tests and the oracle tests read these files; the reference is
never needed at test time (it does not exist on the GPU box).
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

import treescore as ts  # noqa: E402
from treescore.evaluators import batch_kernel  # noqa: E402
from treescore.synth import GenConfig, gen_tree  # noqa: E402


def rand_unbalanced(rng, max_depth, f, prune=0.35, leaf=lambda r: r.random()):
    def build(level):
        if level == max_depth or (level > 0 and rng.random() < prune):
            return ts.Node.leaf(leaf(rng))
        return ts.Node.internal(int(rng.integers(f)), rng.random(), build(level + 1),
                                build(level + 1))
    return ts.Tree(build(0))


def chain(depth, f=2):
    node = ts.Node.leaf(1.0)
    for level in range(depth):
        node = ts.Node.internal(level % f, 0.5 / (level + 2), node, ts.Node.leaf(2.0 + level))
    return ts.Tree(node)


def complete(rng, d, f, thr=lambda r: r.random(), leaf=lambda r: r.standard_normal()):
    def build(level):
        if level == d:
            return ts.Node.leaf(leaf(rng))
        return ts.Node.internal(int(rng.integers(f)), thr(rng), build(level + 1),
                                build(level + 1))
    return ts.Tree(build(0))


def save(name, ens, X):
    X = np.ascontiguousarray(X, dtype=np.float32)
    scores = ts.reference_batch(ens, X)
    vpred = ts.build(ens, "vpredicated", 16).predict_batch(X)
    assert np.array_equal(scores, vpred), name
    T = len(ens.trees)
    ords = np.empty((T, X.shape[0]), np.int32)
    depths = np.empty(T, np.int32)
    rows = np.arange(X.shape[0])
    for t, (tree, _w) in enumerate(ens.trees):
        ct = ts.expand_to_complete(tree)
        depths[t] = ct.depth
        if ct.depth == 0:
            ords[t] = 0
        else:
            ords[t] = batch_kernel(ct.depth)(ct.fids, ct.thetas, X, rows)
    words = (X.shape[1] + 31) // 32
    tbits = np.zeros((X.shape[0], words), np.uint32)
    tleaves = np.empty((T, X.shape[0]), np.int32)
    for i in range(X.shape[0]):
        tr = ts.predict_ensemble_traced(ens, X[i])
        assert tr.score == scores[i]
        for fid in tr.visited_features:
            tbits[i, fid >> 5] |= np.uint32(1 << (fid & 31))
        tleaves[:, i] = tr.visited_leaves
    cov = ts.measure_feature_coverage(ens, ts.Dataset(X))
    with open(os.path.join(HERE, f"{name}.model.txt"), "w") as fh:
        fh.write(ts.serialize_model(ens))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), X=X, scores=scores,
                        scores_vpred=vpred, ordinals=ords, depths=depths, trace_bits=tbits,
                        trace_leaves=tleaves,
                        coverage=np.array([cov.mean_fraction, cov.variance]))
    print(f"{name}: T={T} n={X.shape[0]} f={X.shape[1]} depths={sorted(set(depths.tolist()))}")


def main():
    # 1. tie goes right (ref tests/test_evaluators.py:182-187, test_model.py:73-78)
    ens = ts.Ensemble(1, [ts.Tree(ts.Node.internal(0, 0.5, ts.Node.leaf(-1.0),
                                                    ts.Node.leaf(1.0)))])
    save("tie", ens, np.array([[0.3], [0.5], [0.7], [0.4999], [np.float32(0.5)]]))

    # 2. unbalanced 3-leaf tree (ref tests/test_model.py:153-168): predicated
    #    ordinals {0, 2, 3} vs logical {0, 1, 2}
    ens = ts.Ensemble(2, [ts.Tree(ts.Node.internal(
        0, 0.5, ts.Node.leaf(1.0),
        ts.Node.internal(1, 0.25, ts.Node.leaf(2.0), ts.Node.leaf(3.0))))])
    save("unbalanced3", ens, np.array([[a, b] for a in (0.1, 0.5, 0.9)
                                       for b in (0.1, 0.25, 0.9)]))

    # 3. mixed ensemble in the style of ref tests/conftest.py:28-42 (balanced
    #    generator trees + pruned trees, weights U(0.5,1.5), depth-0 trees)
    rng = np.random.default_rng(2026)
    trees = []
    for t in range(40):
        if t % 2:
            tree = rand_unbalanced(rng, 7, 32)
        else:
            tree = gen_tree(GenConfig(depth=int(rng.integers(0, 8)), num_features=32,
                                      seed=int(rng.integers(2 ** 31))))
        trees.append((tree, float(rng.uniform(0.5, 1.5))))
    save("mixed", ts.Ensemble(32, trees), rng.random((700, 32), dtype=np.float32))

    # 4. config-0 shape in miniature: complete depth-6 trees, F=136, N(0,1) leaves
    rng = np.random.default_rng(0)
    trees = [complete(rng, 6, 136) for _ in range(24)]
    save("complete_d6", ts.Ensemble(136, trees), rng.random((1024, 136), dtype=np.float32))

    # 5. exact ties everywhere: integer counts with integer thresholds (config 1 style)
    rng = np.random.default_rng(1)
    trees = [complete(rng, 5, 12, thr=lambda r: float(r.integers(0, 6)),
                      leaf=lambda r: 0.1 * r.standard_normal()) for _ in range(30)]
    X = rng.integers(0, 6, size=(600, 12)).astype(np.float32)
    save("ties_counts", ts.Ensemble(12, trees), X)

    # 6. deep and unbalanced, up to MAX_DEPTH (chains and pruned trees, d in 9..16)
    rng = np.random.default_rng(6)
    trees = [(chain(16, 3), 1.0), (chain(11, 3), 0.75)]
    trees += [(rand_unbalanced(rng, int(rng.integers(9, 17)), 8, prune=0.45),
               float(rng.uniform(0.5, 1.5))) for _ in range(10)]
    save("deep_unbalanced", ts.Ensemble(8, trees), rng.random((300, 8), dtype=np.float32))

    # 7. trivia: single leaves, zero weights, negative zero leaves, negative weights
    trees = [(ts.Tree(ts.Node.leaf(1.5)), 2.0), (ts.Tree(ts.Node.leaf(-0.0)), 1.0),
             (ts.Tree(ts.Node.internal(1, 0.5, ts.Node.leaf(-0.0), ts.Node.leaf(0.0))), -1.0),
             (complete(np.random.default_rng(7), 3, 4), 0.0),
             (complete(np.random.default_rng(8), 2, 4), -0.5)]
    save("trivia", ts.Ensemble(4, trees),
         np.random.default_rng(9).random((64, 4), dtype=np.float32))

    # 8. thresholds not representable in f32 (narrowing) and subnormals (no FTZ)
    tiny = float(np.float32(1e-40))            # a float32 subnormal
    ens = ts.Ensemble(3, [
        ts.Tree(ts.Node.internal(0, 0.1, ts.Node.leaf(0.1), ts.Node.leaf(0.2))),
        ts.Tree(ts.Node.internal(1, tiny, ts.Node.leaf(1.0),
                                 ts.Node.internal(2, -tiny, ts.Node.leaf(2.0),
                                                  ts.Node.leaf(3.0)))),
        ts.Tree(ts.Node.internal(1, 0.0, ts.Node.leaf(4.0), ts.Node.leaf(5.0))),
    ])
    vals = [0.0, -0.0, tiny, -tiny, 2 * tiny, float(np.float32(0.1)),
            float(np.nextafter(np.float32(0.1), np.float32(0))), 0.1, 1.0]
    X = np.array([[a, b, c] for a in vals for b in vals for c in (vals[0], vals[2], vals[3])],
                 dtype=np.float32)
    save("narrow_subnormal", ens, X)

    # 9. wide features (config 3 style): F=700, zipf fids, 40% exact zeros,
    #    unbalanced 64-leaf trees grown by random leaf splits
    rng = np.random.default_rng(3)
    ranks = np.arange(1, 701, dtype=np.float64)
    p = ranks ** -1.1
    p /= p.sum()
    trees = []
    for _ in range(16):
        leaves = [ts.Node.leaf(0.05 * rng.standard_normal())]
        depth_of = {id(leaves[0]): 0}
        parent = {}
        while len(leaves) < 64:
            cand = [lf for lf in leaves if depth_of[id(lf)] < 16]
            victim = cand[int(rng.integers(len(cand)))]
            a = ts.Node.leaf(0.05 * rng.standard_normal())
            b = ts.Node.leaf(0.05 * rng.standard_normal())
            inner = ts.Node.internal(int(rng.choice(700, p=p)), rng.random(), a, b)
            dd = depth_of[id(victim)]
            depth_of[id(a)] = depth_of[id(b)] = dd + 1
            if id(victim) in parent:
                par, side = parent[id(victim)]
                setattr(par, side, inner)
                parent[id(inner)] = (par, side)
            else:
                root = inner
            parent[id(a)] = (inner, "left")
            parent[id(b)] = (inner, "right")
            leaves.remove(victim)
            leaves += [a, b]
        trees.append((ts.Tree(root), 1.0))
    X = rng.random((256, 700), dtype=np.float32)
    X[rng.random(X.shape) < 0.4] = 0.0
    save("wide_irregular", ts.Ensemble(700, trees), X)

    # 10. config-1 shape in miniature: F=136 with uniform, lognormal and
    #     integer-count columns, complete depth-8 trees whose thresholds are
    #     values of the split column in a sample of rows (exact ties occur)
    rng = np.random.default_rng(10)
    kinds = rng.permutation(np.array([0] * 95 + [1] * 27 + [2] * 14))
    X = np.empty((512, 136), np.float32)
    for c, kind in enumerate(kinds):
        if kind == 0:
            X[:, c] = rng.random(512, dtype=np.float32)
        elif kind == 1:
            X[:, c] = rng.lognormal(0.0, 1.0, 512).astype(np.float32)
        else:
            X[:, c] = rng.integers(0, 51, 512).astype(np.float32)
    trees = []
    for _ in range(12):
        def build(level):
            if level == 8:
                return ts.Node.leaf(0.1 * rng.standard_normal())
            fid = int(rng.integers(136))
            return ts.Node.internal(fid, float(X[int(rng.integers(512)), fid]),
                                    build(level + 1), build(level + 1))
        trees.append(ts.Tree(build(0)))
    save("cfg1_ties_d8", ts.Ensemble(136, trees), X)


if __name__ == "__main__":
    main()
