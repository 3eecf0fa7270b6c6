"""Pin the CPU oracle (numpy and C restatements) to the reference's outputs.

The golden vectors were produced by the reference package itself
(tests/golden/make_golden.py); the known-answer cases below restate the
reference's own tests (cited per test)."""

import numpy as np
import pytest

import oracle
from paper_1212_2287_b200 import Ensemble, Node, Tree
from conftest import GOLDEN_CASES, load_golden


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_numpy_oracle_matches_reference(name):
    ens, g = load_golden(name)
    arrays = ens.flat().arrays()
    tables = oracle.expand(arrays)
    assert [t[0] for t in tables] == g["depths"].tolist()
    ords = oracle.ordinals(tables, g["X"])
    assert np.array_equal(ords, g["ordinals"])
    scores = oracle.score(tables, arrays[1], g["X"], ords)
    assert np.array_equal(scores, g["scores"])          # bit-exact f64
    assert np.array_equal(scores, g["scores_vpred"])


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_c_oracle_matches_reference(name):
    ens, g = load_golden(name)
    c = oracle.COracle(ens.flat().arrays())
    for threads, v in ((1, 1), (3, 16), (8, 64)):
        s, o = c.score(g["X"], threads=threads, with_ordinals=True, v=v)
        assert np.array_equal(s, g["scores"])
        assert np.array_equal(o.astype(np.int64), g["ordinals"])
    assert np.array_equal(c.score_linked(g["X"]), g["scores"])


@pytest.mark.parametrize("name", ["mixed", "deep_unbalanced", "trivia"])
def test_linked_walk_matches_reference(name):
    ens, g = load_golden(name)
    assert np.array_equal(oracle.score_linked(ens.flat().arrays(), g["X"]), g["scores"])


def test_tie_goes_right_known_answer():
    # ref tests/test_model.py:73-78, tests/test_evaluators.py:182-187
    ens = Ensemble(1, [Tree(Node.internal(0, 0.5, Node.leaf(-1.0), Node.leaf(1.0)))])
    c = oracle.COracle(ens.flat().arrays())
    X = np.array([[0.3], [0.5], [0.7], [0.4999]], np.float32)
    s, o = c.score(X, threads=1, with_ordinals=True)
    assert s.tolist() == [-1.0, 1.0, 1.0, -1.0]
    assert o[0].tolist() == [0, 1, 1, 0]


def test_unbalanced_predicated_ordinals_known_answer():
    # ref tests/test_model.py:153-176: the 3-leaf tree's predicated ordinals
    # are {0, 2, 3} (dummy routes left), its logical ordinals {0, 1, 2}.
    tree = Tree(Node.internal(0, 0.5, Node.leaf(1.0),
                              Node.internal(1, 0.25, Node.leaf(2.0), Node.leaf(3.0))))
    tables = oracle.expand(Ensemble(2, [tree]).flat().arrays())
    d, fids, thetas, leaves = tables[0]
    assert d == 2 and fids[1] == 0 and np.isinf(thetas[1])
    assert leaves.tolist() == [1.0, 1.0, 2.0, 3.0]
    X = np.array([[0.1, 0.1], [0.1, 0.9], [0.9, 0.1], [0.9, 0.9]], np.float32)
    assert oracle.ordinals(tables, X)[0].tolist() == [0, 0, 2, 3]


def test_f64_accumulation_order_is_tree_order():
    # acc = ((0 + w0*l0) + w1*l1) + w2*l2 in f64 (ref evaluators.py:529-535);
    # these values are chosen so another order gives a different last bit.
    leaves = [1e16, 1.0, -1e16]
    trees = [(Tree(Node.leaf(v)), 1.0) for v in leaves]
    ens = Ensemble(1, trees)
    c = oracle.COracle(ens.flat().arrays())
    s = c.score(np.zeros((1, 1), np.float32), threads=1)
    expected = 0.0
    for v in leaves:
        expected += float(np.float32(v))
    assert s[0] == expected


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_trace_oracle_matches_reference(name):
    ens, g = load_golden(name)
    bits, leaves = oracle.trace(ens.flat().arrays(), g["X"])
    assert np.array_equal(bits, g["trace_bits"])
    assert np.array_equal(leaves, g["trace_leaves"])
    counts = np.unpackbits(bits.view(np.uint8), axis=1, bitorder="little").sum(axis=1)
    frac = counts / g["X"].shape[1]
    assert frac.mean() == g["coverage"][0] and frac.var() == g["coverage"][1]
