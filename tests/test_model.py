"""Model layer: the reference's model-format and expansion contracts
(ref tests/test_model.py), on the flat representation the packer consumes."""

import math

import numpy as np
import pytest

import oracle
from paper_1212_2287_b200 import (DepthLimitError, Ensemble, MAX_DEPTH, ModelSemanticError,
                                  ModelSyntaxError, Node, Tree, expand_to_complete,
                                  parse_model, reference_predict, serialize_model,
                                  traverse_to_leaf, tree_stats)
from conftest import GOLDEN_CASES, GOLDEN_DIR, load_golden


def chain_tree(depth):
    node = Node.leaf(1.0)
    for level in range(depth):
        node = Node.internal(0, 0.5 / (level + 2), node, Node.leaf(2.0))
    return Tree(node)


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_serialize_is_byte_identical_to_reference(name):
    # the .model.txt files were written by the reference's serialize_model
    text = open(f"{GOLDEN_DIR}/{name}.model.txt").read()
    assert serialize_model(parse_model(text)) == text


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_expand_to_complete_matches_oracle(name):
    ens, g = load_golden(name)
    tables = oracle.expand(ens.flat().arrays())
    for (tree, _w), (d, fids, thetas, leaves) in zip(ens.trees, tables):
        ct = expand_to_complete(tree)
        assert ct.depth == d
        assert np.array_equal(ct.fids, fids)
        assert np.array_equal(ct.thetas, thetas)
        assert np.array_equal(ct.leaf_values, leaves)


@pytest.mark.parametrize("name", ["mixed", "trivia", "deep_unbalanced"])
def test_reference_predict_on_flat_trees(name):
    ens, g = load_golden(name)
    for i in range(0, g["X"].shape[0], 17):
        assert reference_predict(ens, g["X"][i]) == g["scores"][i]


def test_node_narrowing_and_validation():
    assert Node.leaf(0.1).value == float(np.float32(0.1))
    assert Node.internal(0, 0.1, Node.leaf(0), Node.leaf(1)).threshold == float(np.float32(0.1))
    for bad in (math.inf, math.nan, 1e39):
        with pytest.raises(ModelSemanticError):
            Node.leaf(bad)
        with pytest.raises(ModelSemanticError):
            Node.internal(0, bad, Node.leaf(0), Node.leaf(1))
    with pytest.raises(ModelSemanticError):
        Node.internal(-1, 0.5, Node.leaf(0), Node.leaf(1))
    shared = Node.leaf(1.0)
    with pytest.raises(ModelSemanticError):
        Tree(Node.internal(0, 0.5, shared, shared))


def test_tree_stats_and_ensemble_checks():
    t = chain_tree(2)
    assert (t.depth, t.leaf_count, t.node_count) == (2, 3, 5)
    st = tree_stats(Ensemble(8, [chain_tree(2), chain_tree(4)]))
    assert st[:2] == (3.0, 4) and st.avg_depth == 3.0 and st.max_depth == 4
    tree = Tree(Node.internal(5, 0.5, Node.leaf(0.0), Node.leaf(1.0)))
    Ensemble(6, [tree])
    with pytest.raises(ModelSemanticError):
        Ensemble(5, [tree])
    with pytest.raises(ModelSemanticError):
        Ensemble(4, [])
    with pytest.raises(ModelSemanticError):
        Ensemble(4, [(Tree(Node.leaf(1.0)), math.inf)])


def test_tie_goes_right_and_expansion_sentinels():
    tree = Tree(Node.internal(0, 0.5, Node.leaf(-1.0), Node.leaf(1.0)))
    assert traverse_to_leaf(tree.root, np.array([0.5], np.float32)).value == 1.0
    assert traverse_to_leaf(tree.root, np.array([0.4999], np.float32)).value == -1.0
    un = Tree(Node.internal(0, 0.5, Node.leaf(1.0),
                            Node.internal(1, 0.25, Node.leaf(2.0), Node.leaf(3.0))))
    ct = expand_to_complete(un)
    assert ct.fids[1] == 0 and math.isinf(float(ct.thetas[1]))
    assert ct.leaf_values.tolist() == [1.0, 1.0, 2.0, 3.0]
    ct0 = expand_to_complete(Tree(Node.leaf(1.25)))
    assert ct0.depth == 0 and len(ct0.fids) == 0 and ct0.leaf_values.tolist() == [1.25]


def test_depth_limit():
    expand_to_complete(chain_tree(12))
    with pytest.raises(DepthLimitError):
        expand_to_complete(chain_tree(MAX_DEPTH + 1))


def test_parse_errors():
    with pytest.raises(ModelSyntaxError):
        parse_model("")
    with pytest.raises(ModelSyntaxError) as e:
        parse_model("ensemble 2 1\ntree 1.0\nnode 0 0 x 1 2\n")
    assert e.value.line == 3
    with pytest.raises(ModelSemanticError, match="out of range"):
        parse_model("ensemble 2 1\ntree 1.0\nnode 0 2 0.5 1 2\nleaf 1 0\nleaf 2 1\nend\n")
    with pytest.raises(ModelSemanticError, match="dangling"):
        parse_model("ensemble 2 1\ntree 1.0\nnode 0 1 0.5 1 3\nleaf 1 0\nleaf 2 1\nend\n")
    with pytest.raises(ModelSemanticError, match="multiple parents"):
        parse_model("ensemble 2 1\ntree 1.0\nnode 0 1 0.5 1 1\nleaf 1 0\nend\n")
    with pytest.raises(ModelSyntaxError, match="missing 'end'"):
        parse_model("ensemble 2 1\ntree 1.0\nleaf 0 1\n")
    with pytest.raises(ModelSyntaxError, match="after final tree"):
        parse_model("ensemble 2 1\ntree 1.0\nleaf 0 1\nend\nleaf 0 1\n")
    # comments and blank lines are ignored
    ens = parse_model("# hi\n\nensemble 3 1\n  # c\ntree 2.0\nleaf 0 0.5\nend\n")
    assert ens.trees[0][1] == 2.0 and ens.trees[0][0].depth == 0


def test_flat_model_round_trip():
    ens, _ = load_golden("mixed")
    flat = ens.flat()
    assert flat.num_trees == len(ens.trees)
    assert serialize_model(flat.to_ensemble()) == serialize_model(ens)


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not __import__("os").path.isdir(REF_SRC), reason="reference not mounted")
def test_adopts_reference_ensemble_objects():
    # build_gpu accepts the reference's own Ensemble (duck-typed Node graphs);
    # the adopted model must serialize exactly as the reference does.
    import subprocess
    import sys
    code = (
        "import sys; sys.dont_write_bytecode=True; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import numpy as np, treescore as ts\n"
        "from paper_1212_2287_b200 import Ensemble, serialize_model\n"
        "from treescore.synth import GenConfig, gen_tree\n"
        "trees=[(gen_tree(GenConfig(depth=d, num_features=9, seed=d)), 0.5+d) for d in range(5)]\n"
        "ref=ts.Ensemble(9, trees)\n"
        "ours=Ensemble.from_reference(ref)\n"
        "assert serialize_model(ours)==ts.serialize_model(ref)\n"
        "print('ok')\n") % (REF_SRC, __import__("os").path.dirname(GOLDEN_DIR).rsplit("/tests", 1)[0])
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         env={**__import__("os").environ, "PYTHONDONTWRITEBYTECODE": "1"})
    assert out.stdout.strip() == "ok", out.stderr


def _native():
    from paper_1212_2287_b200 import parse_model_native
    from paper_1212_2287_b200._build import build
    build()
    return parse_model_native


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_native_parser_matches_python_parser(name):
    text = open(f"{GOLDEN_DIR}/{name}.model.txt").read()
    a = _native()(text)
    b = parse_model(text).flat()
    assert a.num_features == b.num_features
    for x, y in zip(a.arrays(), b.arrays()):
        assert x.dtype == y.dtype and np.array_equal(x, y)


BAD_DOCS = [
    "",
    "# only a comment\n",
    "ensemble 2\n",
    "ensemble x 1\n",
    "ensemble 0 1\ntree 1\nleaf 0 1\nend\n",
    "ensemble 2 0\n",
    "ensemble 2 1\n",
    "ensemble 2 1\ntree\n",
    "ensemble 2 1\ntree abc\nleaf 0 1\nend\n",
    "ensemble 2 1\ntree 1.0\nnode 0 0 x 1 2\n",
    "ensemble 2 1\ntree 1.0\nnode 0 -1 0.5 1 2\nleaf 1 0\nleaf 2 1\nend\n",
    "ensemble 2 1\ntree 1.0\nnode 0 2 0.5 1 2\nleaf 1 0\nleaf 2 1\nend\n",
    "ensemble 2 1\ntree 1.0\nnode 0 1 1e39 1 2\nleaf 1 0\nleaf 2 1\nend\n",
    "ensemble 2 1\ntree 1.0\nnode 0 1 0.5 1 3\nleaf 1 0\nleaf 2 1\nend\n",
    "ensemble 2 1\ntree 1.0\nnode 0 1 0.5 1 1\nleaf 1 0\nend\n",
    "ensemble 2 1\ntree 1.0\nleaf 0 1\nleaf 0 2\nend\n",
    "ensemble 2 1\ntree 1.0\nleaf 1 1\nend\n",
    "ensemble 2 1\ntree 1.0\nleaf -1 1\nend\n",
    "ensemble 2 1\ntree 1.0\nleaf 0 inf\nend\n",
    "ensemble 2 1\ntree 1.0\nleaf 0 1\n",
    "ensemble 2 1\ntree 1.0\nleaf 0 1\nend x\n",
    "ensemble 2 1\ntree 1.0\nleaf 0 1\nend\nleaf 0 1\n",
    "ensemble 2 1\ntree 1.0\nbranch 0 1\nend\n",
    "ensemble 2 1\ntree inf\nleaf 0 1\nend\n",
    "ensemble 2 2\ntree 1.0\nleaf 0 1\nend\n",
    "ensemble 2 1\ntree 1.0\nnode 0 0 0.5 1 2\nnode 1 0 0.5 0 2\nleaf 2 1\nend\n",
    "ensemble 2 1\ntree 1.0\nnode 0 0 0.5 1 2\nleaf 1 0\nleaf 2 1\nleaf 3 1\nend\n",
]


@pytest.mark.parametrize("doc", BAD_DOCS)
def test_native_parser_errors_match_python(doc):
    native = _native()
    try:
        parse_model(doc)
        py = None
    except (ModelSyntaxError, ModelSemanticError) as exc:
        py = exc
    try:
        native(doc)
        nat = None
    except (ModelSyntaxError, ModelSemanticError) as exc:
        nat = exc
    assert type(py) is type(nat), (py, nat)
    if isinstance(py, ModelSyntaxError):
        assert (py.line, py.col) == (nat.line, nat.col)
    assert str(py) == str(nat)


def test_native_parser_accepts_python_number_forms():
    doc = "ensemble 1_0 1\ntree +1_0.5\nnode 0 0 1e-3 1 2\nleaf 1 -0.0\nleaf 2 INF\nend\n"
    with pytest.raises(ModelSemanticError):
        _native()(doc)
    doc = doc.replace("INF", "2.5")
    a, b = _native()(doc), parse_model(doc).flat()
    for x, y in zip(a.arrays(), b.arrays()):
        assert np.array_equal(x, y)


@pytest.mark.skipif(not __import__("os").path.isdir(REF_SRC), reason="reference not mounted")
def test_native_parser_errors_match_reference_parser():
    import json
    import subprocess
    import sys
    code = ("import sys, json; sys.dont_write_bytecode=True; sys.path.insert(0, %r)\n"
            "import treescore as ts\n"
            "docs=json.load(sys.stdin); res=[]\n"
            "for d in docs:\n"
            "    try:\n"
            "        ts.parse_model(d); res.append(None)\n"
            "    except ts.ModelSyntaxError as e: res.append(['syntax', str(e), e.line, e.col])\n"
            "    except ts.ModelSemanticError as e: res.append(['semantic', str(e)])\n"
            "print(json.dumps(res))\n") % REF_SRC
    out = subprocess.run([sys.executable, "-c", code], input=json.dumps(BAD_DOCS),
                         capture_output=True, text=True,
                         env={**__import__("os").environ, "PYTHONDONTWRITEBYTECODE": "1"})
    ref = json.loads(out.stdout)
    native = _native()
    for doc, r in zip(BAD_DOCS, ref):
        try:
            native(doc)
            got = None
        except ModelSyntaxError as e:
            got = ["syntax", str(e), e.line, e.col]
        except ModelSemanticError as e:
            got = ["semantic", str(e)]
        assert got == r, doc
