"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden vectors and the pinned CPU oracle.  Scores must be bit-exact f64
(same tie rule, dummy routing, fp32 tables and tree-order multiply-then-add);
per-tree predicated leaf ordinals must be bit-exact."""

import numpy as np
import pytest

import oracle
from conftest import GOLDEN_CASES, has_cuda, load_golden

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]


def _ev(model, **kw):
    from paper_1212_2287_b200 import build_gpu
    return build_gpu(model, **kw)


@pytest.fixture(params=[0, 1], ids=["auto", "l1"])
def kernel_path(request):
    from paper_1212_2287_b200 import _lib
    lib = _lib.load()
    assert lib.ts_set_kernel_path(request.param) == 0
    yield request.param
    lib.ts_set_kernel_path(0)


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_golden_scores_and_ordinals(name, kernel_path):
    ens, g = load_golden(name)
    ev = _ev(ens)
    got = ev.predict_batch(g["X"])
    assert np.array_equal(got, g["scores"])                       # bit-exact
    ords = ev.leaf_indices(g["X"])
    assert np.array_equal(ords, g["ordinals"])


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_golden_device_path_and_single_rows(name):
    import torch
    ens, g = load_golden(name)
    ev = _ev(ens)
    x = torch.from_numpy(g["X"]).cuda()
    out = ev.score_device(x)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), g["scores"])
    for i in range(min(5, g["X"].shape[0])):
        assert ev.predict(g["X"][i]) == g["scores"][i]


def test_strided_rows_and_tile_remainders():
    import torch
    ens, g = load_golden("complete_d6")
    ev = _ev(ens)
    X = g["X"]
    for n in (1, 31, 33, 255, 417, 1023):
        wide = torch.zeros((n, 140), dtype=torch.float32, device="cuda")
        wide[:, :136] = torch.from_numpy(X[:n])
        out = ev.score_device(wide[:, :136])   # row stride 140 > f
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), g["scores"][:n]), n


def test_permutation_independence():
    # ref tests/test_evaluators.py:159-169
    ens, g = load_golden("mixed")
    ev = _ev(ens)
    perm = np.random.default_rng(0).permutation(g["X"].shape[0])
    got = ev.predict_batch(g["X"][perm])
    back = np.empty_like(got)
    back[perm] = got
    assert np.array_equal(back, g["scores"])


def test_empty_input_and_shape_errors():
    # ref tests/test_evaluators.py:119-125 (empty), :118-127 (mismatch)
    ens, _ = load_golden("tie")
    ev = _ev(ens)
    assert ev.predict_batch(np.zeros((0, 1), np.float32)).shape == (0,)
    with pytest.raises(ValueError, match="dataset"):
        ev.predict_batch(np.zeros((3, 2), np.float32))
    with pytest.raises(ValueError, match="feature vector"):
        ev.predict(np.zeros(2, np.float32))


def test_nonfinite_inputs_rejected():
    ens, g = load_golden("complete_d6")
    ev = _ev(ens)
    for bad in (np.nan, np.inf, -np.inf):
        X = g["X"][:100].copy()
        X[57, 3] = bad
        with pytest.raises(ValueError, match="non-finite"):
            ev.predict_batch(X)


def test_depth_limit_and_invalid_models():
    # ref tests/test_evaluators.py:51-62: depth 17 -> DepthLimitError
    from paper_1212_2287_b200 import DepthLimitError, Ensemble, Node, Tree
    node = Node.leaf(1.0)
    for level in range(17):
        node = Node.internal(0, 0.5 / (level + 2), node, Node.leaf(2.0))
    with pytest.raises(DepthLimitError):
        _ev(Ensemble(2, [Tree(node)]))


def test_weights_and_many_segments():
    # alternating complete/irregular trees -> one launch per segment, f64
    # accumulation carried across launches in tree order.
    from paper_1212_2287_b200 import Ensemble
    ens, g = load_golden("mixed")
    trees = [(t, w * (1.0 + 0.25 * i)) for i, (t, w) in enumerate(ens.trees)]
    ens2 = Ensemble(ens.num_features, trees)
    ev = _ev(ens2)
    assert ev.model.info["num_segments"] > 3
    c = oracle.COracle(ens2.flat().arrays())
    assert np.array_equal(ev.predict_batch(g["X"]), c.score(g["X"]))


def test_config0_full_vs_oracle(kernel_path):
    from paper_1212_2287_b200 import synth
    w = synth.config0()
    ev = _ev(w.flat)
    c = oracle.COracle(w.flat.arrays())
    ref, ref_ord = c.score(w.x, with_ordinals=True)
    assert np.array_equal(ev.predict_batch(w.x), ref)
    assert np.array_equal(ev.leaf_indices(w.x), ref_ord.astype(np.int64))


def test_config1_ties_subsample_vs_oracle(kernel_path):
    from paper_1212_2287_b200 import synth
    w = synth.config1(n=60_000)
    ev = _ev(w.flat)
    c = oracle.COracle(w.flat.arrays())
    ref, ref_ord = c.score(w.x, with_ordinals=True)
    assert np.array_equal(ev.predict_batch(w.x), ref)
    assert np.array_equal(ev.leaf_indices(w.x[:5000]), ref_ord[:, :5000].astype(np.int64))


@pytest.mark.parametrize("depth", [3, 4, 6, 8, 10, 12])
def test_config2_depths_vs_oracle(depth, kernel_path):
    from paper_1212_2287_b200 import synth
    w = synth.config2(depth, n=4096, trees=200)
    ev = _ev(w.flat)
    c = oracle.COracle(w.flat.arrays())
    ref, ref_ord = c.score(w.x, with_ordinals=True)
    assert np.array_equal(ev.predict_batch(w.x), ref)
    assert np.array_equal(ev.leaf_indices(w.x), ref_ord.astype(np.int64))


def test_config3_irregular_device_generated_rows():
    import torch
    from paper_1212_2287_b200 import synth, _lib
    w = synth.config3(n=20_000, trees=300)
    ev = _ev(w.flat)
    x = torch.empty((w.n, w.f), dtype=torch.float32, device="cuda")
    rc = _lib.load().ts_synth_uniform(x.data_ptr(), w.n, w.f, w.f, w.hash_seed, 0, w.zero_prob,
                                      torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    out = ev.score_device(x)
    host = w.rows(0, w.n)
    assert np.array_equal(x.cpu().numpy(), host)   # device generator == host
    c = oracle.COracle(w.flat.arrays())
    ref, ref_ord = c.score(host, with_ordinals=True)
    assert np.array_equal(out.cpu().numpy(), ref)
    assert np.array_equal(ev.leaf_indices(host[:3000]), ref_ord[:, :3000].astype(np.int64))


def test_wide_features_global_path():
    # F too wide for a shared-memory tile -> the global-read kernel variant.
    from paper_1212_2287_b200 import synth
    flat = synth.irregular_flat(77, 40, 3000, leaves=32)
    X = np.random.default_rng(1).random((700, 3000), dtype=np.float32)
    ev = _ev(flat)
    c = oracle.COracle(flat.arrays())
    ref, ref_ord = c.score(X, with_ordinals=True)
    assert np.array_equal(ev.predict_batch(X), ref)
    assert np.array_equal(ev.leaf_indices(X), ref_ord.astype(np.int64))


def test_launch_counter_advances():
    from paper_1212_2287_b200 import _lib
    ens, g = load_golden("complete_d6")
    ev = _ev(ens)
    before = _lib.launch_count()
    ev.predict_batch(g["X"])
    assert _lib.launch_count() > before


def test_tree_shards_continue_sum_bit_exact():
    # ts_score_ex(accumulate=1): scoring tree shard after tree shard from the
    # running sums reproduces single-model scores bit for bit (what the
    # multi-GPU tree pipeline relies on), on every kernel path.
    import torch
    from paper_1212_2287_b200 import GpuModel, synth
    from paper_1212_2287_b200.distributed import tree_shards
    for w in (synth.config2(8, n=3000, trees=60), synth.config3(n=3000, trees=40)):
        x = torch.from_numpy(w.rows(0, w.n)).cuda()
        full = GpuModel(w.flat).score(x)
        out = torch.empty_like(full)
        for i, (a, b) in enumerate(tree_shards(w.flat.depths(), 3)):
            GpuModel(w.flat.subset(a, b)).score(x, out=out, accumulate=i > 0)
        torch.cuda.synchronize()
        assert torch.equal(out, full)


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_traced_prediction_and_coverage(name):
    # ref predict_ensemble_traced (evaluators.py:599-620) and
    # measure_feature_coverage (bench.py:412-427), bit for bit
    ens, g = load_golden(name)
    ev = _ev(ens, trace=True)
    scores, bits, leaves = ev.trace_batch(g["X"])
    assert np.array_equal(scores, g["scores"])
    assert np.array_equal(bits, g["trace_bits"])
    assert np.array_equal(leaves, g["trace_leaves"])
    cov = ev.feature_coverage(g["X"])
    assert (cov.mean_fraction, cov.variance, cov.num_instances) == \
        (g["coverage"][0], g["coverage"][1], g["X"].shape[0])
    tp = ev.predict_traced(g["X"][0])
    assert tp.score == g["scores"][0]
    assert tp.visited_leaves == tuple(g["trace_leaves"][:, 0].tolist())
    # the reference's module-level names, backed by the same tracer
    from paper_1212_2287_b200 import Dataset, measure_feature_coverage, predict_ensemble_traced
    assert predict_ensemble_traced(ens, g["X"][0]) == tp
    cov2 = measure_feature_coverage(ens, Dataset(g["X"]))
    assert (cov2.mean_fraction, cov2.variance) == (g["coverage"][0], g["coverage"][1])


def test_predict_fvec_streams_files(tmp_path):
    from paper_1212_2287_b200 import write_fvec
    ens, g = load_golden("mixed")
    ev = _ev(ens)
    path = tmp_path / "x.fvec"
    write_fvec(path, g["X"])
    for chunk in (64, 333, 10_000):
        assert np.array_equal(ev.predict_fvec(path, chunk_rows=chunk), g["scores"])
    X = g["X"].copy()
    X[401, 2] = np.nan
    write_fvec(path, X)
    with pytest.raises(ValueError, match="non-finite"):
        ev.predict_fvec(path, chunk_rows=128)


@pytest.mark.parametrize("depth", [13, 16])
def test_deep_complete_trees_l1_path(depth):
    # complete trees deeper than the streaming kernel handles (d > 12) run on
    # the L1-path heap kernel
    from paper_1212_2287_b200 import synth
    rng = np.random.default_rng(depth)
    T, F = 3, 20
    n_int = (1 << depth) - 1
    flat = synth.complete_flat(F, depth, rng.integers(0, F, (T, n_int)),
                               rng.random((T, n_int), dtype=np.float32),
                               rng.standard_normal((T, 1 << depth)).astype(np.float32),
                               weights=[0.5, 1.0, -2.0])
    X = rng.random((777, F), dtype=np.float32)
    ev = _ev(flat)
    c = oracle.COracle(flat.arrays())
    ref, ref_ord = c.score(X, with_ordinals=True)
    assert np.array_equal(ev.predict_batch(X), ref)
    assert np.array_equal(ev.leaf_indices(X), ref_ord.astype(np.int64))


def test_tiny_shapes_and_padded_ordinals():
    import torch
    from paper_1212_2287_b200 import Ensemble, Node, Tree
    ens = Ensemble(1, [Tree(Node.internal(0, 0.25, Node.leaf(-1.5), Node.leaf(2.5))),
                       (Tree(Node.leaf(0.125)), 3.0)])
    ev = _ev(ens)
    assert ev.predict(np.array([0.25], np.float32)) == 2.5 + 3.0 * 0.125
    x = torch.tensor([[0.0], [0.3]], dtype=torch.float32, device="cuda")
    ords = torch.full((2, 64), -1, dtype=torch.int16, device="cuda")   # ld_ord > n
    ev.model.score(x, ordinals=ords)
    torch.cuda.synchronize()
    o = ords.cpu().numpy()
    assert o[:, :2].tolist() == [[0, 1], [0, 0]] and (o[:, 2:] == -1).all()


def test_models_on_concurrent_streams():
    import torch
    from paper_1212_2287_b200 import synth
    w1 = synth.config2(6, n=5000, trees=64)
    ens, g = load_golden("mixed")
    ev1, ev2 = _ev(w1.flat), _ev(ens)
    x1 = torch.from_numpy(w1.x).cuda()
    x2 = torch.from_numpy(g["X"]).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for _ in range(3):
        with torch.cuda.stream(s1):
            o1 = ev1.score_device(x1, stream=s1)
        with torch.cuda.stream(s2):
            o2 = ev2.score_device(x2, stream=s2)
        outs.append((o1, o2))
    torch.cuda.synchronize()
    ref1 = oracle.COracle(w1.flat.arrays()).score(w1.x)
    for o1, o2 in outs:
        assert np.array_equal(o1.cpu().numpy(), ref1)
        assert np.array_equal(o2.cpu().numpy(), g["scores"])


def test_invalid_models_rejected_by_packer():
    from paper_1212_2287_b200 import FlatModel, GpuModel, ModelSemanticError
    bad = [
        FlatModel(2, np.array([0, 3]), np.array([1.0]), np.array([0, -1, -1], np.int32),
                  np.array([0.5, 1, 2], np.float32), np.array([1, -1, -1], np.int32),
                  np.array([1, -1, -1], np.int32)),                    # two parents
        FlatModel(2, np.array([0, 3]), np.array([np.nan]), np.array([0, -1, -1], np.int32),
                  np.array([0.5, 1, 2], np.float32), np.array([1, -1, -1], np.int32),
                  np.array([2, -1, -1], np.int32)),                    # NaN weight
        FlatModel(2, np.array([0, 3]), np.array([1.0]), np.array([0, -1, -1], np.int32),
                  np.array([0.5, 1, 2], np.float32), np.array([1, -1, -1], np.int32),
                  np.array([0, -1, -1], np.int32)),                    # root as child
    ]
    for fm in bad:
        with pytest.raises(ModelSemanticError):
            GpuModel(fm)


@pytest.mark.parametrize("plan", ["2,8,4,1", "2,8,4,2", "1,8,4,1", "1,8,8,2", "4,8,8,2", "2,16,4,1",
                                  "1,16,3,1", "1,16,3,2", "8,8,4,1", "4,16,8,1", "2,16,8,1",
                                  "1,16,8,1", "4,16,4,1"])
@pytest.mark.parametrize("name", ["wide_irregular", "mixed", "deep_unbalanced"])
def test_irregular_kernel_shapes(name, plan, monkeypatch):
    """Every k_cstream shape (G instance groups, W walker warps, K chains) the
    planner can pick, forced with TS_CSTREAM_PLAN at pack and launch time;
    shapes that do not fit fall back to the L1 path, which must agree too."""
    monkeypatch.setenv("TS_CSTREAM_PLAN", plan)
    ens, g = load_golden(name)
    ev = _ev(ens)
    assert np.array_equal(ev.predict_batch(g["X"]), g["scores"])
    assert np.array_equal(ev.leaf_indices(g["X"]), g["ordinals"])


@pytest.mark.parametrize("split", [None, "0", "2", "7"])
@pytest.mark.parametrize("n", [1, 100, 1000, 5000])
def test_small_batch_tree_split(n, split, monkeypatch):
    """Small batches split each tile's trees over several CTAs and fold the
    leaves in tree order afterwards (TS_SPLIT forces / disables it); scores
    and ordinals must not depend on it."""
    from paper_1212_2287_b200.synth import complete_flat
    if split is not None:
        monkeypatch.setenv("TS_SPLIT", split)
    rng = np.random.default_rng(n)
    T, d, F = 300, 6, 40
    n_int = (1 << d) - 1
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         rng.standard_normal((T, 1 << d)), weights=rng.uniform(0.5, 1.5, T))
    x = rng.random((n, F), dtype=np.float32)
    ev = _ev(flat)
    ref = oracle.COracle(flat.arrays())
    s, o = ref.score(x, threads=4, with_ordinals=True)
    assert np.array_equal(ev.predict_batch(x), s)
    assert np.array_equal(ev.leaf_indices(x), o.astype(np.int64))


def _leaf_table(kind, rng, T, d):
    """Leaf values that steer the tree split's fold: 'narrow' lets it prove the
    sum order-independent (fast path); the others must take the tree-order
    chain (dynamic range beyond what f64 holds exactly) or sit on its edges."""
    L = 1 << d
    if kind == "narrow":
        return rng.standard_normal((T, L)) * 0.1
    if kind == "wide":          # 40 decades: partial sums round, order matters
        return rng.standard_normal((T, L)) * 10.0 ** rng.uniform(-30, 10, (T, L))
    if kind == "cancel":        # big +/- pairs around tiny odd multiples of 2^-60
        v = np.where(rng.random((T, L)) < 0.5, 1.0, -1.0) * 2.0 ** rng.integers(20, 30, (T, L))
        tiny = rng.integers(1, 1 << 20, (T, L)) * 2.0 ** -60
        return np.where(rng.random((T, L)) < 0.5, v, tiny)
    if kind == "zeros":         # signed zeros, denormals and a few ordinary values
        v = rng.choice(np.array([0.0, -0.0, 1e-45, -3e-42, 0.25, -1.5], np.float64), (T, L))
        return v
    if kind == "allnegzero":
        return np.full((T, L), -0.0)
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["narrow", "wide", "cancel", "zeros", "allnegzero"])
@pytest.mark.parametrize("n", [1, 77, 1000])
def test_tree_split_fold_fast_path(kind, n, monkeypatch):
    """Unit-weight ensembles: the fold adds the splits' own sums when the
    leaves' dynamic range proves every partial sum exact (ts_stream.cu
    split_sum_exact), else the tree-order chain; both must give the
    reference's sequential f64 sum bit for bit (ref evaluators.py:529-535)."""
    from paper_1212_2287_b200.synth import complete_flat
    rng = np.random.default_rng(len(kind) * 1000 + n)
    T, d, F = 400, 7, 40
    n_int = (1 << d) - 1
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         _leaf_table(kind, rng, T, d))
    x = rng.random((n, F), dtype=np.float32)
    ref = oracle.COracle(flat.arrays()).score(x, threads=4)
    got = {}
    for fast in ("1", "0"):
        monkeypatch.setenv("TS_FOLD_FAST", fast)
        for split in ("3", "11"):
            monkeypatch.setenv("TS_SPLIT", split)
            ev = _ev(flat)
            got[fast, split] = ev.predict_batch(x)
            ev.close()
    for k, v in got.items():
        assert np.array_equal(v.view(np.uint64), ref.view(np.uint64)), k


@pytest.mark.parametrize("kind", ["narrow", "wide", "cancel", "zeros", "allnegzero"])
@pytest.mark.parametrize("n,ctas", [(1, None), (300, "7"), (300, None), (5000, None), (5000, "50"),
                                    (5000, "333")])
def test_balanced_tree_split(kind, n, ctas, monkeypatch):
    """Balanced tree split (TS_SK=1; ts_stream.cu launch_balanced): equal runs
    of (tile, chunk) items per CTA, tiles shared by several CTAs combined from
    their partial sums when provably exact, re-walked in tree order otherwise
    -- scores and ordinals identical to the oracle's either way."""
    from paper_1212_2287_b200.synth import complete_flat
    monkeypatch.setenv("TS_SK", "1")
    if ctas:
        monkeypatch.setenv("TS_SK_CTAS", ctas)
    rng = np.random.default_rng(len(kind) * 77 + n)
    T, d, F = 330, 7, 40
    n_int = (1 << d) - 1
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         _leaf_table(kind, rng, T, d))
    x = rng.random((n, F), dtype=np.float32)
    s, o = oracle.COracle(flat.arrays()).score(x, threads=4, with_ordinals=True)
    ev = _ev(flat)
    assert np.array_equal(ev.predict_batch(x).view(np.uint64), s.view(np.uint64))
    assert np.array_equal(ev.leaf_indices(x), o.astype(np.int64))
    ev.close()


@pytest.mark.parametrize("kind,launches", [("narrow", 2), ("wide", 1)])
def test_balanced_tree_split_default_rule(kind, launches):
    """A batch the planner sends to the balanced split by itself (unit
    weights, d = 8, tiles filling ~0.3 of the CTA slots): the walk and
    k_combine, scores and ordinals equal to the oracle's.  The same shape with
    leaves spread over 40 decades stays on a one-launch kernel: the packer's
    estimate (Segment::slow_rows) says most rows' sums could round, and
    k_combine would walk each of them a second time."""
    from paper_1212_2287_b200 import _lib
    from paper_1212_2287_b200.synth import complete_flat
    rng = np.random.default_rng(12)
    T, d, F, n = 760, 8, 136, 12000
    n_int = (1 << d) - 1
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         _leaf_table(kind, rng, T, d))
    x = rng.random((n, F), dtype=np.float32)
    s, o = oracle.COracle(flat.arrays()).score(x, threads=8, with_ordinals=True)
    import torch
    ev = _ev(flat)
    xd = torch.from_numpy(x).cuda()
    before = _lib.launch_count()
    got = ev.score_device(xd).cpu().numpy()
    assert _lib.launch_count() - before == launches
    assert np.array_equal(got.view(np.uint64), s.view(np.uint64))
    assert np.array_equal(ev.predict_batch(x).view(np.uint64), s.view(np.uint64))
    assert np.array_equal(ev.leaf_indices(x), o.astype(np.int64))
    ev.close()


@pytest.mark.parametrize("d,F", [(1, 40), (2, 40), (4, 40), (5, 136), (6, 40), (8, 136), (9, 40),
                                 (10, 40), (12, 24)])
def test_balanced_tree_split_slow_rows(d, F, monkeypatch):
    """Rows whose sums could round are walked again by k_combine in the model
    blob (split_walk_global): every record form -- no deep levels (d <= 5),
    the 16-byte header and its absence (d = 8), global-leaf depths (rows wide
    enough for 2-byte fids do not fit the streaming kernel's tile) -- with leaf tables that put most rows on that path."""
    from paper_1212_2287_b200.synth import complete_flat
    monkeypatch.setenv("TS_SK", "1")
    monkeypatch.setenv("TS_RANK", "0")
    rng = np.random.default_rng(d * 1000 + F)
    T, n = max(24, 600 >> max(0, d - 6)), 700
    n_int = (1 << d) - 1
    thetas = rng.random((T, n_int))
    thetas[rng.random((T, n_int)) < 0.2] = 0.5  # ties with the rows below
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), thetas,
                         _leaf_table("wide", rng, T, d))
    x = rng.random((n, F), dtype=np.float32)
    x[::7, ::3] = 0.5
    s, o = oracle.COracle(flat.arrays()).score(x, threads=4, with_ordinals=True)
    ev = _ev(flat)
    assert ev.model.info["complete_trees"] == T
    assert np.array_equal(ev.predict_batch(x).view(np.uint64), s.view(np.uint64))
    assert np.array_equal(ev.leaf_indices(x), o.astype(np.int64))
    ev.close()


@pytest.mark.parametrize("n", [200, 6000])
def test_balanced_tree_split_weighted(n, monkeypatch):
    """Non-unit weights: no partial sum is provably exact, so every shared
    tile's rows are added in tree order from the stored ordinals."""
    from paper_1212_2287_b200.synth import complete_flat
    monkeypatch.setenv("TS_SK", "1")
    rng = np.random.default_rng(n)
    T, d, F = 250, 8, 136
    n_int = (1 << d) - 1
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         rng.standard_normal((T, 1 << d)), weights=rng.uniform(0.5, 1.5, T))
    x = rng.random((n, F), dtype=np.float32)
    s, o = oracle.COracle(flat.arrays()).score(x, threads=4, with_ordinals=True)
    ev = _ev(flat)
    assert np.array_equal(ev.predict_batch(x).view(np.uint64), s.view(np.uint64))
    assert np.array_equal(ev.leaf_indices(x), o.astype(np.int64))
    ev.close()


@pytest.mark.parametrize("d,T,n", [(3, 700, 2000), (10, 60, 3000), (11, 40, 1500), (12, 24, 700)])
def test_balanced_tree_split_depths(d, T, n, monkeypatch):
    """Balanced split on the 256-row CTA shape (d >= 10), the global-leaf
    depths (d >= 11) and shallow trees, with a running sum from a first
    segment of another depth."""
    from paper_1212_2287_b200 import Ensemble
    monkeypatch.setenv("TS_SK", "1")
    monkeypatch.setenv("TS_RANK", "0")
    rng = np.random.default_rng(d * 100 + T)
    f = 24
    trees = [(_rand_complete(rng, 5, f), 1.0) for _ in range(40)]
    trees += [(_rand_complete(rng, d, f), 1.0) for _ in range(T)]
    ens = Ensemble(f, trees)
    X = rng.random((n, f), dtype=np.float32)
    s, o = oracle.COracle(ens.flat().arrays()).score(X, threads=4, with_ordinals=True)
    ev = _ev(ens)
    assert np.array_equal(ev.predict_batch(X).view(np.uint64), s.view(np.uint64))
    assert np.array_equal(ev.leaf_indices(X), o.astype(np.int64))
    ev.close()


def test_tree_split_fold_continues_running_sum(monkeypatch):
    """Unit-weight segments of different depths: the second segment's fold
    starts from the first one's sums (acc0 != 0 in the exactness test), also
    when those are too fine-grained for the fast path."""
    from paper_1212_2287_b200 import Ensemble
    monkeypatch.setenv("TS_SPLIT", "5")
    for scale in (1.0, 2.0 ** -45):
        rng = np.random.default_rng(91)
        f = 40
        trees = [(_rand_complete(rng, 6, f, leaf_scale=scale), 1.0) for _ in range(150)]
        trees += [(_rand_complete(rng, 8, f), 1.0) for _ in range(150)]
        ens = Ensemble(f, trees)
        X = rng.random((300, f), dtype=np.float32)
        s = oracle.COracle(ens.flat().arrays()).score(X, threads=4)
        ev = _ev(ens)
        assert ev.model.info["num_segments"] == 2
        assert np.array_equal(ev.predict_batch(X).view(np.uint64), s.view(np.uint64))
        ev.close()


@pytest.mark.parametrize("name", ["complete_d6", "ties_counts", "trivia"])
def test_complete_trees_on_irregular_kernel(name, monkeypatch):
    """TS_FORCE_CSTREAM packs complete trees as child-index records for the
    irregular-tree kernel: same scores and predicated ordinals."""
    monkeypatch.setenv("TS_FORCE_CSTREAM", "1")
    ens, g = load_golden(name)
    ev = _ev(ens)
    assert ev.model.info["compact_trees"] == ev.model.info["num_trees"]
    assert np.array_equal(ev.predict_batch(g["X"]), g["scores"])
    assert np.array_equal(ev.leaf_indices(g["X"]), g["ordinals"])


@pytest.mark.parametrize("n", [64, 1000, 40000])
def test_scoring_captured_in_cuda_graph(n):
    """ts_score is stream-ordered and allocation-free on the host side, so a
    serving loop can capture it once in a CUDA graph and replay it (the
    small-batch tree split's scratch comes from a stream-ordered pool, which
    graphs capture as memory nodes)."""
    import torch
    from paper_1212_2287_b200.synth import complete_flat
    rng = np.random.default_rng(n)
    T, d, F = 400, 8, 64
    n_int = (1 << d) - 1
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         rng.standard_normal((T, 1 << d)))
    ev = _ev(flat)
    x = torch.from_numpy(rng.random((n, F), dtype=np.float32)).cuda()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ev.score_device(x, out)          # warm-up outside capture (smem attributes)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ev.score_device(x, out)
    ref = oracle.COracle(flat.arrays())
    for _ in range(2):
        x.copy_(torch.from_numpy(rng.random((n, F), dtype=np.float32)))
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), ref.score(x.cpu().numpy(), threads=4))


def test_build_accepts_reference_kinds():
    # ref evaluators.py:565-585 argument checks; every kind scores the same
    from paper_1212_2287_b200 import StrategyKind, build
    ens, g = load_golden("mixed")
    for kind, v in (("vpredicated", 16), ("predicated", None), ("heap_linked", None),
                    ("compact_linked", None), ("contiguous", None),
                    (StrategyKind.GPU_VPREDICATED, None)):
        assert np.array_equal(build(ens, kind, v).predict_batch(g["X"]), g["scores"])
    # ref tests/test_evaluators.py:78-82, 238-262: kind and stored_node_count
    from paper_1212_2287_b200 import Ensemble, Node, Tree
    tree = Tree(Node.internal(0, 0.5, Node.leaf(1.0),
                              Node.internal(1, 0.25, Node.leaf(2.0), Node.leaf(3.0))))
    small = Ensemble(2, [tree])
    for kind in ("heap_linked", "compact_linked", "contiguous"):
        ev = build(small, kind)
        assert ev.kind is StrategyKind(kind) and ev.stored_node_count == 5
    assert build(small, "predicated").stored_node_count == 7
    assert build(small, "vpredicated", 8).stored_node_count == 7
    with pytest.raises(ValueError, match="requires a batch_size"):
        build(ens, "vpredicated")
    with pytest.raises(ValueError, match="does not apply"):
        build(ens, "heap_linked", 4)
    with pytest.raises(ValueError, match="compiled"):
        build(ens, "generated")
    with pytest.raises(ValueError):
        build(ens, "no_such_kind")


def _rand_unbalanced(rng, max_depth, f, prune=0.35, leaf=None):
    from paper_1212_2287_b200 import Node, Tree

    def build_node(level):
        if level == max_depth or (level > 0 and rng.random() < prune):
            return Node.leaf(rng.random() if leaf is None else leaf())
        return Node.internal(int(rng.integers(f)), rng.random(), build_node(level + 1),
                             build_node(level + 1))
    return Tree(build_node(0))


def _rand_complete(rng, depth, f, leaf_scale=1.0):
    from paper_1212_2287_b200 import Node, Tree

    def build_node(level):
        if level == depth:
            return Node.leaf(rng.standard_normal() * leaf_scale)
        return Node.internal(int(rng.integers(f)), rng.random(), build_node(level + 1),
                             build_node(level + 1))
    return Tree(build_node(0))


@pytest.mark.parametrize("kind", ["narrow", "wide", "zeros"])
@pytest.mark.parametrize("f,n,ctas", [(40, 1, None), (40, 77, "9"), (40, 1500, None), (700, 300, None),
                                      (136, 5000, "50")])
def test_irregular_balanced_split(kind, f, n, ctas, monkeypatch):
    """Balanced tree split on the irregular-tree kernel (k_cstream<..., SK>):
    runs of (tile, chunk) items per CTA, the accumulator warp's partial sums
    combined when provably exact, rows walked again from the child-index
    records otherwise; unit weights; bit-exact, also from a running sum."""
    import torch
    from paper_1212_2287_b200 import Ensemble
    monkeypatch.setenv("TS_SK", "1")
    if ctas:
        monkeypatch.setenv("TS_SK_CTAS", ctas)
    rng = np.random.default_rng(f + n + len(kind))
    leaf = {"narrow": lambda: rng.standard_normal() * 0.05,
            "wide": lambda: rng.standard_normal() * 10.0 ** rng.uniform(-30, 10),
            "zeros": lambda: float(rng.choice([0.0, -0.0, 1e-45, -3e-42, 0.25, -1.5]))}[kind]
    trees = [(_rand_unbalanced(rng, int(rng.integers(2, 13)), f, prune=0.3, leaf=leaf), 1.0)
             for _ in range(260)]
    ens = Ensemble(f, trees)
    X = rng.random((n, f), dtype=np.float32)
    X[rng.random((n, f)) < 0.3] = 0.0
    s, o = oracle.COracle(ens.flat().arrays()).score(X, threads=4, with_ordinals=True)
    ev = _ev(ens)
    assert ev.model.info["compact_trees"] >= 150   # (a few random trees come out complete)
    assert np.array_equal(ev.predict_batch(X).view(np.uint64), s.view(np.uint64))
    assert np.array_equal(ev.leaf_indices(X), o.astype(np.int64))
    monkeypatch.setenv("TS_FOLD_FAST", "0")   # every shared tile's rows on the second walk
    assert np.array_equal(ev.score_device(torch.from_numpy(X).cuda()).cpu().numpy().view(np.uint64),
                          s.view(np.uint64))
    ev.close()


def test_balanced_split_learns_from_second_walks(monkeypatch):
    """One tiny leaf that every row reaches: the packer's estimate (one leaf
    in ~30,000) lets the planner split, every shared tile's rows then need
    k_combine's second walk, and the model's observed counters
    (DeviceTables::slow_seen) make the next calls walk whole tiles again --
    bit-exact before and after."""
    import torch
    from paper_1212_2287_b200 import Ensemble, Node, Tree, _lib
    monkeypatch.setenv("TS_FORCE_CSTREAM", "1")   # one irregular-kernel segment
    rng = np.random.default_rng(404)
    f = 40
    leaf = lambda: rng.standard_normal() * 0.05  # noqa: E731
    trees = [(_rand_unbalanced(rng, 9, f, prune=0.12, leaf=leaf), 1.0) for _ in range(720)]
    hot = Tree(Node.internal(0, -1.0, Node.leaf(0.1),
                             Node.internal(1, -1.0, Node.leaf(0.2), Node.leaf(1e-12))))
    trees.insert(5, (hot, 1.0))
    ens = Ensemble(f, trees)
    n = 1500
    X = rng.random((n, f), dtype=np.float32)
    s = oracle.COracle(ens.flat().arrays()).score(X, threads=4)
    ev = _ev(ens)
    xd = torch.from_numpy(X).cuda()
    launches = []
    for _ in range(3):
        before = _lib.launch_count()
        got = ev.score_device(xd).cpu().numpy()   # (the copy back synchronises)
        launches.append(_lib.launch_count() - before)
        assert np.array_equal(got.view(np.uint64), s.view(np.uint64))
    assert launches[0] == 2 and launches[-1] == 1, launches
    ev.close()


def test_acceptance_cross_strategy_schedule():
    """The reference's acceptance criterion 1 (ref tests/test_acceptance.py:
    83-125) on the GPU: 200 ensembles over f = 32/128/512 with its schedule
    of shapes (a complete tree of the slot's depth first, then balanced and
    pruned trees; a single d=11 / d=9 tree, 50 d=2 trees, 2 d=7 trees in the
    special slots), weights U(0.5, 1.5), 100 vectors each -- bit-exact
    against the pinned C oracle, scores and ordinals."""
    from paper_1212_2287_b200 import Ensemble
    rng = np.random.default_rng(101)
    for i in range(200):
        f = (32, 128, 512)[i % 3]
        slot = i % 40
        if slot == 7:
            depth, trees = 11, 1
        elif slot == 15:
            depth, trees = 9, 1
        elif slot == 23:
            depth, trees = 2, 50
        elif slot == 31:
            depth, trees = 7, 2
        else:
            depth = int(rng.integers(0, 7))
            trees = min(1 + int(min(rng.geometric(0.35), 49)), max(1, 512 >> depth))
        ts = [(_rand_complete(rng, depth, f), float(rng.uniform(0.5, 1.5)))]
        for t in range(1, trees):
            tree = _rand_complete(rng, int(rng.integers(0, depth + 1)), f) if t % 2 == 0 \
                else _rand_unbalanced(rng, depth, f)
            ts.append((tree, float(rng.uniform(0.5, 1.5))))
        ens = Ensemble(f, ts)
        X = rng.random((100, f), dtype=np.float32)
        s, o = oracle.COracle(ens.flat().arrays()).score(X, threads=2, with_ordinals=True)
        ev = _ev(ens)
        assert np.array_equal(ev.predict_batch(X), s), (i, depth, f, trees)
        assert np.array_equal(ev.leaf_indices(X), o.astype(np.int64)), (i, depth, f, trees)


@pytest.mark.parametrize("depth", [1, 2, 3, 5, 8])
def test_acceptance_per_leaf_probes(depth):
    """The reference's acceptance criterion 2 (ref tests/test_acceptance.py:
    132-161) on the GPU: for a complete tree, one probe vector per reachable
    leaf (built from the path's bounds: right turns need x >= theta, left
    turns x < theta) must come back with that leaf's predicated ordinal."""
    from paper_1212_2287_b200.synth import complete_flat
    rng = np.random.default_rng(depth + 100)
    f = 16
    n_int = (1 << depth) - 1
    fids = rng.integers(0, f, n_int)
    thr = rng.random(n_int).astype(np.float32)
    flat = complete_flat(f, depth, fids[None], thr[None], np.arange(1 << depth)[None] * 1.0)
    probes, want = [], []
    for leaf in range(1 << depth):
        lo = np.full(f, -1.0, np.float64)
        hi = np.full(f, 2.0, np.float64)
        node = 0
        for level in range(depth):
            right = (leaf >> (depth - 1 - level)) & 1
            fid, t = fids[node], float(thr[node])
            if right:
                lo[fid] = max(lo[fid], t)
            else:
                hi[fid] = min(hi[fid], t)
            node = 2 * node + 1 + right
        if np.all(lo < hi):
            x = np.where(lo > -1.0, lo, np.minimum(hi, 0.0) - 0.5).astype(np.float32)
            probes.append(x)   # x = lo exactly satisfies x >= theta; below hi otherwise
            want.append(leaf)
    assert len(want) * 2 > (1 << depth)   # most leaves are reachable (140/256 at d=8)
    X = np.stack(probes)
    ev = _ev(flat)
    got = ev.leaf_indices(X)[0]
    assert got.tolist() == want
    assert np.array_equal(ev.predict_batch(X), np.array(want, np.float64))


@pytest.mark.parametrize("depth", [9, 11])
def test_acceptance_random_probes_deep(depth):
    # ref tests/test_acceptance.py:149-158: 10k random probes at d = 9 and 11
    from paper_1212_2287_b200.synth import complete_flat
    rng = np.random.default_rng(202 + depth)
    f = 32
    n_int = (1 << depth) - 1
    flat = complete_flat(f, depth, rng.integers(0, f, (1, n_int)), rng.random((1, n_int)),
                         rng.standard_normal((1, 1 << depth)))
    X = rng.random((10000, f), dtype=np.float32)
    s, o = oracle.COracle(flat.arrays()).score(X, threads=4, with_ordinals=True)
    ev = _ev(flat)
    assert np.array_equal(ev.leaf_indices(X), o.astype(np.int64))
    assert np.array_equal(ev.predict_batch(X), s)


def test_depth_boundary_per_strategy():
    # ref tests/test_evaluators.py:50-62: predicated kinds stop at MAX_DEPTH,
    # linked kinds walk deeper trees
    from paper_1212_2287_b200 import (DepthLimitError, Ensemble, Node, StrategyKind, Tree, build,
                                      reference_predict)

    def chain(depth):
        node = Node.leaf(1.0)
        for level in range(depth):
            node = Node.internal(level % 2, 0.5 / (level + 2), node, Node.leaf(2.0 + level))
        return Tree(node)
    build(Ensemble(2, [chain(12)]), StrategyKind.PREDICATED)
    ens17 = Ensemble(2, [chain(17)])
    with pytest.raises(DepthLimitError):
        build(ens17, StrategyKind.PREDICATED)
    with pytest.raises(DepthLimitError):
        build(ens17, StrategyKind.VPREDICATED, 8)
    rng = np.random.default_rng(17)
    X = rng.random((300, 2), dtype=np.float32) * 0.3
    for kind in (StrategyKind.HEAP_LINKED, StrategyKind.COMPACT_LINKED, StrategyKind.CONTIGUOUS):
        ev = build(ens17, kind)
        x = np.full(2, 0.9, dtype=np.float32)
        assert ev.predict(x) == reference_predict(ens17, x)
        got = ev.predict_batch(X)
        assert got.tolist() == [reference_predict(ens17, X[i]) for i in range(len(X))]
        with pytest.raises(DepthLimitError):
            ev.leaf_indices(X)
    deep31 = Ensemble(2, [chain(31)])
    assert build(deep31, "heap_linked").predict(np.zeros(2, np.float32)) == \
        reference_predict(deep31, np.zeros(2, np.float32))
    with pytest.raises(DepthLimitError):
        build(Ensemble(2, [chain(32)]), "heap_linked")


def _fuzz_case(rng):
    """A random ensemble mixing every layout the packer chooses: complete
    trees of assorted depths (streamed), pruned trees (irregular kernel),
    single leaves, and occasionally feature counts too wide for a tile."""
    from paper_1212_2287_b200 import Ensemble
    f = int(rng.choice([1, 3, 17, 136, 700, 3000]))
    trees = []
    for _ in range(int(rng.integers(1, 40))):
        kind = rng.random()
        if kind < 0.45:
            tree = _rand_complete(rng, int(rng.integers(0, 11)), f)
        elif kind < 0.9:
            tree = _rand_unbalanced(rng, int(rng.integers(1, 15)), f, prune=float(rng.uniform(0.1, 0.6)))
        else:
            tree = _rand_complete(rng, 0, f)
        w = float(rng.choice([1.0, -1.0, 0.0, rng.uniform(-2, 2)]))
        trees.append((tree, w))
    n = int(rng.choice([1, 31, 33, 200, 1500]))
    X = rng.random((n, f), dtype=np.float32)
    X[rng.random(X.shape) < 0.2] = 0.0
    X[rng.random(X.shape) < 0.01] = -0.0
    return Ensemble(f, trees), X


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_mixed_models(seed):
    rng = np.random.default_rng(1000 + seed)
    ens, X = _fuzz_case(rng)
    s, o = oracle.COracle(ens.flat().arrays()).score(X, threads=2, with_ordinals=True)
    ev = _ev(ens)
    assert np.array_equal(ev.predict_batch(X), s)
    assert np.array_equal(ev.leaf_indices(X), o.astype(np.int64))


@pytest.mark.parametrize("split", [None, "4"])
def test_tree_split_across_segments(split, monkeypatch):
    """Small-batch tree split inside a multi-segment model: each complete
    segment's fold continues (accumulate) the sum of the segments before it."""
    from paper_1212_2287_b200 import Ensemble
    if split:
        monkeypatch.setenv("TS_SPLIT", split)
    rng = np.random.default_rng(77)
    f = 40
    trees = [(_rand_complete(rng, 8, f), float(rng.uniform(0.5, 1.5))) for _ in range(120)]
    trees += [(_rand_unbalanced(rng, 9, f), 1.0) for _ in range(15)]
    trees += [(_rand_complete(rng, 6, f), -0.5) for _ in range(200)]
    ens = Ensemble(f, trees)
    X = rng.random((500, f), dtype=np.float32)
    s, o = oracle.COracle(ens.flat().arrays()).score(X, threads=4, with_ordinals=True)
    ev = _ev(ens)
    assert ev.model.info["num_segments"] >= 3
    assert np.array_equal(ev.predict_batch(X), s)
    assert np.array_equal(ev.leaf_indices(X), o.astype(np.int64))


@pytest.mark.parametrize("x_pinned,out_pinned", [(True, True), (True, False), (False, True),
                                                  (False, False)])
def test_host_path_pinned_and_pageable(x_pinned, out_pinned):
    """ts_score_host stages pageable buffers through pinned memory and uses
    pinned caller buffers directly; every combination scores identically,
    over several chunks and the halving tail pieces."""
    import torch
    from paper_1212_2287_b200.synth import complete_flat
    rng = np.random.default_rng(5)
    T, d, F = 64, 6, 300                        # 1200-byte rows -> 56k-row chunks
    n_int = (1 << d) - 1
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         rng.standard_normal((T, 1 << d)))
    n = 150_000
    X = rng.random((n, F), dtype=np.float32)
    xs = torch.from_numpy(X).pin_memory().numpy() if x_pinned else X
    out = (torch.empty(n, dtype=torch.float64).pin_memory().numpy() if out_pinned
           else np.empty(n, np.float64))
    ev = _ev(flat)
    ev._predict_into(xs, out)
    ref = oracle.COracle(flat.arrays()).score(X, threads=8)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("ws", ["0", "1"])
@pytest.mark.parametrize("d,T,n,F", [(6, 100, 1000, 136), (8, 90, 5000, 40), (3, 37, 70, 13),
                                     (9, 20, 300, 30), (12, 5, 100, 17), (1, 9, 33, 5),
                                     (8, 40, 20000, 24), (6, 50, 3000, 300), (2, 30, 500, 1),
                                     (2, 7, 3000, 3), (5, 64, 777, 2), (7, 33, 4100, 9)])
def test_warp_split_kernel(ws, d, T, n, F, monkeypatch):
    """k_stream_ws (32-row tiles, four walker warps splitting each chunk's
    trees, an accumulator warp folding leaves in tree order) forced on and off
    over depths 1-12, ragged row counts, F not a multiple of 4, more tiles
    than CTAs: scores and ordinals identical to the oracle."""
    from paper_1212_2287_b200.synth import complete_flat
    monkeypatch.setenv("TS_WS", ws)
    rng = np.random.default_rng(d * 1000 + n)
    n_int = (1 << d) - 1
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         rng.standard_normal((T, 1 << d)), weights=rng.uniform(-1.5, 1.5, T))
    x = rng.random((n, F), dtype=np.float32)
    x[:, : F // 3] = np.round(x[:, : F // 3] * 8) / 8        # exact ties
    ev = _ev(flat)
    s, o = oracle.COracle(flat.arrays()).score(x, threads=4, with_ordinals=True)
    assert np.array_equal(ev.predict_batch(x), s)
    assert np.array_equal(ev.leaf_indices(x), o.astype(np.int64))


def test_warp_split_strided_and_accumulate(monkeypatch):
    """k_stream_ws on a strided device view (ld > F) inside a multi-segment
    model (later segments continue the running sums: accumulate)."""
    import torch
    from paper_1212_2287_b200 import Ensemble
    monkeypatch.setenv("TS_WS", "1")
    rng = np.random.default_rng(5)
    f = 24
    trees = [(_rand_complete(rng, 7, f), float(rng.uniform(0.5, 1.5))) for _ in range(50)]
    trees += [(_rand_unbalanced(rng, 9, f), 1.0) for _ in range(7)]
    trees += [(_rand_complete(rng, 5, f), -0.25) for _ in range(60)]
    ens = Ensemble(f, trees)
    X = rng.random((777, f + 5), dtype=np.float32)
    s = oracle.COracle(ens.flat().arrays()).score(np.ascontiguousarray(X[:, :f]), threads=4)
    ev = _ev(ens)
    assert ev.model.info["num_segments"] >= 3
    xd = torch.from_numpy(X).cuda()[:, :f]
    assert np.array_equal(ev.score_device(xd).cpu().numpy(), s)


def test_concurrent_callers_share_one_model():
    """The reference's evaluators are immutable and reentrant:
    twelve host threads score through ONE model at once -- host buffers
    (ts_score_host, its staging under a lock) and device tensors on their own
    streams, batch sizes that pick the warp-split, the two-pass split and the
    full kernel -- and every result equals the oracle.  (It caught the
    two-pass split writing rows past n into the next pool allocation.)"""
    import threading

    import torch
    from paper_1212_2287_b200.synth import complete_flat
    rng = np.random.default_rng(11)
    T, d, F = 400, 7, 50
    n_int = (1 << d) - 1
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         rng.standard_normal((T, 1 << d)), weights=rng.uniform(0.5, 1.5, T))
    ev = _ev(flat)
    ref = oracle.COracle(flat.arrays())
    sizes = [37, 1000, 3000, 9000, 30000, 200, 5000, 60000, 130, 700, 2100, 4999]
    xs = [rng.random((n, F), dtype=np.float32) for n in sizes]
    want = [ref.score(x, threads=2) for x in xs]
    errors = []

    def worker(i):
        try:
            stream = torch.cuda.Stream()
            for rep in range(5):
                if (i + rep) % 2:
                    got = ev.predict_batch(xs[i])
                else:
                    with torch.cuda.stream(stream):
                        xd = torch.from_numpy(xs[i]).cuda()
                        got = ev.score_device(xd).cpu().numpy()
                if not np.array_equal(got, want[i]):
                    errors.append((i, rep))
        except Exception as e:  # noqa: BLE001
            errors.append((i, repr(e)))

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(len(sizes))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert errors == []


@pytest.mark.parametrize("env", [("TS_WS", "1"), ("TS_SPLIT", "3"), ("TS_SPLIT", "0")])
@pytest.mark.parametrize("n,bad_row", [(100, 0), (100, 99), (3000, 2999), (3000, 1500)])
def test_nonfinite_flagged_on_every_kernel_path(env, n, bad_row, monkeypatch):
    """A NaN / inf anywhere in the batch raises ValueError whichever complete-
    tree kernel stages the rows (warp-split, two-pass split, one-pass), on
    the host path and on a CUDA tensor; clean rows still score exactly."""
    import torch
    from paper_1212_2287_b200.synth import complete_flat
    monkeypatch.setenv(*env)
    rng = np.random.default_rng(n + bad_row)
    T, d, F = 60, 6, 20
    n_int = (1 << d) - 1
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         rng.standard_normal((T, 1 << d)))
    ev = _ev(flat)
    x = rng.random((n, F), dtype=np.float32)
    assert np.array_equal(ev.predict_batch(x), oracle.COracle(flat.arrays()).score(x, threads=4))
    for bad in (np.nan, np.inf, -np.inf):
        xb = x.copy()
        xb[bad_row, (bad_row * 7) % F] = bad
        with pytest.raises(ValueError, match="non-finite"):
            ev.predict_batch(xb)
        with pytest.raises(ValueError, match="non-finite"):
            ev.predict_batch(torch.from_numpy(xb).cuda())


@pytest.mark.parametrize("d,T,n", [(11, 37, 700), (12, 23, 530), (12, 3, 40), (12, 180, 300)])
def test_global_leaf_depths(d, T, n):
    """Depths >= 11 stream only node parts and add each group's leaves (read
    from global memory) after the next group's walk: many chunks, a pending
    group carried across chunks and tiles, non-unit weights, a following
    segment continuing the sums -- scores and ordinals identical to the oracle."""
    from paper_1212_2287_b200 import Ensemble
    from paper_1212_2287_b200.synth import complete_flat
    rng = np.random.default_rng(d * 100 + T)
    F = 33
    n_int = (1 << d) - 1
    deep = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         rng.standard_normal((T, 1 << d)), weights=rng.uniform(-2, 2, T))
    ens = deep.to_ensemble()
    mixed = Ensemble(F, list(ens.trees) + [(_rand_complete(rng, 6, F), 0.75) for _ in range(9)])
    x = rng.random((n, F), dtype=np.float32)
    x[:, :5] = np.round(x[:, :5] * 16) / 16                   # exact ties
    for model in (deep, mixed.flat()):
        ev = _ev(model)
        s, o = oracle.COracle(model.arrays()).score(x, threads=4, with_ordinals=True)
        assert np.array_equal(ev.predict_batch(x), s)
        assert np.array_equal(ev.leaf_indices(x), o.astype(np.int64))


@pytest.mark.parametrize("d", [7, 8])
def test_wave_tail_on_warp_split_kernel(d):
    """Past one full wave of 128-row tiles, the last partial wave's rows run
    on k_stream_ws (d = 7-8): scores, ordinals and a following segment's
    continued sums identical to the oracle across the split row."""
    import torch
    from paper_1212_2287_b200 import Ensemble
    from paper_1212_2287_b200.synth import complete_flat
    rng = np.random.default_rng(d)
    T, F = 24, 30
    n_int = (1 << d) - 1
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         rng.standard_normal((T, 1 << d)), weights=rng.uniform(0.5, 1.5, T))
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = 2 * sms * 128 + 777                      # one full wave + a short tail
    x = rng.random((n, F), dtype=np.float32)
    mixed = Ensemble(F, list(flat.to_ensemble().trees) + [(_rand_complete(rng, 5, F), -0.5)])
    for model in (flat, mixed.flat()):
        ev = _ev(model)
        s, o = oracle.COracle(model.arrays()).score(x, threads=8, with_ordinals=True)
        assert np.array_equal(ev.predict_batch(x), s)
        assert np.array_equal(ev.leaf_indices(x), o.astype(np.int64))


def test_concurrent_host_pipelines_overlap():
    """Host-buffer calls sharing one model run their chunked H2D/score/D2H
    pipelines concurrently (one HostScratch lease per caller, ts_capi.cpp
    ScratchLease), each bit-exact: 6 threads, multi-chunk batches (> 16 MB,
    pageable and pinned inputs)."""
    import threading
    import torch
    from paper_1212_2287_b200.synth import complete_flat
    rng = np.random.default_rng(11)
    T, d, F = 50, 6, 136
    n_int = (1 << d) - 1
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         rng.standard_normal((T, 1 << d)))
    ev = _ev(flat)
    ref = oracle.COracle(flat.arrays())
    xs = [rng.random((40_000 + 997 * i, F), dtype=np.float32) for i in range(6)]
    xs[1] = torch.from_numpy(xs[1]).pin_memory().numpy()
    want = [ref.score(x, threads=4) for x in xs]
    errors = []
    barrier = threading.Barrier(len(xs))

    def worker(i):
        try:
            barrier.wait()
            for _ in range(3):
                if not np.array_equal(ev.predict_batch(xs[i]), want[i]):
                    errors.append(i)
        except Exception as e:  # noqa: BLE001
            errors.append((i, repr(e)))

    ts_ = [threading.Thread(target=worker, args=(i,)) for i in range(len(xs))]
    for t in ts_:
        t.start()
    for t in ts_:
        t.join()
    assert errors == []


@pytest.mark.parametrize("n", [1, 2, 31, 120, 1927, 1928, 5000])
def test_host_direct_path_boundary(n):
    """Host batches up to 1 MB of rows take the zero-copy path (mapped pinned
    rows read by the kernel, scores written back over PCIe, ts_capi.cpp
    score_host_direct); larger ones the chunked copy pipeline.  Both sides of
    the boundary (F=136: 1927 / 1928 rows) bit-exact, mixed-depth model (two
    segments: the second accumulates into the mapped output), non-finite
    input still raises."""
    from paper_1212_2287_b200.synth import complete_flat
    from paper_1212_2287_b200.model import FlatModel
    rng = np.random.default_rng(n)
    F = 136
    parts = []
    for d, T in ((4, 30), (7, 20)):
        n_int = (1 << d) - 1
        parts.append(complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                                   rng.standard_normal((T, 1 << d))))
    a, b = parts
    off = np.concatenate([a.tree_off[:-1], b.tree_off + a.tree_off[-1]])
    flat = FlatModel(F, off, np.concatenate([a.weight, b.weight]), np.concatenate([a.fid, b.fid]),
                     np.concatenate([a.value, b.value]), np.concatenate([a.left, b.left]),
                     np.concatenate([a.right, b.right]))
    ev = _ev(flat)
    x = rng.random((n, F), dtype=np.float32)
    ref = oracle.COracle(flat.arrays()).score(x)
    for _ in range(3):
        assert np.array_equal(ev.predict_batch(x), ref)
    if n <= 121:
        assert ev.predict(x[0]) == ref[0]
    x[n // 2, 7] = np.inf
    with pytest.raises(ValueError):
        ev.predict_batch(x)
    x[n // 2, 7] = 0.5
    assert np.array_equal(ev.predict_batch(x), oracle.COracle(flat.arrays()).score(x))


@pytest.mark.parametrize("depth", [11, 12])
@pytest.mark.parametrize("F", [40, 300])
def test_deep_levels_fid_widths(depth, F):
    """Global-leaf depths (>= 11: node parts streamed, leaves read from L2)
    with 1- and 2-byte deep fids (F > 256): scores and every per-tree ordinal
    bit-exact, with exact ties (integer-valued features and thresholds)."""
    import torch
    from paper_1212_2287_b200.synth import complete_flat
    rng = np.random.default_rng(depth * 1000 + F)
    T, n = 24, 3000
    n_int = (1 << depth) - 1
    flat = complete_flat(F, depth, rng.integers(0, F, (T, n_int)),
                         rng.integers(0, 8, (T, n_int)).astype(np.float32),
                         rng.standard_normal((T, 1 << depth)))
    X = rng.integers(0, 8, (n, F)).astype(np.float32)
    s, o = oracle.COracle(flat.arrays()).score(X, threads=4, with_ordinals=True)
    ev = _ev(flat)
    assert np.array_equal(ev.predict_batch(X), s)
    assert np.array_equal(ev.leaf_indices(X), o.astype(np.int64))
    xd = torch.from_numpy(X).cuda()
    assert np.array_equal(ev.score_device(xd).cpu().numpy(), s)


def _rank_case(rng, depth, F, T, ties=False, weights=False):
    """Complete trees with optional exact ties, -0.0 / +0.0 and subnormal
    thresholds, and weights != 1."""
    from paper_1212_2287_b200.synth import complete_flat
    n_int = (1 << depth) - 1
    fids = rng.integers(0, F, (T, n_int))
    if ties:
        thr = rng.integers(-3, 4, (T, n_int)).astype(np.float32)
        thr[rng.random((T, n_int)) < 0.1] = np.float32(-0.0)
    else:
        thr = rng.random((T, n_int), dtype=np.float32)
        thr[rng.random((T, n_int)) < 0.02] = np.float32(1e-40)   # subnormal
    leaves = rng.standard_normal((T, 1 << depth))
    w = rng.uniform(0.25, 2.0, T) if weights else None
    return complete_flat(F, depth, fids, thr, leaves, weights=w)


@pytest.mark.parametrize("depth", [1, 3, 6, 8, 11, 12, 13, 14])
@pytest.mark.parametrize("ties", [False, True])
def test_rank_layout_forced_all_depths(depth, ties, monkeypatch):
    """The rank layout (ts_rank.cu: thresholds -> per-feature ranks, instances
    ranked by the k_rank pre-pass, 4-byte records) forced at every depth with
    TS_RANK_MIN_DEPTH=1: scores and every per-tree ordinal bit-exact against
    the oracle, with exact ties, -0.0/+0.0 and subnormal thresholds, weights
    != 1, ragged n, host and device inputs."""
    import torch
    monkeypatch.setenv("TS_RANK_MIN_DEPTH", "1")
    rng = np.random.default_rng(31 * depth + ties)
    F, T = 40, 37
    flat = _rank_case(rng, depth, F, T, ties=ties, weights=True)
    n = 1000 + 77 * depth
    if ties:
        X = rng.integers(-3, 4, (n, F)).astype(np.float32)
        X[rng.random((n, F)) < 0.05] = np.float32(-0.0)
    else:
        X = rng.random((n, F), dtype=np.float32)
        X[rng.random((n, F)) < 0.01] = np.float32(1e-40)
    s, o = oracle.COracle(flat.arrays()).score(X, threads=4, with_ordinals=True)
    ev = _ev(flat)
    assert ev.model.info["rank_trees"] == T
    assert np.array_equal(ev.predict_batch(X), s)
    assert np.array_equal(ev.leaf_indices(X), o.astype(np.int64))
    assert np.array_equal(ev.score_device(torch.from_numpy(X).cuda()).cpu().numpy(), s)


@pytest.mark.parametrize("depth", [2, 7, 10, 12, 13])
@pytest.mark.parametrize("kind", ["narrow", "wide", "zeros"])
@pytest.mark.parametrize("n,ctas", [(1, None), (700, None), (700, "5"), (5000, "37")])
def test_rank_layout_balanced_split(depth, kind, n, ctas, monkeypatch):
    """Balanced tree split on the rank walk (k_rstream<..., ORD = 2>, the
    same k_combine): tiles shared by several CTAs combined from their partial
    sums when provably exact, else walked again from the rank records and the
    row's rank tile; unit weights, scores against the oracle bit for bit, also
    continuing the running sum of a first segment."""
    import torch
    from paper_1212_2287_b200.synth import complete_flat
    monkeypatch.setenv("TS_RANK_MIN_DEPTH", "1")
    monkeypatch.setenv("TS_SK", "1")
    if ctas:
        monkeypatch.setenv("TS_SK_CTAS", ctas)
    rng = np.random.default_rng(depth * 131 + n + len(kind))
    F = 40
    T = max(12, 400 >> max(0, depth - 6))
    n_int = (1 << depth) - 1
    thr = rng.random((T, n_int))
    thr[rng.random((T, n_int)) < 0.1] = 0.5
    flat = complete_flat(F, depth, rng.integers(0, F, (T, n_int)), thr,
                         _leaf_table(kind, rng, T, depth))
    X = rng.random((n, F), dtype=np.float32)
    X[::5, ::3] = 0.5
    s, o = oracle.COracle(flat.arrays()).score(X, threads=4, with_ordinals=True)
    ev = _ev(flat)
    assert ev.model.info["rank_trees"] == T
    assert np.array_equal(ev.predict_batch(X).view(np.uint64), s.view(np.uint64))
    xd = torch.from_numpy(X).cuda()
    out = torch.full((n,), 0.375, dtype=torch.float64, device="cuda")
    ev.model.score(xd, out=out, accumulate=True)   # continues a running sum
    assert np.array_equal(ev.leaf_indices(X), o.astype(np.int64))
    # tree-order sum started from 0.375: redo on the host in f64, tree by tree
    leaves = flat.value.astype(np.float64)
    exp = np.full(n, 0.375)
    for t in range(T):
        base = int(flat.tree_off[t])
        node = np.zeros(n, np.int64)
        for _ in range(depth):
            f = flat.fid[base + node]
            go = X[np.arange(n), f] >= flat.value[base + node]
            node = np.where(go, flat.right[base + node], flat.left[base + node])
        exp = exp + leaves[base + node]
    assert np.array_equal(out.cpu().numpy().view(np.uint64), exp.view(np.uint64))
    ev.close()


def test_rank_layout_default_choice_and_opt_out(monkeypatch):
    """By default a depth takes the rank layout only with enough trees for
    the walk's savings to pay for the instance-rank pre-pass (ts_pack.cpp
    kRankMinTrees x F / 136: 150 at d = 13, 500 at d = 12, never below
    d = 10): here the 50 depth-13 trees do (F = 40), the 6 depth-12 and 9
    depth-8 trees do not.  TS_RANK=0 and rank=False keep the fp32 layout; all
    give the same bits, and a non-finite input is still flagged."""
    from paper_1212_2287_b200 import GpuModel
    from paper_1212_2287_b200.model import FlatModel
    monkeypatch.delenv("TS_RANK_MIN_DEPTH", raising=False)
    monkeypatch.delenv("TS_RANK", raising=False)
    rng = np.random.default_rng(5)
    F = 40
    parts = [_rank_case(rng, 13, F, 50), _rank_case(rng, 12, F, 6), _rank_case(rng, 8, F, 9)]
    offs, acc = [], 0
    for p_ in parts:
        offs.append(p_.tree_off[:-1] + acc)
        acc += p_.tree_off[-1]
    off = np.concatenate(offs + [np.array([acc])])
    cat = lambda k: np.concatenate([getattr(p_, k) for p_ in parts])  # noqa: E731
    flat = FlatModel(F, off, cat("weight"), cat("fid"), cat("value"), cat("left"), cat("right"))
    X = rng.random((3000, F), dtype=np.float32)
    ref = oracle.COracle(flat.arrays()).score(X, threads=4)
    ev = _ev(flat)
    assert ev.model.info["rank_trees"] == 50
    assert np.array_equal(ev.predict_batch(X), ref)
    assert GpuModel(flat, 0, rank=False).info["rank_trees"] == 0
    monkeypatch.setenv("TS_RANK", "0")
    ev0 = _ev(flat)
    assert ev0.model.info["rank_trees"] == 0
    assert np.array_equal(ev0.predict_batch(X), ref)
    monkeypatch.delenv("TS_RANK")
    X[1234, 17] = np.nan
    with pytest.raises(ValueError):
        ev.predict_batch(X)


def test_rank_layout_segments_chunks_and_host_paths(monkeypatch):
    """The rank path continuing a partial sum (a rank segment after an fp32
    one), rows beyond one 2M-row rank chunk (ts_rank.cu kRankChunkRows: the
    ordinals' row offset, the sums' continuation), and the host small-batch
    path (mapped rows copied to the device before the pre-pass): bit-exact."""
    import torch
    from paper_1212_2287_b200.model import FlatModel
    monkeypatch.setenv("TS_RANK_MIN_DEPTH", "12")
    monkeypatch.delenv("TS_RANK", raising=False)
    rng = np.random.default_rng(77)
    # a depth-6 fp32 segment then a depth-12 rank segment (forced from d = 12)
    F = 50
    a = _rank_case(rng, 6, F, 7, weights=True)
    b = _rank_case(rng, 12, F, 3, weights=True)
    off = np.concatenate([a.tree_off[:-1], b.tree_off + a.tree_off[-1]])
    flat = FlatModel(F, off, np.concatenate([a.weight, b.weight]), np.concatenate([a.fid, b.fid]),
                     np.concatenate([a.value, b.value]), np.concatenate([a.left, b.left]),
                     np.concatenate([a.right, b.right]))
    ev = _ev(flat)
    assert ev.model.info["rank_trees"] == 3
    for n in (1, 100, 5000):
        X = rng.random((n, F), dtype=np.float32)
        s, o = oracle.COracle(flat.arrays()).score(X, threads=4, with_ordinals=True)
        assert np.array_equal(ev.predict_batch(X), s)          # host path (mapped if small)
        assert np.array_equal(ev.leaf_indices(X), o.astype(np.int64))
    # more rows than one rank chunk: small trees forced onto the rank layout
    monkeypatch.setenv("TS_RANK_MIN_DEPTH", "1")
    F2, n2 = 4, (2 << 20) + 777
    flat2 = _rank_case(rng, 3, F2, 5)
    ev2 = _ev(flat2)
    assert ev2.model.info["rank_trees"] == 5
    X2 = torch.rand((n2, F2), device="cuda")
    ords = torch.empty((5, n2), dtype=torch.int16, device="cuda")
    got = ev2.model.score(X2, ordinals=ords).cpu().numpy()
    rows = np.concatenate([np.arange(0, 300), np.arange((2 << 20) - 300, n2)])
    xs = X2[torch.from_numpy(rows).cuda()].cpu().numpy()
    s2, o2 = oracle.COracle(flat2.arrays()).score(xs, threads=4, with_ordinals=True)
    assert np.array_equal(got[rows], s2)
    assert np.array_equal(ords.cpu().numpy().view(np.uint16)[:, rows], o2)


def test_rank_layout_several_rank_spaces(monkeypatch):
    """More distinct thresholds per feature than 15-bit ranks hold: the
    packer splits the rank trees into consecutive rank spaces (one pre-pass
    and segment each, the later ones continuing the running sums); scores
    and ordinals bit-exact."""
    from paper_1212_2287_b200.synth import complete_flat
    monkeypatch.setenv("TS_RANK_MIN_DEPTH", "1")
    rng = np.random.default_rng(123)
    F, d, T = 4, 10, 200          # ~256 thresholds per feature per tree: ~51k in all
    n_int = (1 << d) - 1
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         rng.standard_normal((T, 1 << d)), weights=rng.uniform(0.5, 1.5, T))
    ev = _ev(flat)
    assert ev.model.info["rank_trees"] == T
    assert ev.model.info["num_segments"] >= 2
    X = rng.random((3000, F), dtype=np.float32)
    s, o = oracle.COracle(flat.arrays()).score(X, threads=4, with_ordinals=True)
    assert np.array_equal(ev.predict_batch(X), s)
    assert np.array_equal(ev.leaf_indices(X), o.astype(np.int64))
