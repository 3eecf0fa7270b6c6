"""Synthetic BASELINE workloads: shapes, distributions and determinism."""

import numpy as np

from paper_1212_2287_b200 import synth


def test_hash_uniform_properties():
    a = synth.hash_uniform(7, 0, 1000, 13)
    b = synth.hash_uniform(7, 500, 500, 13)
    assert np.array_equal(a[500:], b)                 # any row window reproduces
    assert a.dtype == np.float32 and a.min() >= 0 and a.max() < 1
    assert abs(a.mean() - 0.5) < 0.01
    z = synth.hash_uniform(7, 0, 2000, 50, zero_prob=0.4)
    assert abs((z == 0).mean() - 0.4) < 0.01
    assert np.all((z * 2 ** 24) == np.floor(z * 2 ** 24))   # exact 24-bit grid


def test_config_shapes_small():
    w0 = synth.config0(n=100)
    assert w0.x.shape == (100, 136) and w0.flat.num_trees == 100
    w1 = synth.config1(n=2000, trees=20)
    kinds = w1.meta["column_kinds"]
    assert (kinds == 0).sum() == 95 and (kinds == 1).sum() == 27 and (kinds == 2).sum() == 14
    counts = w1.x[:, kinds == 2]
    assert np.all(counts == np.round(counts)) and counts.max() <= 50
    ens = w1.flat.to_ensemble()
    assert all(t.depth == 8 for t, _ in ens.trees)


def test_irregular_trees():
    flat = synth.irregular_flat(3, 50, 700)
    ens = flat.to_ensemble()
    depths = [t.depth for t, _ in ens.trees]
    assert all(t.leaf_count == 64 for t, _ in ens.trees)
    assert max(depths) <= 16 and min(depths) >= 6
    assert 8 < np.mean(depths) < 15
