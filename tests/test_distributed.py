"""Multi-process sharding logic on the CPU (gloo, world size 2), with the
oracle standing in for the per-rank CUDA scorer."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1212_2287_b200 import distributed as D
from paper_1212_2287_b200 import synth


def oracle_scorer(flat):
    tables = oracle.expand(flat.arrays())
    w = flat.weight

    def score(x, out, accumulate=False):
        init = out.numpy() if accumulate else None
        out.copy_(torch.from_numpy(oracle.score(tables, w, x.numpy(), init=init)))
        return out
    return score


def _workload():
    flat = synth.irregular_flat(5, 9, 20, leaves=12, max_depth=7)   # mixed depths
    rng = np.random.default_rng(3)
    x = rng.random((203, 20), dtype=np.float32)
    x[:, :5] = np.round(x[:, :5] * 4) / 4          # exact ties
    return flat, x


def _worker(rank, world, port, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        flat, x = _workload()
        n = x.shape[0]
        if mode.startswith("auto"):
            # auto:<l2 bytes>: the driver picks the mode from the table size;
            # the caller scores the rows the plan gives it
            sc = D.ShardedScorer("auto", flat, n, make_scorer=oracle_scorer, chunk_rows=64,
                                 l2_bytes=int(mode.split(":")[1]))
            a, b = sc.plan.rows
            out = sc(torch.from_numpy(x[a:b]))
            q.put((rank, (sc.plan.mode, sc.plan.rows), out.numpy().copy(), None))
        elif mode == "instance":
            a, b = D.row_shard(n, world, rank)
            p, out = D.run_sharded(mode, flat, torch.from_numpy(x[a:b]), n,
                                   make_scorer=oracle_scorer)
            full = D.gather_scores(out, n)
            q.put((rank, p.rows, out.numpy().copy(), None if full is None else full.numpy()))
        else:
            p, out = D.run_sharded(mode, flat, torch.from_numpy(x), n,
                                   make_scorer=oracle_scorer, chunk_rows=64)
            q.put((rank, p.trees, out.numpy().copy(), None))
    finally:
        dist.destroy_process_group()


def _run(mode, world=2):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _reference():
    flat, x = _workload()
    return oracle.score(oracle.expand(flat.arrays()), flat.weight, x)


def test_tree_shards_balance_and_cover():
    depths = [16, 1, 1, 1, 8, 8, 0, 3, 12, 2]
    for world in (1, 2, 3, 4):
        sh = D.tree_shards(depths, world)
        assert sh[0][0] == 0 and sh[-1][1] == len(depths)
        assert all(a < b for a, b in sh) and all(sh[i][1] == sh[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        D.tree_shards([1, 2], 3)
    assert [D.row_shard(10, 3, r) for r in range(3)] == [(0, 3), (3, 6), (6, 10)]


def test_flat_subset_roundtrip():
    flat, x = _workload()
    a = oracle.score(oracle.expand(flat.subset(0, 4).arrays()), flat.weight[:4], x)
    full = oracle.score(oracle.expand(flat.arrays()), flat.weight, x)
    b = oracle.score(oracle.expand(flat.subset(4, 9).arrays()), flat.weight[4:], x, init=a)
    assert np.array_equal(b, full)     # continuing the sum is bit-exact


def test_instance_sharding_gloo():
    res = _run("instance")
    ref = _reference()
    for rank, (a, b), out, _ in res:
        assert np.array_equal(out, ref[a:b])
    assert np.array_equal(res[0][3], ref)


def test_tree_pipeline_bit_exact_gloo():
    res = _run("tree-pipeline")
    ref = _reference()
    assert np.array_equal(res[-1][2], ref)          # last rank holds the final sums


def test_tree_reduce_gloo():
    res = _run("tree-reduce")
    ref = _reference()
    np.testing.assert_allclose(res[0][2], ref, rtol=1e-12, atol=1e-12)


def test_table_bytes_and_choose_mode():
    from paper_1212_2287_b200.synth import complete_flat
    rng = np.random.default_rng(0)
    T, d, F = 20, 10, 30
    n_int = (1 << d) - 1
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         rng.standard_normal((T, 1 << d)))
    per_tree = 8 * n_int + 4 * (1 << d)        # 8-B nodes + 4-B leaves
    assert D.table_bytes(flat) == T * per_tree
    # config 4b: 20,000 depth-10 trees = 245.6 MB of tables, beyond a 126 MB L2
    assert 20_000 * per_tree == 245_600_000
    irr, _ = _workload()
    nodes = np.diff(irr.tree_off)
    assert D.table_bytes(irr) == int((nodes * 8).sum())   # no complete tree among them
    assert D.choose_mode(flat, T * per_tree) == "instance"
    assert D.choose_mode(flat, T * per_tree - 1) == "tree-reduce"
    assert D.choose_mode(flat, 0, combine="pipeline") == "tree-pipeline"
    with pytest.raises(ValueError):
        D.choose_mode(flat, 0, combine="bogus")


@pytest.mark.parametrize("l2", [1 << 30, 1])
def test_auto_mode_gloo(l2):
    """mode="auto": small tables -> instance shards, tables beyond L2 -> tree
    shards combined by the sum-reduce; both give the reference scores."""
    res = _run(f"auto:{l2}")
    ref = _reference()
    modes = {r[1][0] for r in res}
    if l2 > 1:
        assert modes == {"instance"}
        for rank, (_, (a, b)), out, _ in res:
            assert np.array_equal(out, ref[a:b])
    else:
        assert modes == {"tree-reduce"}
        np.testing.assert_allclose(res[0][2], ref, rtol=1e-12, atol=1e-12)
