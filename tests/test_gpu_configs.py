"""Parity at the BASELINE ensemble sizes (SURVEY 8(c) sampling protocol).

Every BASELINE.json configuration with its FULL ensemble -- config 2 at each
depth with T=1000, config 3 with all 5,000 irregular trees at F=700, config
4a's 64M-row matrix, config 4b's 20,000 depth-10 trees (also tree-sharded) --
scored on the GPU through the C ABI and compared with the C oracle:
scores bit-exact (f64, tree order: ref evaluators.py:529-535) and per-tree
predicated leaf ordinals bit-exact (ref ``batch_kernel`` on
``expand_to_complete``, evaluators.py:90-99, model.py:315-349) on sampled
rows.  Rows for configs 3/4 are generated on the device and reproduced on the
host by ``synth.hash_uniform`` (checked here too)."""

import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

import oracle
from conftest import has_cuda

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]


def _device_rows(w, n=None, row0=0):
    import torch
    from paper_1212_2287_b200 import _lib
    n = w.n if n is None else n
    if w.x is not None:
        return torch.from_numpy(w.x[row0:row0 + n]).cuda()
    x = torch.empty((n, w.f), dtype=torch.float32, device="cuda")
    rc = _lib.load().ts_synth_uniform(x.data_ptr(), n, w.f, w.f, w.hash_seed, row0, w.zero_prob,
                                      torch.cuda.current_stream().cuda_stream)
    assert rc == 0, _lib.last_error()
    return x


def _score_with_ordinals(model, x):
    """(scores f64 [n], ordinals uint16 [T, n]) from one ts_score launch set."""
    import torch
    n = x.shape[0]
    ords = torch.empty((model.num_trees, n), dtype=torch.int16, device="cuda")
    out = model.score(x, ordinals=ords)
    torch.cuda.synchronize()
    return out.cpu().numpy(), ords.cpu().numpy().view(np.uint16)


def _check(flat, host, scores, ords=None):
    c = oracle.COracle(flat.arrays())
    if ords is None:
        ref = c.score(host)
        assert np.array_equal(scores, ref), f"max |err| {np.max(np.abs(scores - ref))}"
        return
    ref, ref_ord = c.score(host, with_ordinals=True)
    assert np.array_equal(scores, ref), f"max |err| {np.max(np.abs(scores - ref))}"
    bad = np.argwhere(ords != ref_ord)
    assert bad.size == 0, f"{len(bad)} ordinals differ, first (tree, row) {bad[:3].tolist()}"


@pytest.mark.parametrize("depth", [3, 4, 6, 8, 10, 12])
def test_config2_full_ensemble(depth):
    """Config 2: T=1000 complete trees per depth, 20k rows, every row's score
    and every (tree, row) ordinal."""
    from paper_1212_2287_b200 import GpuModel, synth
    w = synth.config2(depth, n=20_000)
    assert w.flat.num_trees == 1000
    m = GpuModel(w.flat, 0)
    scores, ords = _score_with_ordinals(m, _device_rows(w))
    _check(w.flat, w.x, scores, ords)
    m.close()


def test_config3_full_ensemble():
    """Config 3: all 5,000 irregular trees (depth <= 16, Zipf fids, F=700,
    40% exact zeros), 20k device-generated rows; ordinals on 4,096 rows."""
    from paper_1212_2287_b200 import GpuModel, synth
    w = synth.config3(n=20_000)
    assert w.flat.num_trees == 5000
    m = GpuModel(w.flat, 0)
    x = _device_rows(w)
    host = w.rows(0, w.n)
    assert np.array_equal(x.cpu().numpy(), host)       # device generator == host
    out = m.score(x).cpu().numpy()
    _check(w.flat, host, out)
    s4, o4 = _score_with_ordinals(m, x[:4096])
    assert np.array_equal(s4, out[:4096])
    _check(w.flat, host[:4096], s4, o4)
    m.close()


def test_config4a_64m_rows_sampled():
    """Config 4a: the full 64M x 136 matrix (34.8 GB) generated on the device
    and scored in one pass; 4,096 rows sampled over the whole range (head,
    tail, random 32-row blocks) against the oracle, ordinals included."""
    import torch
    from paper_1212_2287_b200 import GpuModel, synth
    w = synth.config4a()
    assert w.n == 64_000_000
    m = GpuModel(w.flat, 0)
    x = _device_rows(w)
    out = m.score(x)
    rows = oracle.sample_rows(w.n, 4096, seed=4)
    assert rows[0] == 0 and rows[-1] == w.n - 1
    idx = torch.from_numpy(rows).cuda()
    xs = x.index_select(0, idx)
    got = out.index_select(0, idx).cpu().numpy()
    host = np.concatenate([w.rows(a, k) for a, k in oracle.runs_of(rows)])
    assert np.array_equal(xs.cpu().numpy(), host)
    del x, out
    torch.cuda.empty_cache()
    s, o = _score_with_ordinals(m, xs)
    assert np.array_equal(s, got)               # sample re-scored == full pass
    _check(w.flat, host, got, o)
    m.close()


def test_config4b_full_ensemble():
    """Config 4b: all 20,000 depth-10 trees (245.6 MB of node tables, beyond
    L2); 8,192 rows with every (tree, row) ordinal, plus the full 8M-row pass
    sampled at 1,024 rows."""
    import torch
    from paper_1212_2287_b200 import GpuModel, synth
    w = synth.config4b()
    assert w.flat.num_trees == 20_000
    m = GpuModel(w.flat, 0)
    x = _device_rows(w, 8192)
    s, o = _score_with_ordinals(m, x)
    _check(w.flat, w.rows(0, 8192), s, o)
    del x, o
    xf = _device_rows(w)
    out = m.score(xf)
    rows = oracle.sample_rows(w.n, 1024, seed=41)
    got = out.index_select(0, torch.from_numpy(rows).cuda()).cpu().numpy()
    host = np.concatenate([w.rows(a, k) for a, k in oracle.runs_of(rows)])
    _check(w.flat, host, got)
    m.close()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _shard_worker(rank, world, port, mode, n, q):
    try:
        import torch
        import torch.distributed as dist
        from paper_1212_2287_b200 import synth
        from paper_1212_2287_b200.distributed import ShardedScorer
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        w = synth.config4b(n=n)
        x = _device_rows(w)
        sc = ShardedScorer(mode, w.flat, n, device=0, serialize=True, chunk_rows=2048)
        out = torch.zeros(n, dtype=torch.float64, device="cuda")
        sc(x, out)
        torch.cuda.synchronize()
        res = out.cpu().numpy()
        trees = sc.plan.trees
        sc.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, (trees, res)))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc() + repr(e)))


@pytest.mark.parametrize("mode", ["tree-pipeline", "tree-p2p", "tree-reduce"])
def test_config4b_tree_sharded(mode):
    """Config 4b's 20,000 trees split over two ranks (two processes sharing
    the one GPU; gloo for the host plumbing; the p2p ranks serialised so no
    kernel waits on a kernel that has not run).  The pipelined modes continue
    the running f64 sums across shards: bit-exact.  tree-reduce adds two
    partial sums: within the north star's 1e-5 relative bound."""
    from paper_1212_2287_b200 import synth
    n, world = 4096, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, mode, n, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    assert res[0][0] == (0, res[1][0][0]) and res[1][0][1] == 20_000
    w = synth.config4b(n=n)
    host = w.rows(0, n)
    c = oracle.COracle(w.flat.arrays())
    ref = c.score(host)
    final = res[0][1] if mode == "tree-reduce" else res[world - 1][1]
    if mode == "tree-reduce":
        tol = oracle.score_tolerance(c, host, ref)
        assert np.all(np.abs(final - ref) <= tol)
        assert np.all(np.abs(final - ref) <= tol * 1e-7)    # ~1e-12 of the magnitude
    else:
        assert np.array_equal(final, ref)
