"""Fused cross-GPU running-sum pipeline (``ts_score_pipe``, tree sharding).

Only one GPU is available to the tests, and the pipeline's kernels wait on one
another, so the ranks run ONE AFTER ANOTHER here: rank r's kernel finishes
(publishing every block's sums and flags) before rank r+1's starts, so no
kernel ever waits on a kernel that is not already complete.  The result must
equal single-model scoring bit for bit (same tree-order f64 additions)."""

import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

import oracle
from conftest import has_cuda

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]


def _workload(T=48, d=6, F=136, n=5000, seed=11):
    from paper_1212_2287_b200.synth import complete_flat
    rng = np.random.default_rng(seed)
    n_int = (1 << d) - 1
    flat = complete_flat(F, d, rng.integers(0, F, (T, n_int)), rng.random((T, n_int)),
                         rng.standard_normal((T, 1 << d)),
                         weights=rng.uniform(0.5, 1.5, T))
    x = rng.random((n, F), dtype=np.float32)
    return flat, x


def _run_sequential(flat, x, world, epochs=2):
    import torch
    from paper_1212_2287_b200.distributed import tree_shards
    from paper_1212_2287_b200.evaluator import GpuModel, PipeBuffers
    shards = tree_shards(flat.depths(), world)
    models = [GpuModel(flat.subset(a, b), 0, rank=False) for a, b in shards]
    bufs = [None] + [PipeBuffers(x.shape[0], 0) for _ in range(world - 1)]
    xd = torch.from_numpy(x).cuda()
    outs = []
    for epoch in range(1, epochs + 1):
        out = torch.full((x.shape[0],), np.nan, dtype=torch.float64, device="cuda")
        for r, m in enumerate(models):
            kw = {}
            if r > 0:
                kw.update(sums_in=bufs[r].sums, flags_in=bufs[r].flags)
            if r < world - 1:
                kw.update(sums_out=bufs[r + 1].sums, flags_out=bufs[r + 1].flags)
            m.score_pipe(xd, out, epoch=epoch, **kw)
            torch.cuda.synchronize()
        outs.append(out.cpu().numpy())
        xd = xd.flip(0).contiguous()      # epoch 2 scores different rows
    return outs


@pytest.mark.parametrize("world", [2, 3])
def test_pipe_sequential_bit_exact(world):
    from paper_1212_2287_b200 import build_gpu
    flat, x = _workload()
    outs = _run_sequential(flat, x, world)
    ev = build_gpu(flat.to_ensemble())
    assert np.array_equal(outs[0], ev.predict_batch(x))
    assert np.array_equal(outs[1], ev.predict_batch(x[::-1].copy()))
    ref = oracle.COracle(flat.arrays()).score(x, threads=4)
    assert np.array_equal(outs[0], ref)


@pytest.mark.parametrize("d,T", [(10, 20), (12, 9)])
def test_pipe_ragged_rows_and_deep_trees(d, T):
    # d = 12: global-leaf mode -- the deferred leaves of the last K-group must
    # be in the running sums before they are published to the next rank
    flat, x = _workload(T=T, d=d, F=40, n=33 * 32 + 7, seed=5)
    outs = _run_sequential(flat, x, 2, epochs=1)
    assert np.array_equal(outs[0], oracle.COracle(flat.arrays()).score(x, threads=4))


def test_pipe_rejects_irregular_models():
    import torch
    from conftest import load_golden
    from paper_1212_2287_b200.evaluator import GpuModel
    ens, g = load_golden("deep_unbalanced")       # depths up to 16: not streamable
    m = GpuModel(ens, 0)
    with pytest.raises(RuntimeError, match=r"\(7\)"):
        m.score_pipe(torch.from_numpy(g["X"]).cuda())


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist
        from paper_1212_2287_b200.distributed import ShardedScorer
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        flat, x = _workload(n=4099)
        sc = ShardedScorer("tree-p2p", flat, x.shape[0], device=0, serialize=True)
        xd = torch.from_numpy(x).cuda()
        res = []
        for _ in range(2):                      # two epochs through the same buffers
            out = torch.zeros(x.shape[0], dtype=torch.float64, device="cuda")
            sc(xd, out)
            res.append(out.cpu().numpy())
        sc.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))


def test_pipe_two_processes_cuda_ipc():
    """ShardedScorer("tree-p2p") across two processes (CUDA IPC handles over
    gloo), serialized on the one GPU."""
    flat, x = _workload(n=4099)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert not isinstance(res[r], str), res[r]
    ref = oracle.COracle(flat.arrays()).score(x, threads=4)
    assert np.array_equal(res[1][0], ref)
    assert np.array_equal(res[1][1], ref)


def _reduce_worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist
        from paper_1212_2287_b200.distributed import NcclReducer
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        red = NcclReducer(0)
        part = torch.arange(1000, dtype=torch.float64, device="cuda") * 0.5
        out = red.reduce(part)
        red.wait(timeout_ms=60_000)       # polls ncclCommGetAsyncError
        torch.cuda.synchronize()
        red.close()
        dist.destroy_process_group()
        q.put((rank, out.cpu().numpy()))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))


def test_native_nccl_reduce_world1():
    """ts_reduce_partials (the C ABI's NCCL f64 sum-reduce) through its own
    communicator; one GPU, so world size 1 (the sum is the partial itself)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_reduce_worker, args=(0, 1, _free_port(), q))
    p.start()
    rank, res = q.get(timeout=300)
    p.join(timeout=60)
    assert not isinstance(res, str), res
    assert np.array_equal(res, np.arange(1000) * 0.5)
