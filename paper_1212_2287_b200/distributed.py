"""Multi-GPU driver: one process per GPU, torch.distributed for the plumbing.

SURVEY.md section 8(e): instances are independent, so the path shards two ways.

* Instance sharding (configs 0-3, 4a): rank r owns the contiguous row range
  :func:`row_shard`; every rank holds the whole packed ensemble; no collective
  touches the data path.  Scores stay sharded (``gather_scores`` collects them
  on one rank when a caller wants them in one place).
* Tree sharding (config 4b, tables beyond L2): rank r owns the contiguous tree
  range :func:`tree_shards` (balanced by sum of depths, global tree order kept)
  and scores ALL rows against it.  Two ways to combine:
    - ``"reduce"``: every rank scores from +0.0 and one NCCL sum
      (``ncclFloat64``, NVLink/NVSwitch) adds the partials.  The cross-shard
      sum order differs from the reference's sequential order, so scores agree
      to ~1e-16 relative, not bit for bit.
    - ``"pipeline"``: row chunks flow rank 0 -> 1 -> ... -> R-1; each rank
      continues the f64 accumulation of the previous shard (``ts_score_ex``
      with ``accumulate``) and sends the running sums on with point-to-point
      NCCL send/recv.  Every addition happens in the reference's tree order,
      so the final scores are bit-identical to single-GPU scoring; the cost is
      (R - 1) chunk times of pipeline fill.
    - ``"p2p"``: the same bit-exact order, fused into the scoring kernel
      (``ts_score_pipe``): each 32-row block of rank r waits on a
      system-scope flag that rank r-1's kernel releases after storing the
      block's running sums straight into rank r's HBM over NVLink (CUDA IPC
      peer pointers).  No NCCL and no host round trip on the data path; the
      transfers overlap the walks block by block.  Needs one process per GPU:
      the ranks' kernels wait on each other, so they must run concurrently
      (``serialize=True`` runs the ranks one after another for tests that
      share one GPU).

The per-rank scorer is injected (``make_scorer``) so the same driver runs on
GPUs (the CUDA library) and, in the CPU test-suite, under ``gloo`` with the
oracle standing in for the kernel.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .model import FlatModel


def _global(group, r: int) -> int:
    """Global rank of ``group``'s rank ``r`` (torch's collectives and
    send/recv take global ranks even when a subgroup is passed)."""
    import torch.distributed as dist
    return dist.get_global_rank(group, r) if group is not None else r


def row_shard(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous rows ``[a, b)`` of rank ``rank`` (sizes differ by at most 1)."""
    return n * rank // world, n * (rank + 1) // world


def tree_shards(depths, world: int) -> list[tuple[int, int]]:
    """Split trees into ``world`` contiguous ranges with balanced sum of depths.

    Node visits per instance are sum(d_t), so balancing the
    depth sum balances the kernel time; every range is non-empty when
    ``len(depths) >= world``.
    """
    depths = np.asarray(depths, dtype=np.float64)
    T = len(depths)
    if world < 1 or T < world:
        raise ValueError(f"cannot split {T} trees over {world} ranks")
    cost = np.maximum(depths, 1.0)          # depth-0 trees still cost a leaf read
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    cuts = [0]
    for r in range(1, world):
        target = cum[-1] * r / world
        c = int(np.searchsorted(cum, target))
        c = min(max(c, cuts[-1] + 1), T - (world - r))
        cuts.append(c)
    cuts.append(T)
    return [(cuts[i], cuts[i + 1]) for i in range(world)]


def table_bytes(flat: FlatModel, depths=None) -> int:
    """Node-table bytes of the packed ensemble (8-byte nodes and
    4-byte leaves over each complete tree's heap; irregular trees keep their
    own nodes as 8-byte child-index records)."""
    d = np.asarray(flat.depths() if depths is None else depths, dtype=np.int64)
    nodes = np.diff(np.asarray(flat.tree_off, dtype=np.int64))
    complete = nodes == (np.int64(2) << d) - 1
    pw = np.int64(1) << d
    per_tree = np.where(complete, (pw - 1) * 8 + pw * 4, nodes * 8)
    return int(per_tree.sum())


def choose_mode(flat: FlatModel, l2_bytes: int, depths=None, combine: str = "reduce") -> str:
    """``"instance"`` while the node tables fit the GPU's L2 (every rank keeps
    the whole ensemble hot), else tree sharding (north star: the NCCL
    sum-reduce variant is for tables beyond L2); ``combine`` picks
    ``"reduce"``, ``"pipeline"`` or ``"p2p"``."""
    if combine not in ("reduce", "pipeline", "p2p"):
        raise ValueError(f"unknown combine {combine!r}")
    return "instance" if table_bytes(flat, depths) <= l2_bytes else f"tree-{combine}"


@dataclass
class ShardPlan:
    mode: str                      # "instance" | "tree-reduce" | "tree-pipeline" | "tree-p2p"
    world: int
    rank: int
    rows: tuple[int, int]          # rows this rank scores
    trees: tuple[int, int]         # trees this rank holds


def plan(mode: str, n: int, flat: FlatModel, world: int, rank: int,
         depths=None) -> ShardPlan:
    if mode == "instance":
        return ShardPlan(mode, world, rank, row_shard(n, world, rank), (0, flat.num_trees))
    if mode in ("tree-reduce", "tree-pipeline", "tree-p2p"):
        d = flat.depths() if depths is None else depths
        return ShardPlan(mode, world, rank, (0, n), tree_shards(d, world)[rank])
    raise ValueError(f"unknown shard mode {mode!r}")


def gpu_scorer(flat: FlatModel, device: int, rank: bool = True):
    """Default per-rank scorer: the CUDA library on ``device``.

    Returns ``score(x, out, accumulate)`` over torch CUDA tensors.
    ``rank=False`` packs the fp32 layout (the fused tree-p2p pipeline).
    """
    from .evaluator import GpuModel
    model = GpuModel(flat, device, rank=rank)

    def score(x, out, accumulate=False):
        model.score(x, out=out, accumulate=accumulate)
        return out
    score.model = model
    return score


class ShardedScorer:
    """This rank's share of a sharded scoring job; packs its shard once.

    ``x_local``: this rank's instances -- its row shard for ``"instance"``,
    all ``n_total`` rows for the tree modes (``self.plan.rows`` either way;
    ``mode="auto"`` picks between them with :func:`choose_mode`).  ``__call__`` returns the rank's
    row-shard scores for ``"instance"``; for the tree modes the full f64
    ``[n_total]`` scores land on rank 0 (``"tree-reduce"``) or on the last
    rank (``"tree-pipeline"``, ``"tree-p2p"``), partial sums elsewhere.
    """

    def __init__(self, mode: str, flat: FlatModel, n_total: int, *, group=None,
                 make_scorer: Callable | None = None, device=None, depths=None,
                 chunk_rows: int = 1 << 17, serialize: bool = False,
                 l2_bytes: int | None = None, combine: str = "reduce"):
        import torch.distributed as dist
        if mode == "auto":
            # instance sharding unless the tables exceed L2 (choose_mode); the
            # caller passes x_local = rows[plan.rows[0]:plan.rows[1]]
            if l2_bytes is None:
                import torch
                dev = torch.cuda.current_device() if device is None else int(device)
                l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
            mode = choose_mode(flat, l2_bytes, depths, combine)
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n_total = n_total
        self.chunk_rows = chunk_rows
        self.serialize = serialize
        self.plan = plan(mode, n_total, flat, self.world, self.rank, depths)
        shard = flat if mode == "instance" else flat.subset(*self.plan.trees)
        # the fused pipeline (tree-p2p) runs on the fp32 complete-tree layout
        self.score = (make_scorer or (lambda fm: gpu_scorer(fm, device,
                                                            rank=mode != "tree-p2p")))(shard)
        # gloo moves CPU tensors only: CUDA payloads are staged through the host
        self._stage = dist.get_backend(group) == "gloo"
        # tree-reduce on GPUs over NCCL goes through the C ABI's own reduction
        # (ts_reduce_partials, with async-error polling); other backends and
        # the CPU test scorers use torch.distributed
        self.reducer = None
        if mode == "tree-reduce" and make_scorer is None and not self._stage:
            import torch
            dev = torch.cuda.current_device() if device is None else int(device)
            self.reducer = NcclReducer(dev, group)
        if mode == "tree-p2p":
            self._setup_p2p(device)

    def _send(self, t, dst):
        import torch.distributed as dist
        dist.send(t.cpu() if self._stage and t.is_cuda else t, dst=dst, group=self.group)

    def _recv(self, t, src):
        import torch.distributed as dist
        if self._stage and t.is_cuda:
            h = t.cpu()
            dist.recv(h, src=src, group=self.group)
            t.copy_(h)
        else:
            dist.recv(t, src=src, group=self.group)

    def _setup_p2p(self, device):
        """Allocate this rank's receive buffers, publish their IPC handles and
        map the next rank's (all_gather_object on the host; once)."""
        import torch
        import torch.distributed as dist
        from .evaluator import PeerBuffers, PipeBuffers
        model = getattr(self.score, "model", None)
        if model is None:
            raise ValueError("tree-p2p needs the CUDA scorer (gpu_scorer)")
        dev = torch.cuda.current_device() if device is None else int(device)
        self.recv = PipeBuffers(self.n_total, dev) if self.rank > 0 else None
        handles = [None] * self.world
        dist.all_gather_object(handles, self.recv.handles if self.recv else None,
                               group=self.group)
        self.send = PeerBuffers(handles[self.rank + 1]) if self.rank < self.world - 1 else None
        self.epoch = 0

    def __call__(self, x_local, out=None):
        import torch
        import torch.distributed as dist
        mode, rank, world, grp = self.plan.mode, self.rank, self.world, self.group
        dev = x_local.device
        if mode == "instance":
            if out is None:
                out = torch.empty(x_local.shape[0], dtype=torch.float64, device=dev)
            self.score(x_local, out, False)
            return out
        if out is None:
            out = torch.empty(self.n_total, dtype=torch.float64, device=dev)
        if mode == "tree-reduce":
            self.score(x_local, out, False)
            # scores land on the GROUP's rank 0
            if self.reducer is not None:
                self.reducer.reduce(out, out)          # in place on the root
                self.reducer.wait()
            elif self._stage and out.is_cuda:
                h = out.cpu()
                dist.reduce(h, dst=_global(grp, 0), op=dist.ReduceOp.SUM, group=grp)
                if rank == 0:
                    out.copy_(h)
            else:
                dist.reduce(out, dst=_global(grp, 0), op=dist.ReduceOp.SUM, group=grp)
            return out
        if mode == "tree-p2p":
            return self._call_p2p(x_local, out)
        # tree-pipeline: chunk c visits ranks 0..R-1 in order; rank r receives
        # the running sums of chunk c from r-1, continues them over its trees
        # and sends them on.
        for c0 in range(0, self.n_total, self.chunk_rows):
            c1 = min(self.n_total, c0 + self.chunk_rows)
            seg = out[c0:c1]
            if rank > 0:
                self._recv(seg, _global(grp, rank - 1))
            self.score(x_local[c0:c1], seg, rank > 0)
            if rank < world - 1:
                self._send(seg, _global(grp, rank + 1))
        return out


    def _call_p2p(self, x_local, out):
        import torch
        import torch.distributed as dist
        self.epoch += 1
        model = self.score.model
        kw = dict(epoch=self.epoch)
        if self.recv is not None:
            kw.update(sums_in=self.recv.sums, flags_in=self.recv.flags)
        if self.send is not None:
            kw.update(sums_out=self.send.sums, flags_out=self.send.flags)
        steps = range(self.world) if self.serialize else (self.rank,)
        for step in steps:
            if step == self.rank:
                model.score_pipe(x_local, out, **kw)
                torch.cuda.current_stream(x_local.device).synchronize()
            if self.serialize:
                dist.barrier(group=self.group)
        if not self.serialize:
            # the next call may overwrite the next rank's sums only after it
            # consumed this call's (flags are per epoch, buffers are not)
            torch.cuda.current_stream(x_local.device).synchronize()
            dist.barrier(group=self.group)
        return out

    def close(self):
        for b in (getattr(self, "recv", None), getattr(self, "send", None),
                  getattr(self, "reducer", None)):
            if b is not None:
                b.close()


class NcclReducer:
    """The C ABI's NCCL reduction of tree-shard partials (``ts_reduce_partials``,
    SURVEY 8(b)): a communicator of its own over the ranks of ``group``, the
    unique id broadcast from rank 0 on the host."""

    def __init__(self, device: int, group=None):
        import ctypes
        import torch.distributed as dist
        from . import _lib
        self._lib = lib = _lib.load()
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0 and lib.ts_nccl_get_unique_id(uid) != _lib.TS_OK:
            raise RuntimeError(f"ts_nccl_get_unique_id: {_lib.last_error()}")
        box = [uid.raw if self.rank == 0 else None]
        dist.broadcast_object_list(box, src=_global(group, 0), group=group)
        uid = ctypes.create_string_buffer(box[0], 128)
        comm = ctypes.c_void_p()
        if lib.ts_nccl_comm_init(uid, self.world, self.rank, int(device),
                                 ctypes.byref(comm)) != _lib.TS_OK:
            raise RuntimeError(f"ts_nccl_comm_init: {_lib.last_error()}")
        self.comm = comm

    def reduce(self, partial, out=None, root: int = 0):
        """``out`` (valid on ``root``) = sum over ranks of the f64 ``partial``."""
        import ctypes
        import torch
        from . import _lib
        if out is None:
            out = torch.empty_like(partial)
        rc = self._lib.ts_reduce_partials(self.comm, ctypes.c_void_p(partial.data_ptr()),
                                          ctypes.c_void_p(out.data_ptr()), partial.numel(),
                                          root, ctypes.c_void_p(
                                              torch.cuda.current_stream(partial.device).cuda_stream))
        if rc != _lib.TS_OK:
            raise RuntimeError(f"ts_reduce_partials: {_lib.last_error()}")
        return out

    def wait(self, timeout_ms: int = 60_000):
        """Block until the reduction on the current stream finished, polling
        NCCL's async error state (``ts_nccl_wait``): a dead peer or a timeout
        aborts the communicator and raises instead of hanging."""
        import ctypes
        import torch
        from . import _lib
        stream = torch.cuda.current_stream().cuda_stream
        rc = self._lib.ts_nccl_wait(self.comm, ctypes.c_void_p(stream), int(timeout_ms))
        if rc != _lib.TS_OK:
            raise RuntimeError(f"ts_nccl_wait: {_lib.last_error()}")

    def close(self):
        if getattr(self, "comm", None) is not None and self.comm.value:
            self._lib.ts_nccl_comm_destroy(self.comm)
            self.comm = None


def run_sharded(mode: str, flat: FlatModel, x_local, n_total: int, **kw):
    """One-shot :class:`ShardedScorer`; returns ``(plan, scores)``."""
    sc = ShardedScorer(mode, flat, n_total, **kw)
    return sc.plan, sc(x_local)


def gather_scores(local, n_total: int, group=None, dst: int = 0):
    """Collect instance-sharded scores on ``dst`` (not part of the hot path)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [row_shard(n_total, world, r) for r in range(world)]
    width = max(b - a for a, b in sizes)
    buf = torch.zeros(width, dtype=torch.float64, device=local.device)
    buf[:local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, parts, dst=_global(group, dst), group=group)
    if rank != dst:
        return None
    return torch.cat([parts[r][:b - a] for r, (a, b) in enumerate(sizes)])
