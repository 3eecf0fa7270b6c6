"""Multi-GPU scale-out (BASELINE config 4), one process per GPU:

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/bench_multi.py \
        --mode instance|tree-reduce|tree-pipeline|tree-p2p [--rows R] [--reps K]

instance: config 4a (64M x 136, T=1000 d=8), each rank generates and scores
its contiguous row shard in place on its GPU (no collective on the data path).
tree-*: config 4b (8M x 136, T=20,000 d=10), each rank holds a balanced tree
shard and scores all rows; partials combined by an NCCL f64 sum-reduce
("tree-reduce"), by the bit-exact rank-to-rank pipeline over NCCL
send/recv ("tree-pipeline"), or by the same bit-exact pipeline fused into
the scoring kernel over NVLink peer memory ("tree-p2p", ts_score_pipe).
Timing: barrier + synchronize around K passes, CUDA events, max over ranks.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1212_2287_b200 import _lib, synth  # noqa: E402
from paper_1212_2287_b200 import distributed as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="instance", choices=["instance", "tree-reduce", "tree-pipeline",
                                                             "tree-p2p"])
    ap.add_argument("--rows", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--check", type=int, default=512,
                    help="rows checked against the C oracle on the rank holding the result")
    a = ap.parse_args()
    # TS_BENCH_BACKEND=gloo: flow test of the instance / tree-reduce modes with
    # several ranks on fewer GPUs (ranks never wait on one another inside a
    # kernel); not a scaling measurement.
    backend = os.environ.get("TS_BENCH_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = torch.device("cuda", local)
    w = synth.config4a(a.rows or 64_000_000) if a.mode == "instance" \
        else synth.config4b(a.rows or 8_000_000)
    if a.mode == "instance":
        r0, r1 = D.row_shard(w.n, world, rank)
    else:
        r0, r1 = 0, w.n
    x = torch.empty((r1 - r0, w.f), dtype=torch.float32, device=dev)
    _lib.load().ts_synth_uniform(x.data_ptr(), r1 - r0, w.f, w.f, w.hash_seed, r0, w.zero_prob,
                                 torch.cuda.current_stream().cuda_stream)
    depths = None if a.mode == "instance" else [10] * w.flat.num_trees
    scorer = D.ShardedScorer(a.mode, w.flat, w.n, device=local, depths=depths)  # packs once
    out = scorer(x)                                                               # warm-up
    dist.barrier()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.reps):
        scorer(x, out)
    e.record()
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([s.elapsed_time(e) / a.reps], dtype=torch.float64,
                     device=dev if backend == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # parity on the rank that holds full scores: every rank (instance), rank 0
    # (tree-reduce), the last rank (tree-pipeline, tree-p2p)
    holder = {"instance": rank, "tree-reduce": 0}.get(a.mode, world - 1)
    exact = None
    if a.check and rank == holder:
        import numpy as np
        import oracle
        k = min(a.check, r1 - r0)
        rows = np.linspace(0, r1 - r0 - 1, k).astype(np.int64)
        xs = np.concatenate([w.rows(r0 + int(i), 1) for i in rows])
        ref = oracle.COracle(w.flat.arrays()).score(np.ascontiguousarray(xs), threads=8)
        got = out.cpu().numpy()[rows]
        exact = bool(np.array_equal(got, ref)) if a.mode != "tree-reduce" else \
            bool(np.allclose(got, ref, rtol=1e-12, atol=1e-12))
    flags = [None] * world
    dist.all_gather_object(flags, exact)
    if rank == 0:
        evals = w.n * w.flat.num_trees
        print(json.dumps({"mode": a.mode, "world": world, "workload": w.name,
                          "ms_per_pass": float(t.item()),
                          "tree_evals_per_s": evals / (float(t.item()) / 1e3),
                          "parity": [f for f in flags if f is not None]}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
