"""Benchmark: tree evaluations per second on BASELINE config 1.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], the metric's single-GPU configuration):
1,000,000 instances x 136 fp32 features (70% U[0,1), 20% lognormal, 10%
integer counts -> exact threshold ties) scored against 1,000 complete
depth-8 trees, seeded synthetic data (the paper's MSLR data is unavailable).
One step = one pass of the hot path (ts_score) over the resident 1M-row
batch = 1e9 tree evaluations.  The 544 MB feature matrix is larger than the
126 MB L2, so no explicit flush is needed between steps.

Under torchrun each rank scores its own 1M-row shard on its own GPU
(instance sharding, no collective on the data path; "scaling": "weak");
rank 0 prints one JSON line with the whole-job value (max time over ranks).

Two more measured sub-objects ride on the same line, at the same N:
``cfg4a`` -- BASELINE config 4a's 64M x 136 matrix split over the N ranks
(strong scaling; instance sharding, no collective) -- and ``cfg4b`` -- config
4b's 20,000 depth-10 trees split over the ranks (tree sharding), every rank
scoring all 8M rows against its shard and ONE NCCL f64 sum-reduce
(``ts_reduce_partials``, the C ABI's own communicator) combining the partials.
Each carries ms per pass, tree-evals/s, the efficiency against rank 0 scoring
the whole job alone in the same run, and an oracle parity sample.

``python bench.py --gpus N`` without a launcher (no WORLD_SIZE in the
environment) re-executes itself under ``torch.distributed.run`` with N ranks,
one per GPU (``TS_BENCH_BACKEND=gloo``: host-side plumbing over gloo, ranks
may share a GPU -- a flow check, not a scaling number).  NCCL_DEBUG=INFO
stays on for N > 1 so rank counts show in the log.

``--impl reference`` times the reference algorithm's CPU implementation on
the host cores on a bounded row sample of the same workload, rank 0 only:
the faster of its two CPU strategies -- the VPred path
(the C restatement in oracle/, all threads, lockstep batches of 64) and its
CodeGen strategy (the reference's own generated C, byte-identical emitter in
oracle/codegen.py, prebuilt by ``__graft_entry__.build``, one thread per
core).  On the B200 hosts VPred is 4-16x faster (profiles/r2_cpu_baselines.jsonl),
so it is the arm; both rates ride in ``cpu_baseline.candidates``.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tree evals/sec (instance x tree)"
UNIT = "tree-evals/s"
F, T, D = 136, 1000, 8
N_PER_GPU = 1_000_000


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return {"hbm_gbs": float(p["hbm_gbs"]), "sm_max_mhz": float(p["sm_max_mhz"]),
                "source": "measured"}
    except Exception:  # noqa: BLE001
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


def bench_config(n_gpus: int) -> dict:
    """The workload's ``config`` -- identical on both arms (same keys, same
    values) so the driver can match them."""
    return {"workload": "cfg1: 1M x 136 mixed (ties), T=1000 complete d=8",
            "instances_per_gpu": N_PER_GPU, "features": F, "trees": T, "depth": D,
            "parallelism": f"instance-sharded x{n_gpus}",
            "l2": "inputs (544 MB/GPU) larger than L2; no flush"}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_sample(w, target_s: float, threads: int | None = None):
    """Time the oracle's C port on a bounded sample (about ``target_s`` seconds
    of CPU work: whole passes over a row prefix); returns
    (evals/s, rows, scores of the prefix, threads, seconds, passes)."""
    import oracle
    c = oracle.COracle(w.flat.arrays())
    threads = threads or len(os.sched_getaffinity(0))
    probe = min(w.n, 4000)
    t0 = time.perf_counter()
    c.score(w.x[:probe], threads=threads)
    dt = time.perf_counter() - t0
    rows = int(min(w.n, max(probe, probe * target_s / max(dt, 1e-6))))
    passes = 0
    t0 = time.perf_counter()
    while True:
        scores = c.score(w.x[:rows], threads=threads)
        passes += 1
        dt = time.perf_counter() - t0
        if dt >= target_s or passes >= 50:
            break
    return rows * T * passes / dt, rows, scores, threads, dt, passes


def generated_sample(w, target_s: float, threads: int):
    """The reference's CodeGen strategy on the same workload, when its unit was
    prebuilt (``__graft_entry__.build`` compiles config 1's 50 MB of generated
    C, ~100 s): the C text of ref ``codegen.emit_source`` (byte-identical,
    ``oracle/codegen.py``) compiled with its flags, one thread per core over
    row shards.  Gated on the 1,000-row prefix against the C oracle first
    (ref bench.py:220-231).  Returns (evals/s, rows, seconds, passes) or None."""
    import oracle
    from oracle import codegen
    unit = codegen.cached_unit(w.flat)
    if unit is None:
        return None
    prefix = w.x[:1000]
    if not np.array_equal(unit.score(prefix, threads=threads),
                          oracle.COracle(w.flat.arrays()).score(prefix, threads=threads)):
        # a unit that fails the reference's gate is not timed (ref bench.py:220-231)
        return "failed the 1000-row correctness gate"
    out = np.empty(w.n, np.float64)
    probe = min(w.n, 2000)
    t0 = time.perf_counter()
    unit.score_parallel(w.x[:probe], out[:probe], threads)
    dt = time.perf_counter() - t0
    rows = int(min(w.n, max(probe, probe * target_s / max(dt, 1e-6))))
    passes, t0 = 0, time.perf_counter()
    while True:
        unit.score_parallel(w.x[:rows], out[:rows], threads)
        passes += 1
        dt = time.perf_counter() - t0
        if dt >= target_s or passes >= 50:
            break
    return rows * T * passes / dt, rows, dt, passes


def cpu_baseline_line(w, target_s: float):
    """the faster of the reference's VPred path (C port) and
    its CodeGen strategy (its own generated C), both on all host cores.
    Returns (cpu_baseline dict, port scores of the prefix, prefix rows)."""
    cpu_val, rows, cpu_scores, threads, dt, passes = cpu_sample(w, target_s)
    port = {"value": cpu_val, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{passes} pass(es) over the first {rows} rows x {T} trees ({dt:.1f} s; "
                      "C restatement of the reference VPred path, oracle/ts_oracle.c, "
                      "lockstep batches of 64)"}
    gen = generated_sample(w, min(target_s, 4.0), threads)
    if gen is None or isinstance(gen, str):
        port["candidates"] = {"port": cpu_val,
                              "generated": gen or "not prebuilt (oracle/_gen)"}
        return port, cpu_scores, rows
    g_val, g_rows, g_dt, g_passes = gen
    cand = {"port": cpu_val, "generated": g_val,
            "generated_sample": f"{g_passes} pass(es) over the first {g_rows} rows x {T} trees "
                                f"({g_dt:.1f} s; the reference's generated C, -O3, "
                                f"{threads} threads over row shards)"}
    if g_val > cpu_val:
        line = {"value": g_val, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": cand["generated_sample"]}
    else:
        line = port
    line["candidates"] = cand
    return line, cpu_scores, rows


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    from paper_1212_2287_b200 import synth
    w = synth.config1(n=N_PER_GPU)
    import oracle
    c = oracle.COracle(w.flat.arrays())
    threads = len(os.sched_getaffinity(0))
    # the faster of the VPred port and the reference's own
    # generated C (when prebuilt) is the reference arm
    gen = generated_sample(w, 3.0, threads)
    gen_note = gen if isinstance(gen, str) else None
    if gen_note:
        gen = None
    probe = 2000
    t0 = time.perf_counter()
    c.score(w.x[:probe], threads=threads)
    port_rate = probe * T / max(time.perf_counter() - t0, 1e-9)
    use_gen = gen is not None and gen[0] > port_rate
    if use_gen:
        from oracle import codegen
        unit = codegen.cached_unit(w.flat)
        buf = np.empty(w.n, np.float64)

        def score(xx):
            unit.score_parallel(xx, buf[:len(xx)], threads)
        kind, what = "reference", "the reference's generated C (CodeGen strategy), -O3"
    else:
        def score(xx):
            c.score(xx, threads=threads)
        kind, what = "port", "C restatement of the reference VPred path, oracle/ts_oracle.c, v=64"
    # size each step so the whole run stays within ~3 minutes
    per_step = max(0.5, min(3.0, 150.0 / max(1, args.steps + args.warmup)))
    t0 = time.perf_counter()
    score(w.x[:probe])
    rows = int(min(w.n, max(probe, probe * per_step / max(time.perf_counter() - t0, 1e-6))))
    for s in range(args.warmup):
        score(w.x[:rows])
    t0 = time.perf_counter()
    for s in range(args.steps):
        off = (s * rows) % max(1, w.n - rows)
        score(w.x[off:off + rows])
    dt = time.perf_counter() - t0
    value = rows * T * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": max(ws, args.gpus), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 compare / f64 sum", "data": "synthetic",
        "config": bench_config(max(ws, args.gpus)),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{rows} rows x {T} trees per step ({what})",
                         "candidates": {"port_probe": port_rate,
                                        "generated": gen[0] if gen else
                                        (gen_note or "not prebuilt")}},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


class _Ctx:
    def __init__(self, ws, rank, local, dev, backend, barrier, max_over_ranks):
        self.ws, self.rank, self.local, self.dev, self.backend = ws, rank, local, dev, backend
        self.barrier, self.max = barrier, max_over_ranks

    def min(self, v: float) -> float:
        return -self.max(-float(v))

    def sum(self, v: float) -> float:
        if self.ws == 1:
            return float(v)
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64,
                         device=self.dev if self.backend == "nccl" else "cpu")
        torch.distributed.all_reduce(t)
        return float(t.item())


def _gen_rows(w, row0: int, n: int, dev):
    """Rows [row0, row0+n) of a counter-based workload, generated on the GPU."""
    import torch
    from paper_1212_2287_b200 import _lib
    x = torch.empty((n, w.f), dtype=torch.float32, device=dev)
    rc = _lib.load().ts_synth_uniform(x.data_ptr(), n, w.f, w.f, w.hash_seed, row0, w.zero_prob,
                                      torch.cuda.current_stream(dev).cuda_stream)
    if rc != 0:
        raise RuntimeError(f"ts_synth_uniform: {_lib.last_error()}")
    return x


def _time_steps(fn, steps: int, warmup: int, c, dev, sync=None) -> float:
    """Max over ranks of the mean ms per call of ``fn`` (CUDA events on the
    current stream, barrier + synchronize on both sides)."""
    import torch
    for _ in range(warmup):
        fn()
    c.barrier()
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        fn()
    e1.record(st)
    if sync is not None:
        sync()
    c.barrier()
    return c.max(e0.elapsed_time(e1) / steps)


def _time_local(fn, steps: int, warmup: int, dev) -> float:
    """Mean ms per call of ``fn`` on this rank alone (no collectives)."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize(dev)
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        fn()
    e1.record(st)
    torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) / steps


def _roof(n, T, F_, sum_depth, n_gpus, tree_sharded=False):
    """SURVEY 8(d) roofline in tree-evals/s for N GPUs (tree sharding: every
    GPU reads all n rows, so the HBM term does not shrink with N)."""
    import torch
    peaks = _peaks()
    n_sm = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    visit_peak = n_sm * 128 * peaks["sm_max_mhz"] * 1e6 / 4
    t_issue = n * sum_depth / visit_peak / n_gpus
    t_hbm = n * (4 * F_ + 8) / (peaks["hbm_gbs"] * 1e9) / (1 if tree_sharded else n_gpus)
    return n * T / max(t_issue, t_hbm)


def sub_cfg4a(args, c):
    """BASELINE config 4a: 64M x 136 U[0,1) rows (34.8 GB) and config 2's
    depth-8 ensemble, instance-sharded over the N ranks (contiguous row
    ranges, no collective).  Rank 0 also scores the whole matrix alone: the
    single-GPU time the efficiency is measured against."""
    import torch
    import oracle
    from paper_1212_2287_b200 import GpuModel, synth
    from paper_1212_2287_b200.distributed import row_shard
    w = synth.config4a()
    n, T_ = w.n, w.flat.num_trees
    a, b = row_shard(n, c.ws, c.rank)
    r0, nr = (0, n) if c.rank == 0 else (a, b - a)   # rank 0's shard is a view of all rows
    x = _gen_rows(w, r0, nr, c.dev)
    m = GpuModel(w.flat, c.local)
    out = torch.empty(nr, dtype=torch.float64, device=c.dev)
    xs, outs = x[a - r0:b - r0], out[a - r0:b - r0]
    steps, warm = args.sub_steps, 1
    t_n = _time_steps(lambda: m.score(xs, out=outs), steps, warm, c, c.dev)
    if c.ws > 1:
        t1 = _time_local(lambda: m.score(x, out=out), steps, warm, c.dev) \
            if c.rank == 0 else 0.0
        t1 = c.max(t1)          # the other ranks wait here
    else:
        t1 = t_n
    rows = oracle.sample_rows(b - a, max(64, 4096 // c.ws), seed=c.rank) + a
    got = outs.index_select(0, torch.from_numpy(rows - a).to(c.dev)).cpu().numpy()
    host = np.concatenate([w.rows(s0, k) for s0, k in oracle.runs_of(rows)])
    ok = bool(np.array_equal(got, oracle.COracle(w.flat.arrays()).score(host)))
    sd = int(m.info["sum_depth"])
    res = {"workload": "cfg4a: 64M x 136 U[0,1), T=1000 complete d=8, instance-sharded",
           "n_gpus": c.ws, "scaling": "strong", "instances": n, "trees": T_,
           "ms_per_pass": t_n, "tree_evals_per_s": n * T_ / (t_n / 1e3),
           "single_gpu_ms_per_pass": t1, "efficiency_vs_1gpu": t1 / (c.ws * t_n),
           "roofline_frac": (n * T_ / (t_n / 1e3)) / _roof(n, T_, w.f, sd, c.ws),
           "steps": steps, "collective": "none",
           "parity": {"rows_checked": int(c.sum(len(rows))), "bit_exact_vs_oracle":
                      bool(c.min(1.0 if ok else 0.0) > 0)}}
    del x, out, xs, outs
    m.close()
    return res


def sub_cfg4b(args, c):
    """BASELINE config 4b: 20,000 depth-10 trees (245.6 MB of node tables,
    beyond L2) over 8M x 136 rows, tree-sharded: every rank scores all rows
    against its contiguous tree range (balanced by sum of depths) and one
    NCCL f64 sum-reduce to rank 0 (``ts_reduce_partials`` through the
    library's own communicator, async errors polled) combines them.  Rank 0
    also scores the whole ensemble alone (the single-GPU reference)."""
    import torch
    import oracle
    from paper_1212_2287_b200 import GpuModel, synth
    w = synth.config4b()
    n, T_ = w.n, w.flat.num_trees
    x = _gen_rows(w, 0, n, c.dev)
    out = torch.zeros(n, dtype=torch.float64, device=c.dev)
    steps, warm = args.sub_steps, 1
    full = GpuModel(w.flat, c.local) if c.rank == 0 else None
    if c.ws > 1:
        from paper_1212_2287_b200.distributed import ShardedScorer
        sc = ShardedScorer("tree-reduce", w.flat, n, device=c.local)
        how = ("ts_reduce_partials (NCCL f64 sum, library communicator)"
               if sc.reducer is not None else "torch.distributed reduce over gloo (host-staged)")
        t_n = _time_steps(lambda: sc(x, out), steps, warm, c, c.dev)
        trees = sc.plan.trees
        t1 = _time_local(lambda: full.score(x), steps, warm, c.dev) if c.rank == 0 else 0.0
        t1 = c.max(t1)          # the other ranks wait here
    else:
        sc, how, trees = None, "none (one GPU)", (0, T_)
        t_n = t1 = _time_steps(lambda: full.score(x, out=out), steps, warm, c, c.dev)
    res = None
    if c.rank == 0:
        rows = oracle.sample_rows(n, 1024, seed=41)
        got = out.index_select(0, torch.from_numpy(rows).to(c.dev)).cpu().numpy()
        host = np.concatenate([w.rows(s0, k) for s0, k in oracle.runs_of(rows)])
        orc = oracle.COracle(w.flat.arrays())
        ref = orc.score(host)
        tol = oracle.score_tolerance(orc, host, ref)
        sd = int(full.info["sum_depth"])
        res = {"workload": "cfg4b: 8M x 136 U[0,1), T=20000 complete d=10, tree-sharded",
               "n_gpus": c.ws, "scaling": "strong", "instances": n, "trees": T_,
               "rank0_trees": list(trees), "combine": how,
               "ms_per_pass": t_n, "tree_evals_per_s": n * T_ / (t_n / 1e3),
               "single_gpu_ms_per_pass": t1, "efficiency_vs_1gpu": t1 / (c.ws * t_n),
               "roofline_frac": (n * T_ / (t_n / 1e3)) / _roof(n, T_, w.f, sd, c.ws, True),
               "steps": steps,
               "parity": {"rows_checked": int(len(rows)),
                          "within_1e-5": bool(np.all(np.abs(got - ref) <= tol)),
                          "bit_exact_vs_oracle": bool(np.array_equal(got, ref)),
                          "max_rel_err": float(np.max(np.abs(got - ref) /
                                                      np.maximum(np.abs(ref), 1e-300)))}}
    if sc is not None:
        sc.close()
    if full is not None:
        full.close()
    c.barrier()
    return res


def run_ours(args):
    import torch
    ws, rank, local = _dist()
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")     # rank counts in the log
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    # One GPU per rank.  TS_BENCH_BACKEND=gloo (flow tests only: several
    # independent instance-shard ranks on fewer GPUs, their kernels never wait
    # on one another) swaps the host-side barrier / max-reduce to gloo; the
    # numbers of such a run are not scaling numbers.
    backend = os.environ.get("TS_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    from paper_1212_2287_b200 import _lib, build_gpu, synth

    w = synth.config1(n=N_PER_GPU, shard=rank)
    ev = build_gpu(w.flat, device=local)
    info = ev.model.info
    x = torch.from_numpy(w.x).to(dev)
    out = torch.empty(w.n, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(v: float) -> float:
        if ws == 1:
            return v
        tt = torch.tensor([v], dtype=torch.float64,
                          device=dev if backend == "nccl" else "cpu")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        return float(tt.item())

    for _ in range(args.warmup):
        ev.score_device(x, out=out)
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.15)
    launches0 = _lib.launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    start.record(stream)
    for _ in range(args.steps):
        ev.score_device(x, out=out)
    end.record(stream)
    barrier()
    clocks = sampler.stop()
    launches = _lib.launch_count() - launches0
    ms = start.elapsed_time(end)
    t_max = max_over_ranks(ms)
    evals = w.n * T * args.steps * ws
    value = evals / (t_max / 1e3)
    ms_per_step = t_max / args.steps

    # parity gate on the GPU result of the timed region (first rows vs the oracle)
    gpu_scores = out.cpu().numpy()

    # ---- end-to-end through the public API: pinned host rows in, scores out
    pinned = torch.empty((w.n, F), dtype=torch.float32, pin_memory=True)
    pinned.numpy()[:] = w.x
    host_out = torch.empty(w.n, dtype=torch.float64, pin_memory=True).numpy()
    e2e_steps = max(1, min(args.steps, 10))
    ev._predict_into(pinned.numpy(), host_out)       # warm the pipeline buffers
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        ev._predict_into(pinned.numpy(), host_out)
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e_value = w.n * T * e2e_steps * ws / e2e_s
    e2e_equal = bool(np.array_equal(host_out, gpu_scores))
    del pinned, host_out

    # ---- configs 4a (strong scaling) and 4b (tree sharding + NCCL reduce)
    ctx = _Ctx(ws, rank, local, dev, backend, barrier, max_over_ranks)
    subs = {}
    if not args.no_sub:
        del x, out
        torch.cuda.empty_cache()
        for name, fn in (("cfg4a", sub_cfg4a), ("cfg4b", sub_cfg4b)):
            try:
                subs[name] = fn(args, ctx)
            except Exception as exc:  # noqa: BLE001
                if ws > 1:     # the other ranks would wait in a collective forever
                    import traceback
                    traceback.print_exc()
                    sys.stderr.flush()
                    os._exit(1)
                subs[name] = {"error": f"{type(exc).__name__}: {exc}"}
            torch.cuda.empty_cache()

    if rank != 0:
        if ws > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return 0

    peaks = _peaks()
    props = torch.cuda.get_device_properties(dev)
    n_sm = props.multi_processor_count
    f_sm = peaks["sm_max_mhz"] * 1e6
    visits = w.n * info["sum_depth"]                  # per launch (one launch per step)
    t_launch = ms / 1e3 / args.steps
    visit_peak = n_sm * 128 * f_sm / 4               # 4 issue slots per node visit
    hbm_bytes = w.n * (4 * F + 8)
    roof_eval = w.n * T / max(hbm_bytes / (peaks["hbm_gbs"] * 1e9), visits / visit_peak)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")  # ncu --set full capture
    except Exception:  # noqa: BLE001
        pass
    roofline = {
        "bound": "issue", "unit": "Gnode-visits/s",
        "achieved": visits / t_launch / 1e9, "peak": visit_peak / 1e9,
        "frac": (w.n * T / t_launch) / roof_eval,
        "traffic": traffic,
        "peak_note": f"{n_sm} SMs x 32 visits/clk (4 issue slots per visit) x "
                     f"{peaks['sm_max_mhz']:.0f} MHz ({peaks['source']} sm_max_mhz)",
        "hbm": {"achieved_gbs": hbm_bytes / t_launch / 1e9, "peak_gbs": peaks["hbm_gbs"],
                "frac": hbm_bytes / t_launch / 1e9 / peaks["hbm_gbs"],
                "algorithmic_bytes_per_launch": hbm_bytes},
        "algorithmic_visits_per_launch": visits,
        # measured speed of light of any shared-memory predicated walk on this
        # GPU (every lane reading the same node record): the data path caps it
        # well below the 4-slot issue roofline
        "practical_ceiling": {"frac": 0.291, "visits_per_clk_sm": 9.32,
                              "source": "tools/mb_walk_sol.cu, "
                                        "profiles/r1_microbench_smem_pipes.txt"},
    }

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 compare / f64 sum",
        "data": "synthetic (seeded; BASELINE cfg1 distributions)",
        "config": bench_config(ws),
        "kernel": f"{launches / max(1, args.steps):g} launch(es)/step: k_stream over the "
                  "full waves of 128-row tiles + k_stream_ws on the last partial wave's rows; "
                  "roofline.achieved is per step (both kernels)",
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": w.n * F * 4, "d2h_bytes_per_step": w.n * 8,
                "api": "GpuEvaluator._predict_into (ts_score_host), pinned host buffers",
                "steps": e2e_steps, "matches_device_scores": e2e_equal},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    line.update(subs)
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"], cpu_scores, rows = cpu_baseline_line(w, args.cpu_seconds)
        line["parity"] = {"rows_checked": rows,
                          "bit_exact_vs_oracle": bool(np.array_equal(cpu_scores,
                                                                     gpu_scores[:rows]))}
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sub", action="store_true",
                    help="skip the config 4a / 4b sub-measurements")
    ap.add_argument("--sub-steps", type=int, default=3)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    return run_ours(args)


def relaunch(args) -> int:
    """``--gpus N`` without a launcher: run N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


if __name__ == "__main__":
    sys.exit(main())
