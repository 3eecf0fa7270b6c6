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

``--impl reference`` times the reference algorithm's CPU implementation on
the host cores (the C restatement in oracle/, all threads, VPred lockstep
batches) on a bounded row sample of the same workload; rank 0 only.
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


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    from paper_1212_2287_b200 import synth
    w = synth.config1(n=N_PER_GPU)
    import oracle
    c = oracle.COracle(w.flat.arrays())
    threads = len(os.sched_getaffinity(0))
    # size each step so the whole run stays within ~3 minutes
    per_step = max(0.5, min(3.0, 150.0 / max(1, args.steps + args.warmup)))
    probe = 2000
    t0 = time.perf_counter()
    c.score(w.x[:probe], threads=threads)
    rows = int(min(w.n, max(probe, probe * per_step / max(time.perf_counter() - t0, 1e-6))))
    for s in range(args.warmup):
        c.score(w.x[:rows], threads=threads)
    t0 = time.perf_counter()
    for s in range(args.steps):
        off = (s * rows) % max(1, w.n - rows)
        c.score(w.x[off:off + rows], threads=threads)
    dt = time.perf_counter() - t0
    value = rows * T * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 compare / f64 sum", "data": "synthetic",
        "config": {"workload": "cfg1: 1M x 136 mixed (ties), T=1000 complete d=8",
                   "instances": w.n, "features": F, "trees": T, "depth": D,
                   "sample_rows_per_step": rows},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{rows} rows x {T} trees per step (C restatement of the "
                                   "reference VPred path, oracle/ts_oracle.c, v=64)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    ws, rank, local = _dist()
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
        "config": {"workload": "cfg1: 1M x 136 mixed (ties), T=1000 complete d=8",
                   "instances_per_gpu": w.n, "features": F, "trees": T, "depth": D,
                   "parallelism": f"instance-sharded x{ws}",
                   "l2": "inputs (544 MB/GPU) larger than L2; no flush",
                   "kernel": f"{launches / max(1, args.steps):g} launch(es)/step: k_stream over the "
                             "full waves of 128-row tiles + k_stream_ws on the last partial wave's rows; "
                             "roofline.achieved is per step (both kernels)"},
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": w.n * F * 4, "d2h_bytes_per_step": w.n * 8,
                "api": "GpuEvaluator._predict_into (ts_score_host), pinned host buffers",
                "steps": e2e_steps, "matches_device_scores": e2e_equal},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if ws == 1 and not args.no_cpu_baseline:
        cpu_val, rows, cpu_scores, threads, dt, passes = cpu_sample(w, args.cpu_seconds)
        line["cpu_baseline"] = {
            "value": cpu_val, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{passes} pass(es) over the first {rows} rows x {T} trees ({dt:.1f} s; "
                      "C restatement of the reference VPred path, oracle/ts_oracle.c, "
                      "lockstep batches of 64)"}
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
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
