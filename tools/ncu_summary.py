"""Summarise an ncu report: key throughput metrics and per-LDS wavefronts.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--lds]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "smsp__warps_issue_stalled_mio_throttle_per_warp_active.pct",
        "smsp__warps_issue_stalled_short_scoreboard_per_warp_active.pct",
        "smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warps_issue_stalled_barrier_per_warp_active.pct",
        "launch__registers_per_thread", "sm__cycles_active.avg"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]], rows[1]


def main():
    rep = sys.argv[1]
    recs, units = raw(rep)
    for rec in recs:
        print(rec.get("Kernel Name", "")[:90])
        for k in KEYS:
            if k in rec:
                print(f"  {k:70s} {rec[k]}")
    if "--lds" in sys.argv:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                              "sass"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        h = rows[1]
        src, wf, ex = h.index("Source"), h.index("L1 Wavefronts Shared"), \
            h.index("Instructions Executed")
        for r in rows[2:]:
            if "LDS" in r[src] or "STS" in r[src]:
                w, e = int(r[wf] or 0), int(r[ex] or 0)
                if e:
                    print(f"{w:>11d} {e:>10d} {w / e:6.2f}  {r[src].strip()}")


if __name__ == "__main__":
    main()
