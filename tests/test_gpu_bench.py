"""The driver contract of ``bench.py`` at N > 1 without a launcher.

``python bench.py --gpus 2`` (no WORLD_SIZE) must start two ranks itself and
print ONE JSON line with ``n_gpus: 2`` and the measured config 4a (strong
scaling) and config 4b (tree-sharded, reduced) sub-objects.  One GPU here:
TS_BENCH_BACKEND=gloo lets both ranks share it (a flow check; its numbers are
not scaling numbers)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, has_cuda

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]


def _json_line(stdout: str) -> dict:
    lines = [ln for ln in stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, stdout[-4000:]
    return json.loads(lines[0])


def test_bench_two_ranks_self_launched():
    env = dict(os.environ, TS_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--steps", "2", "--warmup", "3", "--sub-steps", "1"],
                         capture_output=True, text=True, env=env, timeout=1500, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-4000:]
    line = _json_line(res.stdout)
    assert line["n_gpus"] == 2
    assert line["config"]["parallelism"] == "instance-sharded x2"
    assert line["value"] > 0 and line["e2e"]["matches_device_scores"]
    a, b = line["cfg4a"], line["cfg4b"]
    assert a["n_gpus"] == 2 and a["instances"] == 64_000_000
    assert a["parity"]["bit_exact_vs_oracle"] and a["parity"]["rows_checked"] >= 4096
    assert 0 < a["efficiency_vs_1gpu"] and a["tree_evals_per_s"] > 0
    assert b["n_gpus"] == 2 and b["trees"] == 20_000 and b["rank0_trees"][0] == 0
    assert 0 < b["rank0_trees"][1] < 20_000
    assert b["parity"]["within_1e-5"] and b["parity"]["max_rel_err"] < 1e-9


def test_bench_one_gpu_line_and_reference_config():
    """N=1 line carries the sub-objects; the reference arm's config is the
    same dict as ours (the driver matches them)."""
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3",
                          "--warmup", "3", "--sub-steps", "1", "--cpu-seconds", "2"],
                         capture_output=True, text=True, timeout=1500, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-4000:]
    ours = _json_line(res.stdout)
    assert ours["n_gpus"] == 1 and ours["parity"]["bit_exact_vs_oracle"]
    # both CPU strategies timed, the faster one reported
    cand = ours["cpu_baseline"]["candidates"]
    assert cand["port"] > 0 and "generated" in cand
    assert ours["cfg4a"]["parity"]["bit_exact_vs_oracle"]
    assert ours["cfg4b"]["parity"]["bit_exact_vs_oracle"]
    ref = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert ref.returncode == 0, ref.stderr[-4000:]
    theirs = _json_line(ref.stdout)
    assert theirs["impl"] == "reference" and theirs["config"] == ours["config"]
    assert (theirs["metric"], theirs["unit"]) == (ours["metric"], ours["unit"])
