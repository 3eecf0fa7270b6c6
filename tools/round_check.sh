#!/bin/bash
# What the driver runs at round end, in one go on a GPU box (each step bounded
# by its own timeout so a hang cannot eat the whole call):
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/round_check.sh'
# Results land in gpurun_out/round_check/.
set -u
out=gpurun_out/round_check
mkdir -p "$out"
run() {  # name, timeout seconds, command...
    local name=$1 t=$2
    shift 2
    timeout "$t" "$@" > "$out/$name.log" 2>&1
    echo "$name: exit $?"
}
run pytest_gpu 900 python -m pytest tests -m gpu -x -q
run smoke 300 python -c "import __graft_entry__ as g; g.smoke()"
run bench 600 python bench.py
run bench_reference 600 python bench.py --impl reference
tail -n 1 "$out/bench.log" | cut -c 1-400
tail -n 1 "$out/bench_reference.log" | cut -c 1-300
tail -n 2 "$out/pytest_gpu.log"
