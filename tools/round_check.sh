#!/bin/bash
# What the driver runs at round end, in one go on a GPU box (each step bounded
# by its own timeout so a hang cannot eat the whole call), plus the ncu
# evidence for profiles/ (launch list of the bench command, one full capture
# of the dominant kernel), each only after its own command ran clean:
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/round_check.sh'
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
if [ "${NCU:-1}" = 1 ]; then
    run ncu_launches 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file "$out/ncu_launches.csv" python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sub
    run ncu_full 900 ncu --set full --import-source on --clock-control none -k regex:"k_stream" \
        --launch-skip 2 --launch-count 1 -o "$out/bench_k_stream" python bench.py --steps 3 --no-sub \
        --warmup 3 --no-cpu-baseline
fi
tail -n 1 "$out/bench.log" | cut -c 1-400
tail -n 1 "$out/bench_reference.log" | cut -c 1-300
tail -n 2 "$out/pytest_gpu.log"
if [ "${CONFIGS:-0}" = 1 ]; then
    run configs 900 python tools/bench_configs.py --out "$out/configs.jsonl"
fi
