#!/bin/bash
# Memory-safety pass for the kernels (compute-sanitizer is closed on this pool):
# build a bounds-checked library (-DTS_DEBUG: every shared load of the walks is
# range-checked and traps) and run the GPU parity suite and all configs on it.
# Usage on the GPU box: bash tools/debug_check.sh   (build it here first with
#   TS_NVCC_EXTRA=-DTS_DEBUG TS_GPU_SO=$PWD/paper_1212_2287_b200/_ts_gpu_debug.so \
#   python paper_1212_2287_b200/_build.py --force)
set -e
export TS_GPU_SO=$PWD/paper_1212_2287_b200/_ts_gpu_debug.so
python -m pytest tests -m gpu -x -q
python tools/bench_configs.py --configs 0,1,2:3,2:10,2:12,3 --reps 1
