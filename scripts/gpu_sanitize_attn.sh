#!/bin/bash
# racecheck + synccheck over the tcgen05 attention kernels of the final build
S=/usr/local/cuda/bin/compute-sanitizer
run() { echo "== $*"; timeout -s KILL 1700 "$@" 2>&1 | grep -E "SUMMARY|passed|failed" | tail -4; }
run $S --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_attention.py -q -m gpu -x
run $S --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_attention.py -q -m gpu -x
