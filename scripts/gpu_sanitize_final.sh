#!/bin/bash
# compute-sanitizer memcheck / synccheck over the paths changed late in round 2: decode (own-key
# attention layout, fused row scales, stream-K / split-K GEMMs), the parity suite (stream-K shapes,
# agglomerate global-state path) and the fullwidth suite
S=/usr/local/cuda/bin/compute-sanitizer
run() { echo "== $*"; timeout -s KILL 1500 "$@" 2>&1 | grep -E "ERROR SUMMARY|passed|failed|Error|error" | tail -6; }
run $S --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_decode.py tests/test_gpu_fork.py tests/test_gpu_paged_kv.py -q -m gpu -x
run $S --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "not gemm_tcgen05"
run $S --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_decode.py -q -m gpu -x
