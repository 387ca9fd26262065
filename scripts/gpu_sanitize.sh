#!/bin/bash
# compute-sanitizer over the kernel tests: memcheck (all kernels incl. paged KV / forks / GNN /
# clustering / prompts) and racecheck + synccheck on the attention and GEMM kernels
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
run() { echo "== $*"; timeout -s KILL 1200 "$@" 2>&1 | grep -E "ERROR SUMMARY|passed|failed|Error|error" | tail -8; }
run $S --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_attention.py tests/test_gpu_paged_kv.py tests/test_gpu_fork.py -q -m gpu -x
run $S --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "not gemm_tcgen05"
run $S --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "gemm_tcgen05 and 1000"
run $S --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_attention.py -q -m gpu -x
run $S --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_attention.py -q -m gpu -x
run $S --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "gemm_tcgen05 and 1000"
