#!/bin/bash
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "gemm or c1 or prefill" 2>&1 | tail -2
bash scripts/gpu_fam.sh; bash scripts/gpu_fam.sh
export SGC_PROFILE=1
N="--set full --clock-control none --import-source on --kernel-name-base demangled"
B="python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-gen --waves 1"
timeout -s KILL 900 ncu $N -k regex:'gemm2_kernel<.int.3' -s 32 -c 1 -o gpurun_out/prof_tanh_hint $B > gpurun_out/ncu_tanh.out 2>&1; echo "tanh rc=$?"
