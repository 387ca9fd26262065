#!/bin/bash
# ncu --set full of one extend layer's residual GEMMs (Wo then W2) at C3
mkdir -p gpurun_out
export SGC_PROFILE=1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'gemm2_kernel<.int.2' -s 64 -c 2 -o gpurun_out/prof_resid2 python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-gen --waves 1 > gpurun_out/ncu_resid2.out 2>&1; echo "resid rc=$?"; grep -E "PROF|WARN|ERR" gpurun_out/ncu_resid2.out | head -5
