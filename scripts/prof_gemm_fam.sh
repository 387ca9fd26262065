#!/bin/bash
mkdir -p gpurun_out
export SGC_PROFILE=1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'gemm2_kernel<.int.4' -s 32 -c 1 -o gpurun_out/prof_qkv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-gen --waves 1 > gpurun_out/ncu_qkv.out 2>&1; echo "qkv rc=$?"; grep -E "PROF|WARN|ERR" gpurun_out/ncu_qkv.out | head -5
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'gemm2_kernel<.int.2' -s 64 -c 1 -o gpurun_out/prof_resid python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-gen --waves 1 > gpurun_out/ncu_resid.out 2>&1; echo "resid rc=$?"; grep -E "PROF|WARN|ERR" gpurun_out/ncu_resid.out | head -5
