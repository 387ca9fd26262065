#!/bin/bash
mkdir -p gpurun_out
export SGC_PROFILE=1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm2_kernel<4" -s 32 -c 1 -o gpurun_out/prof_qkv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-gen --waves 1 > /dev/null 2>gpurun_out/ncu_qkv.err; echo "qkv rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm2_kernel<2" -s 64 -c 1 -o gpurun_out/prof_resid python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-gen --waves 1 > /dev/null 2>gpurun_out/ncu_resid.err; echo "resid rc=$?"
