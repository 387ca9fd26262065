#!/bin/bash
# ncu --set full of the extend W1 (tanh), QKV and residual (Wo) GEMMs of layer 0 (--waves 1)
mkdir -p gpurun_out
export SGC_PROFILE=1
N="--set full --clock-control none --import-source on --kernel-name-base demangled"
B="python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-gen --waves 1"
timeout -s KILL 900 ncu $N -k regex:'gemm2_kernel<.int.3' -s 32 -c 1 -o gpurun_out/prof_tanh $B > gpurun_out/ncu_tanh.out 2>&1; echo "tanh rc=$?"
timeout -s KILL 900 ncu $N -k regex:'gemm2_kernel<.int.4' -s 32 -c 1 -o gpurun_out/prof_qkv $B > gpurun_out/ncu_qkv.out 2>&1; echo "qkv rc=$?"
timeout -s KILL 900 ncu $N -k regex:'gemm2_kernel<.int.2' -s 64 -c 1 -o gpurun_out/prof_resid $B > gpurun_out/ncu_resid.out 2>&1; echo "resid rc=$?"
