#!/bin/bash
# round profile refresh: launch list of one C3 step + ncu --set full of the extend W1 (tanh), QKV,
# residual (Wo) GEMMs and of an extend attention launch (--waves 1: fixed launch indices)
mkdir -p gpurun_out
export SGC_PROFILE=1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 0 --no-cpu --no-e2e --no-gen > gpurun_out/prof_c3.json 2> gpurun_out/prof_c3.err; echo "launches rc=$?"
N="--set full --clock-control none --import-source on --kernel-name-base demangled"
B="python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-gen --waves 1"
timeout -s KILL 900 ncu $N -k regex:'gemm2_kernel<.int.3' -s 32 -c 1 -o gpurun_out/prof_tanh $B > gpurun_out/ncu_tanh.out 2>&1; echo "tanh rc=$?"
timeout -s KILL 900 ncu $N -k regex:'gemm2_kernel<.int.4' -s 32 -c 1 -o gpurun_out/prof_qkv $B > gpurun_out/ncu_qkv.out 2>&1; echo "qkv rc=$?"
timeout -s KILL 900 ncu $N -k regex:'gemm2_kernel<.int.2' -s 64 -c 1 -o gpurun_out/prof_resid $B > gpurun_out/ncu_resid.out 2>&1; echo "resid rc=$?"
timeout -s KILL 900 ncu $N -k regex:attn_tc -s 40 -c 1 -o gpurun_out/prof_attn $B > gpurun_out/ncu_attn.out 2>&1; echo "attn rc=$?"
