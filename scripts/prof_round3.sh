#!/bin/bash
# round evidence refresh: default bench line (all keys) + launch list of one C3 step + ncu --set full
# of the extend W1 (tanh), QKV and residual GEMMs and of an extend attention launch
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout -s KILL 900 python bench.py > gpurun_out/bench_full.json 2>gpurun_out/bench_full.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_full.err
bash scripts/prof_round2.sh
