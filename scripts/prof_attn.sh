#!/bin/bash
# ncu --set full of one extend attention launch per kernel variant (C3, one wave: fixed launch
# index); KERNELS="1 0" compares the one-tile kernel (default) with the two-tile kernel
mkdir -p gpurun_out
N="--set full --clock-control none --import-source on --kernel-name-base demangled"
B="python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-gen --no-parity --no-c1-pair --waves 1"
for k in ${KERNELS:-0}; do
timeout -s KILL 900 ncu $N -k regex:attn_ -s 40 -c 1 -o gpurun_out/prof_attn_k$k $B --attn-kernel $k > gpurun_out/ncu_attn_k$k.out 2>&1; echo "attn k=$k rc=$?"
done
