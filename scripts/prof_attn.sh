#!/bin/bash
# attention evidence: phase counters (debug build) + one ncu --set full capture of an extend
# attention launch (C3, one wave: fixed launch index)
mkdir -p gpurun_out
TAG=${TAG:-attn}
SGC_LIB=paper_2505_10951_b200/libsgc_b200_prof.so timeout -s KILL 600 python scripts/attn_prof.py > gpurun_out/${TAG}_phases.txt 2>&1; echo "phases rc=$?"
N="--set full --clock-control none --import-source on --kernel-name-base demangled"
B="python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-gen --no-parity --no-c1-pair --waves 1"
timeout -s KILL 900 ncu $N -k regex:attn_tc -s 40 -c 1 -o gpurun_out/prof_${TAG} $B > gpurun_out/ncu_${TAG}.out 2>&1; echo "attn rc=$?"
cat gpurun_out/${TAG}_phases.txt
