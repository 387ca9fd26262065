#!/bin/bash
# attention kernel: phase counters (debug lib) + one ncu --set full capture of an extend launch
mkdir -p gpurun_out
SGC_LIB=paper_2505_10951_b200/libsgc_b200_prof.so timeout -s KILL 300 python scripts/attn_prof.py 2>&1 | tail -12
SGC_PROFILE=1 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 40 -c 1 -o gpurun_out/prof_attn python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --waves 1 > /dev/null 2>gpurun_out/ncu_attn.err; tail -2 gpurun_out/ncu_attn.err
