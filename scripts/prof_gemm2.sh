#!/bin/bash
SGC_PROFILE=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm2_kernel -s 130 -c 2 -o gpurun_out/prof_gemm2 python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --waves 1 > /dev/null 2>gpurun_out/ncu_gemm2.err; tail -2 gpurun_out/ncu_gemm2.err
