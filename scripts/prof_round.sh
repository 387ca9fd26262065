#!/bin/bash
# round profile set: launch list of one C3 step, ncu --set full of the extend W1 GEMM and of an
# extend attention launch (both --waves 1 so the launch indices are fixed)
mkdir -p gpurun_out
export SGC_PROFILE=1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/prof_c3.json 2> gpurun_out/prof_c3.err; echo "launches rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm2_kernel -s 130 -c 1 -o gpurun_out/prof_gemm2 python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --waves 1 > /dev/null 2>gpurun_out/ncu_gemm2.err; echo "gemm rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 40 -c 1 -o gpurun_out/prof_attn python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --waves 1 > /dev/null 2>gpurun_out/ncu_attn.err; echo "attn rc=$?"
