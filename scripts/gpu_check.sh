#!/bin/bash
# parity (attention-related) + C3 bench + ncu full captures of the top kernels
set -x
timeout -s KILL 400 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -k "prefill or members or soft or c1 or capacity or immutable" 2>&1 | tail -5
timeout -s KILL 400 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e > gpurun_out/b_c3d.json 2>gpurun_out/b_c3d.err; tail -3 gpurun_out/b_c3d.err; cat gpurun_out/b_c3d.json
SGC_PROFILE=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 70 -c 1 -o gpurun_out/prof_gemm python bench.py --config c3 --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>gpurun_out/ncu_gemm.err; tail -2 gpurun_out/ncu_gemm.err
SGC_PROFILE=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 40 -c 1 -o gpurun_out/prof_attn python bench.py --config c3 --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>gpurun_out/ncu_attn.err; tail -2 gpurun_out/ncu_attn.err
ls -la gpurun_out
