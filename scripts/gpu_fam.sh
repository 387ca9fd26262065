#!/bin/bash
timeout -s KILL 400 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-gen > gpurun_out/b_fam.json 2>gpurun_out/b_fam.err; tail -2 gpurun_out/b_fam.err
python -c "import json;d=json.load(open('gpurun_out/b_fam.json'));print(d['ms_per_step'],d['value'],d['ttft_p50_ms']);print(d['gemm_families']);print(d['kernel_ms_per_step']);print(d['roofline']['achieved'], d['clocks'])"
