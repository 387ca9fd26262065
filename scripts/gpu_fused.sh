#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -q -x --timeout 200 2>&1 | tail -4
timeout -s KILL 400 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-gen > gpurun_out/b_quick.json 2>gpurun_out/b_quick.err; echo "bench rc=$?"; tail -2 gpurun_out/b_quick.err
python -c "import json;d=json.load(open('gpurun_out/b_quick.json'));print(d['ms_per_step'],d['value'],d['ttft_p50_ms'],d['stage_ms'],d['kernel_ms_per_step'],d['gpu_idle_ms_per_step'],d['roofline']['achieved'],d['clocks'])"
