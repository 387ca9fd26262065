#!/bin/bash
# attention parity + a short C3 bench
timeout -s KILL 400 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -k "prefill or members or soft or c1 or capacity or immutable" 2>&1 | tail -5
timeout -s KILL 400 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_quick.json 2>gpurun_out/b_quick.err; tail -3 gpurun_out/b_quick.err
python -c "import json;d=json.load(open('gpurun_out/b_quick.json'));print(d['ms_per_step'],d['value'],d['stage_ms'],d['kernel_ms_per_step'],d['roofline']['achieved'],d['clocks'])"
