#!/bin/bash
# dynamic-scheduler check: GPU tests then the C3 kernel-family bench (twice)
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -x -m gpu --timeout 300 2>&1 | tail -6
for i in 1 2; do
timeout -s KILL 400 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-gen > gpurun_out/b_sched$i.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b_sched$i.json'));k=d['kernel_ms_per_step'];print(d['ms_per_step'], d['value'], d['ttft_p50_ms'], 'attn', k['attention'], d['gemm_families'], d['clocks']['sm_mhz'])"
done
