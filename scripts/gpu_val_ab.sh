#!/bin/bash
# headline A/B (value with per-kernel timing on, e2e without) of library variants, alternating
for i in 1 2; do
for lib in "$@"; do
SGC_LIB=paper_2505_10951_b200/$lib timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-gen > gpurun_out/b_vab.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b_vab.json'));print('$lib', d['ms_per_step'], d['value'], 'idle', d['gpu_idle_ms_per_step'], 'e2e', round(d['e2e']['value'],1), 'ttft', d['ttft_p50_ms'], d['clocks']['sm_mhz'])"
done; done
