#!/bin/bash
# A/B of library variants at C3 (kernel-family bench incl. encode / cluster stages), alternating
for i in 1 2; do
for lib in "$@"; do
SGC_LIB=paper_2505_10951_b200/$lib timeout -s KILL 400 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-gen > gpurun_out/b_ab.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b_ab.json'));k=d['kernel_ms_per_step'];print('$lib', d['ms_per_step'], d['value'], d['ttft_p50_ms'], 'gnn', k['gnn_encode'], 'aggl', k['agglomerate'], 'attn', k['attention'], 'stages', d['stage_ms'], d['clocks']['sm_mhz'])"
done; done
