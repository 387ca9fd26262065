#!/bin/bash
# A/B: dynamic unit claiming (libsgc_b200.so) vs the static stride (libsgc_b200_profstatic.so), alternating
for i in 1 2; do
for lib in libsgc_b200.so libsgc_b200_profstatic.so; do
SGC_LIB=paper_2505_10951_b200/$lib timeout -s KILL 400 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-gen > gpurun_out/b_ab.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b_ab.json'));k=d['kernel_ms_per_step'];g=d['gemm_families'];print('$lib', d['ms_per_step'], d['value'], 'attn', k['attention'], 'qkv', g['gemm_qkv']['ms_per_step'], 'resid', g['gemm_resid']['ms_per_step'], 'tanh', g['gemm_tanh']['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
