#!/bin/bash
# A/B of library variants at C3 (kernel-family bench), alternating: bash scripts/gpu_libs_ab.sh lib1 lib2 ...
for i in 1 2; do
for lib in "$@"; do
SGC_LIB=paper_2505_10951_b200/$lib timeout -s KILL 400 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-gen > gpurun_out/b_ab.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b_ab.json'));k=d['kernel_ms_per_step'];g=d['gemm_families'];print('$lib', d['ms_per_step'], d['value'], 'attn', k['attention'], 'qkv', g['gemm_qkv']['ms_per_step'], 'resid', g['gemm_resid']['ms_per_step'], 'tanh', g['gemm_tanh']['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
