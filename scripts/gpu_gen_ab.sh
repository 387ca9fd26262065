#!/bin/bash
# generation A/B (decode) of library variants at C3
for i in 1 2; do
for lib in "$@"; do
SGC_LIB=paper_2505_10951_b200/$lib timeout -s KILL 600 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_gab.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b_gab.json'));g=d['generation'];r=g['decode_roofline'];print('$lib', d['ms_per_step'], 'gen ms', g['ms_per_batch'], 'rt p50', g['rt_p50_ms'], 'dec gemm ms', r['gemm_ms_per_batch'], 'GB/s', r['achieved'], r['frac'])"
done; done
