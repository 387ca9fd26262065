#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests/test_gpu_attention.py tests/test_gpu_parity.py tests/test_gpu_decode.py -q -x --timeout 200 2>&1 | tail -3
for sp in 1 0; do
timeout -s KILL 400 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-gen --attn-split $sp > gpurun_out/b_split$sp.json 2>gpurun_out/b_split$sp.err; echo "bench split=$sp rc=$?"; tail -2 gpurun_out/b_split$sp.err
python -c "import json;d=json.load(open('gpurun_out/b_split$sp.json'));print(d['ms_per_step'],d['value'],d['ttft_p50_ms'],d['kernel_ms_per_step']['attention'],d['kernel_ms_per_step']['gemm'],d['gpu_idle_ms_per_step'],d['clocks'])"
SGC_ATTN_SPLIT=$sp SGC_LIB=paper_2505_10951_b200/libsgc_b200_prof.so timeout -s KILL 300 python scripts/attn_prof.py 2>&1 | tail -11
done
