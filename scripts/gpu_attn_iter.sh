#!/bin/bash
# attention iteration: full-size attention parity, LM parity subset, C3 quick bench, phase profile
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_attention.py -q -x --timeout 120 2>&1 | tail -3
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -k "prefill or members or soft or c1 or capacity or immutable or waves" 2>&1 | tail -3
timeout -s KILL 400 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_quick.json 2>gpurun_out/b_quick.err; echo "bench rc=$?"; tail -2 gpurun_out/b_quick.err
python -c "import json;d=json.load(open('gpurun_out/b_quick.json'));print(d['ms_per_step'],d['value'],d['ttft_p50_ms'],d['stage_ms'],d['kernel_ms_per_step'],d['roofline']['achieved'],d['clocks'])"
SGC_LIB=paper_2505_10951_b200/libsgc_b200_prof.so timeout -s KILL 300 python scripts/attn_prof.py 2>&1 | tail -10
