#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity.py -q -x --timeout 200 -k "gemm or decode or c1" 2>&1 | tail -3
timeout -s KILL 600 python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_gen.json 2>gpurun_out/b_gen.err; echo "bench rc=$?"; tail -2 gpurun_out/b_gen.err
python -c "import json;d=json.load(open('gpurun_out/b_gen.json'));print(d['ms_per_step'],d['value'],d['ttft_p50_ms']);print(d['generation'])"
