#!/bin/bash
# round-2 validation: new parity + multi-rank tests, then a 2-rank bench sharing the GPU (gloo)
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/test_gpu_fullwidth.py tests/test_gpu_multirank.py -x -q -s -m gpu --timeout 900 2>&1 | tail -40
SGC_DIST_BACKEND=gloo timeout -s KILL 600 python bench.py --gpus 2 --steps 2 --warmup 3 --config c3 --no-cpu --no-gen \
   > gpurun_out/bench_mr2.json 2> gpurun_out/bench_mr2.err; echo "mr2 rc=$?"; tail -5 gpurun_out/bench_mr2.err
python -c "import json; j=json.load(open('gpurun_out/bench_mr2.json')); print({k: j[k] for k in ('value','n_gpus','ms_per_step','ttft_p50_ms')}, j['config']['prefix_tokens_mean'], j['roofline']['achieved'], j['gemm_families'])"
