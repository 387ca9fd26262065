#!/bin/bash
# cost of the sealed-prefix digest re-check after serving (cache_engine.cpp:210): C3 steps with
# and without it, alternating
for rep in 1 2; do for v in "" "--no-verify-prefix"; do
  timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-gen --no-parity --no-c1-pair --no-e2e $v > gpurun_out/vf.json 2> gpurun_out/vf.err
  python -c "import json; j=json.load(open('gpurun_out/vf.json')); print('${v:-verify}', j['ms_per_step'], j['ttft_p50_ms'], j['kernel_ms_per_step'].get('gnn_encode'), j['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
