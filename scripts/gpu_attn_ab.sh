#!/bin/bash
# same-box A/B of the attention kernels, alternating runs
for rep in 1 2; do for k in 0 1; do
  timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-gen --no-parity --no-c1-pair --no-e2e --attn-kernel $k > gpurun_out/ab_attn$k.json 2> gpurun_out/ab_attn$k.err
  python -c "import json; j=json.load(open('gpurun_out/ab_attn$k.json')); print('k=$k', j['ms_per_step'], j['ttft_p50_ms'], j['kernel_ms_per_step']['attention'], j['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
