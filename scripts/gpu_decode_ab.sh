#!/bin/bash
# decode prefix attention kernel A/B (generation batch at C3), alternating
for rep in 1 2; do for k in 0 1; do
  timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-parity --no-c1-pair --no-e2e --attn-kernel-partial $k > gpurun_out/dab.json 2> gpurun_out/dab.err
  python -c "import json; j=json.load(open('gpurun_out/dab.json')); g=j['generation']; print('partial=$k', j['ms_per_step'], g['ms_per_batch'], g['rt_p50_ms'], g['decode_stage_ms'], g['kernel_ms_per_batch']['attention'], g['kernel_ms_per_batch']['attn_decode'])" 2>&1 | tail -1
done; done
