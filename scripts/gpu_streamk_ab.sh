#!/bin/bash
# decode GEMM A/B (generation batch at C3): stream-K policy (1) / every decode shape (2) / off (0)
for rep in 1 2; do for k in ${MODES:-1 0}; do
  timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-parity --no-c1-pair --no-e2e --gemm-streamk $k > gpurun_out/skab.json 2> gpurun_out/skab.err
  python -c "import json; j=json.load(open('gpurun_out/skab.json')); g=j['generation']; k=g['kernel_ms_per_batch']; print('streamk=$k', j['ms_per_step'], g['ms_per_batch'], g['rt_p50_ms'], g['decode_stage_ms'], round(k['gemm_qkv']+k['gemm_resid']+k['gemm_tanh'],1), g['decode_roofline']['frac'], j['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
