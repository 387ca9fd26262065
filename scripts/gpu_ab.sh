#!/bin/bash
# A/B of bench options at C3: bash scripts/gpu_ab.sh "<opts A>" "<opts B>" ...
mkdir -p gpurun_out
i=0
for o in "$@"; do
  timeout -s KILL 600 python bench.py --steps 4 --warmup 3 --no-cpu --no-gen --no-parity --no-e2e $o > gpurun_out/ab_$i.json 2>/dev/null
  python -c "import json,sys; j=json.load(open('gpurun_out/ab_$i.json')); print(sys.argv[1], j['ms_per_step'], j['ttft_p50_ms'], j['stage_ms'], j['gpu_idle_ms_per_step'], j['clocks']['sm_mhz'])" "$o"
  i=$((i+1))
done
