#!/bin/bash
# every BASELINE config through bench.py once (robustness + numbers): c1, c2, c4 (c = 8, 64, 256), c5
for args in "--config c1" "--config c2" "--config c4 --clusters 8" "--config c4 --clusters 64" "--config c4 --clusters 256" "--config c5"; do
  tag=$(echo $args | tr -d ' -')
  timeout -s KILL 900 python bench.py $args --steps 2 --warmup 3 --no-cpu --no-e2e --no-gen --no-parity > gpurun_out/cfg_$tag.json 2> gpurun_out/cfg_$tag.err
  echo "$args rc=$?"; tail -2 gpurun_out/cfg_$tag.err | grep -v warning
  python -c "import json;d=json.load(open('gpurun_out/cfg_$tag.json'));print(' ', d['config']['workload'], d['ms_per_step'], d['value'], d['ttft_p50_ms'], d['roofline']['achieved'], d['config']['prefix_tokens_mean'], d['ttft_semantics'].split('(')[1].split(')')[0], d['clocks']['sm_mhz'])" 2>/dev/null
done
