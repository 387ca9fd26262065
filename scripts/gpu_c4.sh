#!/bin/bash
for args in "--config c4 --clusters 256" "--config c5" "--config c4 --clusters 8"; do
  tag=$(echo $args | tr -d ' -')
  timeout -s KILL 900 python bench.py $args --steps 2 --warmup 3 --no-cpu --no-e2e --no-gen > gpurun_out/cfg_$tag.json 2> gpurun_out/cfg_$tag.err
  echo "$args rc=$?"; tail -2 gpurun_out/cfg_$tag.err | grep -v warning
  python -c "import json;d=json.load(open('gpurun_out/cfg_$tag.json'));print(' ', d['config']['workload'], d['ms_per_step'], d['value'], d['ttft_p50_ms'], d['roofline']['achieved'], d['config']['prefix_tokens_mean'], d['ttft_semantics'][-40:])" 2>/dev/null
done
