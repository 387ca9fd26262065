#!/bin/bash
# every BASELINE config through bench.py once (robustness + numbers): c1, c2, the C4 cluster-count
# sweep (reuse ratio = prefill tokens without / with the cache), c5
for args in "--config c1" "--config c2" "--config c4 --clusters 8" "--config c4 --clusters 16" "--config c4 --clusters 64" "--config c4 --clusters 256" "--config c5"; do
  tag=$(echo $args | tr -d ' -')
  timeout -s KILL 900 python bench.py $args --steps 2 --warmup 3 --no-cpu --no-e2e --no-gen --no-parity --no-c1-pair > gpurun_out/cfg_$tag.json 2> gpurun_out/cfg_$tag.err
  echo "$args rc=$?"; tail -2 gpurun_out/cfg_$tag.err | grep -v warning
  python -c "import json;d=json.load(open('gpurun_out/cfg_$tag.json'));c=d['config'];print(' ', c['workload'], 'ms/step', d['ms_per_step'], 'q/s', d['value'], 'TTFT p50', d['ttft_p50_ms'], 'GEMM TF/s', d['roofline']['achieved'], 'prefix', round(c['prefix_tokens_mean'], 1), 'reuse', c.get('reuse_ratio'), 'MHz', d['clocks']['sm_mhz'])" 2>/dev/null
done
