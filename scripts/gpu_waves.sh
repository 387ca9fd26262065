#!/bin/bash
# TTFT p50 / throughput trade-off of the cluster-wave count at C3
for wv in ${WAVES:-1 2 3 4 6 8 16}; do
timeout -s KILL 400 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-gen --waves $wv > gpurun_out/b_w$wv.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b_w$wv.json'));print('waves', $wv, 'ms/step', d['ms_per_step'], 'q/s', d['value'], 'ttft p50/p90', d['ttft_p50_ms'], d['ttft_p90_ms'], 'attn', d['kernel_ms_per_step']['attention'], 'idle', d['gpu_idle_ms_per_step'], 'MHz', d['clocks']['sm_mhz'])"
done
