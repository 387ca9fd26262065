#!/bin/bash
for wv in 4 8 16; do
timeout -s KILL 400 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-gen --waves $wv > gpurun_out/b_w$wv.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b_w$wv.json'));print($wv, d['ms_per_step'],d['value'],d['ttft_p50_ms'],d['ttft_p90_ms'],d['kernel_ms_per_step']['attention'],d['gpu_idle_ms_per_step'],d['clocks']['sm_mhz'])"
done
