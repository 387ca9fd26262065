#!/bin/bash
# full GPU suite + smoke + default bench (C3)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout -s KILL 1500 python -m pytest tests -q -m gpu --timeout 900 -x 2>&1 | tail -30
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python - <<'P'
import json
j = json.load(open('gpurun_out/bench.json'))
print({k: j.get(k) for k in ('value', 'ms_per_step', 'ttft_p50_ms')}, j['roofline']['frac'], j['e2e']['value'])
print('kernels', j['kernel_ms_per_step'])
print('gen', {k: j['generation'][k] for k in ('ms_per_batch', 'rt_p50_ms')} if j.get('generation') else None)
print('parity', json.dumps(j.get('parity')))
P
