#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 300 python tests/golden/make_c3_labels.py 2>&1 | tail -2
cp tests/golden/c3_labels.json gpurun_out/ 2>/dev/null
timeout -s KILL 1200 python -m pytest tests -q -m gpu -x --timeout 900 2>&1 | tail -5
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_r02.err
python - <<'P'
import json
j = json.load(open('gpurun_out/bench_r02.json'))
print({k: j.get(k) for k in ('value', 'ms_per_step', 'ttft_p50_ms', 'ttft_dequeue_p50_ms')}, j['roofline']['frac'], j['e2e']['value'])
print('embedding', j.get('embedding'))
print('cpu', json.dumps(j.get('cpu_baseline'))[:1500])
print('c1', json.dumps(j.get('c1_pair')))
P
