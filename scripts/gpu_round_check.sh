#!/bin/bash
# round check of the current build: GPU suite + smoke + default bench line, then compute-sanitizer
# over the attention / paged-KV / fork suites (memcheck, synccheck, racecheck) and ncu captures of
# one extend attention launch and the C3 launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout -s KILL 900 python -m pytest tests -q -m gpu --timeout 600 -x 2>&1 | tail -3
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout -s KILL 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - <<'P'
import json
j = json.load(open('gpurun_out/bench.json'))
print({k: j.get(k) for k in ('value', 'ms_per_step', 'ttft_p50_ms')}, j['roofline']['frac'], j['e2e']['value'], j['clocks'])
print('kernels', j['kernel_ms_per_step'])
print('gen', {k: j['generation'][k] for k in ('ms_per_batch', 'rt_p50_ms')})
P
S=/usr/local/cuda/bin/compute-sanitizer
run() { echo "== $*"; timeout -s KILL 1500 "$@" 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" | tail -4; }
run $S --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_attention.py tests/test_gpu_paged_kv.py tests/test_gpu_fork.py tests/test_gpu_decode.py -q -m gpu -x
run $S --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_attention.py -q -m gpu -x
run $S --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_attention.py -q -m gpu -x
KERNELS=1 bash scripts/prof_attn.sh
export SGC_PROFILE=1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 0 --no-cpu --no-e2e --no-gen --no-parity --no-c1-pair > /dev/null 2>&1; echo "launches rc=$?"
