#!/bin/bash
# round-end evidence: GPU suite + smoke, the default bench line, the reference arm, the C3 launch
# list and ncu --set full of the three GEMM families and the attention (one C3 wave)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv,noheader
timeout -s KILL 900 python -m pytest tests -q -m gpu --timeout 600 -x 2>&1 | tail -2
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout -s KILL 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
export SGC_PROFILE=1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 0 --no-cpu --no-e2e --no-gen --no-parity --no-c1-pair > /dev/null 2>&1; echo "launches rc=$?"
N="--set full --clock-control none --import-source on --kernel-name-base demangled"
B="python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-gen --no-parity --no-c1-pair --waves 1"
timeout -s KILL 900 ncu $N -k regex:'gemm2_kernel<.int.3' -s 32 -c 1 -o gpurun_out/prof_tanh $B > /dev/null 2>&1; echo "tanh rc=$?"
timeout -s KILL 900 ncu $N -k regex:'gemm2_kernel<.int.4' -s 32 -c 1 -o gpurun_out/prof_qkv $B > /dev/null 2>&1; echo "qkv rc=$?"
timeout -s KILL 900 ncu $N -k regex:'gemm2_kernel<.int.2' -s 64 -c 1 -o gpurun_out/prof_resid $B > /dev/null 2>&1; echo "resid rc=$?"
timeout -s KILL 900 ncu $N -k regex:attn_tc -s 40 -c 1 -o gpurun_out/prof_attn_k1 $B > /dev/null 2>&1; echo "attn rc=$?"
timeout -s KILL 600 ncu $N -k regex:gnn_layer_dmma -s 1 -c 1 -o gpurun_out/prof_gnn_dmma python scripts/prof_embed.py > /dev/null 2>&1; echo "gnn rc=$?"
python - <<'P'
import json
j = json.load(open('gpurun_out/bench.json'))
print({k: j.get(k) for k in ('value', 'ms_per_step', 'ttft_p50_ms')}, j['roofline']['frac'], j['e2e']['value'], j['clocks'])
print('kernels', j['kernel_ms_per_step'])
r = json.load(open('gpurun_out/bench_ref.json'))
print('ref', {k: r.get(k) for k in ('value', 'unit', 'ms_per_step')})
P
