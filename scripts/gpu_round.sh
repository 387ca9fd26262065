#!/bin/bash
# round validation: GPU tests, smoke, bench (ours, C3 default)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 900 python -m pytest tests -q -m gpu --timeout 300 2>&1 | tail -25
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout -s KILL 600 python bench.py > gpurun_out/bench_full.json 2>gpurun_out/bench_full.err; tail -3 gpurun_out/bench_full.err; cat gpurun_out/bench_full.json
