#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_decode.py -q -x --timeout 200 2>&1 | tail -25
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_attention.py -q -x --timeout 120 2>&1 | tail -3
