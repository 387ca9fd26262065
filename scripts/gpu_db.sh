#!/bin/bash
timeout -s KILL 300 python -m pytest tests/test_gpu_attention.py -q -x --timeout 120 2>&1 | tail -3
timeout -s KILL 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode.py tests/test_gpu_fullsize.py -q -x --timeout 200 -m gpu 2>&1 | grep -E "assert |FAILED|passed|failed" | head
bash scripts/gpu_fam.sh
