#!/bin/bash
# compute-sanitizer over the stream-K decode GEMM (cross-CTA flags + fp32 partial slots) and the
# decode path that runs it
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  echo "== $S --tool $tool python -m pytest tests/test_gpu_parity.py -k 'streamk and (77 or 300) and 12288' -q"
  timeout -s KILL 900 $S --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "streamk and (77 or 300) and 12288" 2>&1 | grep -E "passed|failed|SUMMARY|rror" | tail -4
done
echo "== $S --tool memcheck python -m pytest tests/test_gpu_decode.py -q"
timeout -s KILL 900 $S --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_decode.py -q -m gpu -x 2>&1 | grep -E "passed|failed|SUMMARY|rror" | tail -4
