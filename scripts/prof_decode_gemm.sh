#!/bin/bash
# ncu --set full of one decode-step GEMM launch (QKV weights, 200 rows) on the stream-K kernel
# and on the dynamic-tile pair kernel (scripts/decode_gemm_sweep.py drives both)
mkdir -p gpurun_out
for mode in 1 0; do
  MODES=$mode ROWS=200 timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:gemm \
    --launch-skip 5 --launch-count 1 -o gpurun_out/dec_gemm_sk$mode -f python scripts/decode_gemm_sweep.py > gpurun_out/ncu_dec_sk$mode.log 2>&1
  tail -2 gpurun_out/ncu_dec_sk$mode.log
done
