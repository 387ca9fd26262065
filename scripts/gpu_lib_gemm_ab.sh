#!/bin/bash
# same-box A/B of library builds on the C3 step's GEMM families (LIBS="default tag ..." -> libsgc_b200[_prof<tag>].so)
for rep in 1 2 3; do for v in ${LIBS:-default}; do
  lib=paper_2505_10951_b200/libsgc_b200.so; [ "$v" != default ] && lib=paper_2505_10951_b200/libsgc_b200_prof$v.so
  SGC_LIB=$lib timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-gen --no-parity --no-c1-pair --no-e2e > gpurun_out/lg.json 2> gpurun_out/lg.err
  python -c "import json; j=json.load(open('gpurun_out/lg.json')); k=j['kernel_ms_per_step']; print('$v', j['ms_per_step'], k['gemm_qkv'], k['gemm_resid'], k['gemm_tanh'], j['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
