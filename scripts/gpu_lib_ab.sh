#!/bin/bash
# same-box A/B of library builds (LIBS="default _vf ..." -> libsgc_b200[_prof<tag>].so), alternating
for rep in 1 2 3; do for v in ${LIBS:-default}; do
  lib=paper_2505_10951_b200/libsgc_b200.so; [ "$v" != default ] && lib=paper_2505_10951_b200/libsgc_b200_prof$v.so
  SGC_LIB=$lib timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-gen --no-parity --no-c1-pair --no-e2e > gpurun_out/lib_ab.json 2> gpurun_out/lib_ab.err
  python -c "import json; j=json.load(open('gpurun_out/lib_ab.json')); print('$v', j['ms_per_step'], j['ttft_p50_ms'], j['kernel_ms_per_step']['attention'], j['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
