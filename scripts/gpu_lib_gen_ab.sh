#!/bin/bash
# same-box A/B of library builds on the generation batch (LIBS="default old" -> libsgc_b200[_prof<tag>].so)
for rep in 1 2; do for v in ${LIBS:-default}; do
  lib=paper_2505_10951_b200/libsgc_b200.so; [ "$v" != default ] && lib=paper_2505_10951_b200/libsgc_b200_prof$v.so
  SGC_LIB=$lib timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-parity --no-c1-pair --no-e2e > gpurun_out/lgab.json 2> gpurun_out/lgab.err
  python -c "import json; j=json.load(open('gpurun_out/lgab.json')); g=j['generation']; k=g['kernel_ms_per_batch']; print('$v', j['ms_per_step'], g['ms_per_batch'], g['rt_p50_ms'], g['decode_stage_ms'], k['attn_decode'], k['attention'], j['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
