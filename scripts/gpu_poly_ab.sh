#!/bin/bash
# share of exp2 pairs on the FMA pipe (polynomial) vs MUFU, attention kernel at C3: variant builds
# (make prof PROF_TAG=_pNM PROF_BASE= PROF_DEFS="-DSGC_POLY_NUM=N -DSGC_POLY_DEN=M"), alternating
for rep in 1 2; do for v in "" _p14 _p25 _p12; do
  lib=paper_2505_10951_b200/libsgc_b200${v:+_prof$v}.so
  SGC_LIB=$lib timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-gen --no-parity --no-c1-pair --no-e2e > gpurun_out/poly.json 2> gpurun_out/poly.err
  python -c "import json; j=json.load(open('gpurun_out/poly.json')); print('${v:-_p13}', j['ms_per_step'], j['kernel_ms_per_step']['attention'], j['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
