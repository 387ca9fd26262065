#!/bin/bash
# GEMM raster A/B at C3 (same box, alternating), then an ncu DRAM-bytes pass per GEMM family
for rep in 1 2; do for r in 0 1; do
  timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-gen --no-parity --no-c1-pair --no-e2e --gemm-raster $r > gpurun_out/ab_r$r.json 2> gpurun_out/ab_r$r.err
  python -c "import json; j=json.load(open('gpurun_out/ab_r$r.json')); print('raster=$r', j['ms_per_step'], j['kernel_ms_per_step']['gemm_qkv'], j['kernel_ms_per_step']['gemm_resid'], j['kernel_ms_per_step']['gemm_tanh'], j['kernel_ms_per_step']['attention'], j['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
for r in 0 1; do
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm2_kernel --csv --log-file gpurun_out/raster$r.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-gen --no-parity --no-c1-pair --no-e2e --waves 1 --gemm-raster $r > /dev/null 2>&1; echo "ncu r=$r rc=$?"
done
