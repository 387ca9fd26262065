#!/bin/bash
# phase counters of the attention kernels (debug build): one line set per kernel variant
for k in ${KERNELS:-0 1}; do
  echo "== attn_kernel $k"
  SGC_ATTN_KERNEL=$k SGC_LIB=paper_2505_10951_b200/libsgc_b200_prof.so timeout -s KILL 240 python scripts/attn_prof.py 2>&1 | tail -30
done
