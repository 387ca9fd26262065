#!/bin/bash
for t in "" p2 p0; do echo "== variant '$t'"; SGC_LIB=paper_2505_10951_b200/libsgc_b200_prof$t.so timeout -s KILL 300 python scripts/attn_prof.py 2>&1 | tail -11; done
