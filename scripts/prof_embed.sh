#!/bin/bash
# launch list + ncu --set full of the embedding / clustering / representative kernels at C3
mkdir -p gpurun_out
export GNN_TILE=${GNN_TILE:-1}
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/embed_launches.csv python scripts/prof_embed.py > /dev/null 2>&1; echo "launches rc=$?"
N="--set full --clock-control none --import-source on --kernel-name-base demangled"
timeout -s KILL 600 ncu $N -k regex:gnn_layer_gemm -s 1 -c 1 -o gpurun_out/prof_gnn_gemm python scripts/prof_embed.py > /dev/null 2>&1; echo "gemm rc=$?"
timeout -s KILL 600 ncu $N -k regex:gnn_aggregate -s 1 -c 1 -o gpurun_out/prof_gnn_agg python scripts/prof_embed.py > /dev/null 2>&1; echo "agg rc=$?"
timeout -s KILL 600 ncu $N -k regex:"gnn_pool|union_prompt|prompt_gather|pairwise|agglomerate|text_feature" -c 6 -o gpurun_out/prof_embed_misc python scripts/prof_embed.py > /dev/null 2>&1; echo "misc rc=$?"
