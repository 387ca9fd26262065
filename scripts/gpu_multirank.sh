#!/bin/bash
# N ranks sharing one GPU through the torchrun path (gloo collectives): exercises the sharded
# encode -> all-gather -> redundant clustering -> LPT ownership -> per-rank serving path
export SGC_DIST_BACKEND=gloo
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c3 --steps 2 --warmup 3 --no-cpu > gpurun_out/b_mr2.json 2> gpurun_out/b_mr2.err; echo "rc=$?"; tail -3 gpurun_out/b_mr2.err
python -c "import json;d=json.load(open('gpurun_out/b_mr2.json'));print(d['n_gpus'],d['ms_per_step'],d['value'],d['ttft_p50_ms'],d['config']['parallelism'],d['gpu_launches'])"
