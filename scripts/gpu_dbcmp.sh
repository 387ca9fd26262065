#!/bin/bash
# attention kernel A/B at C3: 128-key single-buffer (attn_db 0) vs 64-key double-buffer (attn_db 1)
for db in 0 1 0 1; do
  timeout -s KILL 400 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-gen --attn-db $db > gpurun_out/b_db$db.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b_db$db.json'));k=d['kernel_ms_per_step'];print('db=$db', d['ms_per_step'], d['value'], 'attn', k['attention'], 'decode', k.get('attn_decode'), d['clocks']['sm_mhz'])"
done
