set -x
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/prof_c3.json 2> gpurun_out/prof_c3.err
tail -3 gpurun_out/prof_c3.err
timeout -s KILL 300 python bench.py --config c3 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/b_c3b.json 2>/dev/null; cat gpurun_out/b_c3b.json
