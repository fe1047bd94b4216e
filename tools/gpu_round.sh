# round-end style measurement: tests, default bench (both modes), launch list of the default
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -m pytest tests/ -q -m gpu 2>&1 | tail -2
python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
timeout 900 python bench.py --dh-mode atomic --no-cpu-baseline > gpurun_out/bench_atomic.json 2> gpurun_out/bench_atomic.err; cat gpurun_out/bench_atomic.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 90 -c 60 --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 30 --warmup 30 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1; wc -l gpurun_out/launches_default.csv
