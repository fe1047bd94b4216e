set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/bench_r01a.json 2> gpurun_out/bench_r01a.err; tail -3 gpurun_out/bench_r01a.err
cat gpurun_out/bench_r01a.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 61 -c 40 --csv --log-file gpurun_out/launches_r01a.csv python bench.py --steps 20 --warmup 20 --no-cpu-baseline --e2e-steps 5 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows -s 25 -c 1 -o gpurun_out/prof_ks_r01a python bench.py --steps 5 --warmup 25 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
