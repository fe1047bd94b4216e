python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -4
for mode in atomic csc; do
  timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --e2e-steps 100 --dh-mode $mode > gpurun_out/mode_$mode.json 2>gpurun_out/mode_$mode.err
  python -c "import json; d=json.load(open('gpurun_out/mode_$mode.json')); print('$mode', round(d['value']), 'ms/step', round(d['ms_per_step'],4), 'ks_ms', round(d['roofline']['avg_launch_ms'],4), 'share', round(d['roofline']['kernel_share_of_step'],3), 'e2e', round(d['e2e']['value']))" || tail -5 gpurun_out/mode_$mode.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 70 -c 30 --csv --log-file gpurun_out/launches_csc.csv python bench.py --steps 20 --warmup 20 --no-cpu-baseline --e2e-steps 3 --dh-mode csc > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rows|k_dh_csc" -s 24 -c 2 -o gpurun_out/prof_csc python bench.py --steps 3 --warmup 12 --no-cpu-baseline --e2e-steps 3 --dh-mode csc > gpurun_out/ncu_csc.log 2>&1; tail -1 gpurun_out/ncu_csc.log
