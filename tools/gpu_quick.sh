for mode in csc atomic; do
  timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --e2e-steps 20 --dh-mode $mode > gpurun_out/q_$mode.json 2>gpurun_out/q_$mode.err
  python -c "import json; d=json.load(open('gpurun_out/q_$mode.json')); print('$mode', round(d['value']), 'ms/step', round(d['ms_per_step'],4), 'row_ms', round(d['roofline']['avg_launch_ms'],4), 'pred', round(d['predict']['value']))" || tail -5 gpurun_out/q_$mode.err
  timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --e2e-steps 20 --dh-mode $mode --loss sqh --margin-bias 3 > gpurun_out/q_$mode.json 2>gpurun_out/q_$mode.err
  python -c "import json; d=json.load(open('gpurun_out/q_$mode.json')); print('$mode sqh3', round(d['value']), 'ms/step', round(d['ms_per_step'],4), 'row_ms', round(d['roofline']['avg_launch_ms'],4))" || tail -5 gpurun_out/q_$mode.err
done
