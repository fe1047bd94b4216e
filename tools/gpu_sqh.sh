for mode in csc atomic; do
  timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --e2e-steps 5 --dh-mode $mode > gpurun_out/s.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/s.json')); c=d['config']; print('$mode bce', round(d['value']), 'ms/step', round(d['ms_per_step'],4))" || tail -3 gpurun_out/s.json
  for mb in 0 1 2 3 5; do
    timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --e2e-steps 5 --dh-mode $mode --loss sqh --margin-bias $mb > gpurun_out/s.json 2>&1
    python -c "import json; d=json.load(open('gpurun_out/s.json')); c=d['config']; print('$mode sqh mb=$mb skip', round(c['grad_skip_fraction'],4), round(d['value']), 'ms/step', round(d['ms_per_step'],4), 'row', round(d['roofline']['avg_launch_ms'],4))" || tail -3 gpurun_out/s.json
  done
done
