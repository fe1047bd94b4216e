python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for rep in 1 2; do for mode in csc atomic; do
  timeout 300 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline --e2e-steps 20 --dh-mode $mode > gpurun_out/ab.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$mode', round(d['value']), 'ms/step', round(d['ms_per_step'],4), 'row_ms/launch', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.json
done; done
