python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for f in build/lib_*.so; do for mode in csc atomic; do
  FIXEDFANIN_LIB=$PWD/$f timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 20 --dh-mode $mode > gpurun_out/sw.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('$f $mode', round(d['value']), 'ms/step', round(d['ms_per_step'],4), 'row_ms/launch', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/sw.json
done; done
