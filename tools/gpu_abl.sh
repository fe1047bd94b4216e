python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
FIXEDFANIN_LIB=$PWD/build/ovl_r2_c1.so timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --e2e-steps 5 --flags 8 > gpurun_out/ab.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('no-overlap', 'ms/step', round(d['ms_per_step'],4), 'row_ms/launch', round(d['roofline']['avg_launch_ms'],4))" || tail -3 gpurun_out/ab.json
for f in build/ovl_*.so; do
  FIXEDFANIN_LIB=$PWD/$f timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --e2e-steps 5 > gpurun_out/ab.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$f', 'ms/step', round(d['ms_per_step'],4), 'row_ms/launch', round(d['roofline']['avg_launch_ms'],4))" || tail -3 gpurun_out/ab.json
done
