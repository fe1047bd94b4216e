# round-1 dev sweep of row-kernel block shapes (libs prebuilt in build/)
python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
for f in build/lib_*.so; do
  FIXEDFANIN_LIB=$PWD/$f timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 50 > gpurun_out/sweep_$(basename $f .so).json 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep_$(basename $f .so).json')); print('$f', round(d['value']), 'ks_ms', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],4), 'pred', round(d['predict']['value']))"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows -s 12 -c 1 -o gpurun_out/prof_ks_r01b python bench.py --steps 3 --warmup 12 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ncu_full_b.log 2>&1; tail -2 gpurun_out/ncu_full_b.log
