python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
run() {  # label lib flags mode
  FIXEDFANIN_LIB=$2 timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --e2e-steps 20 --dh-mode $4 --flags $3 > gpurun_out/sw.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('$1 $4', round(d['value']), 'ms/step', round(d['ms_per_step'],4), 'row_ms/launch', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/sw.json
}
for mode in csc atomic; do
  run pipe $PWD/paper_2306_03725_b200/libfixedfanin.so 0 $mode
  for f in build/lib_ring_*.so; do run $(basename $f .so) $PWD/$f 8 $mode; done
done
