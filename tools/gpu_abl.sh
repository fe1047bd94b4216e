python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "pipelined or full_size or fused" 2>&1 | tail -1
for rep in 1 2; do for f in build/*.so; do for mode in atomic csc; do
  FIXEDFANIN_LIB=$PWD/$f timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --e2e-steps 5 --dh-mode $mode > gpurun_out/ab.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$f $mode', 'ms/step', round(d['ms_per_step'],4), 'row_ms/launch', round(d['roofline']['avg_launch_ms'],4))" || tail -3 gpurun_out/ab.json
done; done; done
