python -m pytest tests/test_gpu_parity.py -q -m gpu -k full_size 2>&1 | tail -2
for sh in tiny wiki10-31k wiki-500k amazon-670k amazon-670k-m16k amazon-670k-k64-m65k amazon-3m; do
  timeout 600 python bench.py --shape $sh --steps 500 --warmup 10 --e2e-steps 50 --no-cpu-baseline > gpurun_out/sh.json 2>gpurun_out/sh.err
  python -c "import json; d=json.load(open('gpurun_out/sh.json')); r=d['roofline']; print('$sh', round(d['value']), 'samples/s', round(d['ms_per_step'],4), 'ms/step', 'row_frac', round(r['frac'],3), 'step_frac', round(d['hbm_step']['frac'],3), 'pred', round(d['predict']['value']), 'mem_MB', round(d['memory']['workspace_bytes_per_gpu']/1e6))" || tail -3 gpurun_out/sh.err
done
