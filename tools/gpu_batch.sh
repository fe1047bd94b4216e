python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for bb in 16 32 64 128 256; do
timeout 300 python bench.py --no-cpu-baseline --steps 200 --warmup 5 --e2e-steps 5 --batch $bb 2>gpurun_out/batch.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B', $bb, 'samples/s', round(d['value']), 'ms/step', round(d['ms_per_step'],4), 'row_frac', round(d['roofline']['frac'],3), 'step_frac', round(d['hbm_step']['frac'],3), 'pred/s', round(d['predict']['value']))" || tail -3 gpurun_out/batch.err
done
