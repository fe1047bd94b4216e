python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_dense.py -q -m gpu -x 2>&1 | tail -4
timeout 900 python bench.py --no-cpu-baseline --steps 300 > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err; tail -3 gpurun_out/bench_m.err
tail -1 gpurun_out/bench_m.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['model']; print(d['ms_per_step'], m['ms_per_step'], m['dense_fwd']['ms'], m['dense_fwd']['frac'], m['dense_bwd_adam']['ms'], m['dense_bwd_adam']['frac'])"
