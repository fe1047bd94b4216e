python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_dense.py -q -m gpu -x 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline --steps 200 --e2e-steps 10 > gpurun_out/bench_q7.json 2> gpurun_out/bench_q7.err; tail -2 gpurun_out/bench_q7.err
tail -1 gpurun_out/bench_q7.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['model']; print(d['ms_per_step'], m['ms_per_step'], m['dense_fwd']['ms'], m['dense_bwd_adam']['ms'], m['dense_bwd_adam']['frac'], d['predict']['ms_per_batch'])"
