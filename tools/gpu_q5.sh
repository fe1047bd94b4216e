python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_dense.py -q -m gpu -x 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline --steps 300 --e2e-steps 20 > gpurun_out/bench_q5.json 2> gpurun_out/bench_q5.err; tail -3 gpurun_out/bench_q5.err
tail -1 gpurun_out/bench_q5.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['model']; print(d['ms_per_step'], m['ms_per_step'], m['dense_fwd']['ms'], m['dense_bwd_adam']['ms'], m['dense_bwd_adam']['frac'], d['predict']['ms_per_batch'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dense" -s 0 -c 2 \
  -o gpurun_out/prof5 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu5.log 2>&1; tail -1 gpurun_out/ncu5.log
