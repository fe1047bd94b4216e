python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline --steps 300 > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err; tail -3 gpurun_out/bench_m.err
tail -1 gpurun_out/bench_m.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], json.dumps(d['predict']), json.dumps(d['model'], indent=1))"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dense|k_dropout" -s 20 -c 4 \
  -o gpurun_out/prof_dense python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_dense.log 2>&1; tail -1 gpurun_out/ncu_dense.log
