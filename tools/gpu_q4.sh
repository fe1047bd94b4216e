python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests -q -m gpu -x -k "predict or host or tiny or model" 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline --steps 500 > gpurun_out/bench_q4.json 2> gpurun_out/bench_q4.err; tail -3 gpurun_out/bench_q4.err
tail -1 gpurun_out/bench_q4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['value'], d['predict'], d['inference_large_batch']['predict_ms_per_batch'], d['model']['ms_per_step'])"
