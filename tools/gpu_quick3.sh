python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "predict or tiny or shard" 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/bench_q3.json 2> gpurun_out/bench_q3.err; tail -1 gpurun_out/bench_q3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['predict'], d['inference_large_batch'])"
