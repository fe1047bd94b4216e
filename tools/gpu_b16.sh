# Half-line B <= 16 train kernel: parity tests touching it, then the batch sweep of the bench.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "pipelined_step or lockstep or fused_step or check_finite or graph_replay or host_entry" 2>&1 | tail -4
for B in 1 8 16 32; do timeout 300 python bench.py --batch $B --no-cpu-baseline --steps 500 --e2e-steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B=$B', round(d['value']), 'samples/s', round(d['ms_per_step'],4), 'ms/step')"; done
