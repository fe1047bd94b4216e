python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fused or tiny or sharded" 2>&1 | tail -2
for mode in atomic csc; do
timeout 300 python bench.py --no-cpu-baseline --steps 300 --e2e-steps 10 --dh-mode $mode 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$mode', d['ms_per_step'], d['roofline']['avg_launch_ms'])"
done
