python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for mode in atomic csc; do
timeout 300 python bench.py --no-cpu-baseline --steps 300 --e2e-steps 10 --dh-mode $mode 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$mode', d['ms_per_step'], d['roofline']['avg_launch_ms'])"
done
for sh in tiny wiki10-31k; do
timeout 300 python bench.py --no-cpu-baseline --steps 300 --e2e-steps 10 --shape $sh 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sh', d['ms_per_step'], d['roofline']['avg_launch_ms'])"
done
