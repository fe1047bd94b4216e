python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --no-cpu-baseline --steps 300 --e2e-steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['model']; print(d['ms_per_step'], m['ms_per_step'], json.dumps(m['dense_fwd']))"
