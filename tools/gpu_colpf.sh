python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -q -m gpu -x -k "csc or hybrid or sharded or full_size or model" 2>&1 | tail -2
for r in 1 2; do for mode in csc; do
timeout 300 python bench.py --no-cpu-baseline --steps 300 --e2e-steps 10 --dh-mode $mode 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$mode', d['ms_per_step'], d['roofline']['avg_launch_ms'])"
done; done
timeout 600 ncu --set full --clock-control none -k regex:"k_dh_csc" -s 6 -c 1 -o gpurun_out/prof_col python bench.py --steps 3 --warmup 5 --no-cpu-baseline --e2e-steps 2 --dh-mode csc > /dev/null 2>&1; echo ncu done
