python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
for mode in atomic csc; do
  timeout 300 python bench.py --no-cpu-baseline --steps 300 --e2e-steps 10 --dh-mode $mode > gpurun_out/hy_$mode.json 2>/dev/null
  echo $mode $(tail -1 gpurun_out/hy_$mode.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['launches_per_step'])")
done
for f in 0.3 0.45 0.6 0.75; do
  timeout 300 python bench.py --no-cpu-baseline --steps 300 --e2e-steps 10 --dh-mode hybrid --hybrid-frac $f > gpurun_out/hy_$f.json 2>/dev/null
  echo hybrid $f $(tail -1 gpurun_out/hy_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['launches_per_step'])")
done
