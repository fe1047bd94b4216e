python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for lib in paper_2306_03725_b200/libfixedfanin.so build/libs/*.so; do
  FIXEDFANIN_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --steps 300 --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['ms_per_step'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done
