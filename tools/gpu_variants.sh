# Library variants (build/libs/*.so from tools/variants.py NAME="-DMACRO=V ...") A/B against the
# working tree: the default bench's step, row kernel, predict and whole-architecture times, twice.
# Usage on the box: VAR_ARGS="--loss sqh --margin-bias 3" bash tools/gpu_variants.sh
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for i in 1 2; do for lib in paper_2306_03725_b200/libfixedfanin.so $(ls build/libs/*.so 2>/dev/null); do
  FIXEDFANIN_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --steps 500 --e2e-steps 50 --repeats 1 ${VAR_ARGS:-} 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '${VAR_ARGS:-}', 'step', round(d['ms_per_step'],4), 'kern', round(d['roofline']['avg_launch_ms'],4), 'pred', round(d['predict']['ms_per_batch'],4), 'model', round(d['model']['ms_per_step'],4))"
done; done
