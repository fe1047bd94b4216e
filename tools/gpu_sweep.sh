# A/B of library variants: bash tools/gpu_sweep.sh "<bench args>" lib1.so lib2.so ...
# (the working-tree library is always the first arm); prints ms/step per arm, 3 rounds interleaved.
ARGS="$1"; shift
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for r in 1 2 3; do
  for lib in paper_2306_03725_b200/libfixedfanin.so "$@"; do
    FIXEDFANIN_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --train-only --repeats 3 $ARGS 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],4), round(d['row_kernel_ms_per_step'],4), d['row_launches_per_step'])"
  done
done
