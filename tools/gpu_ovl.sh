# Overlapped CSC / hybrid tiles: parity tests of the CSC modes, then the dh-mode x split x variant sweep
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -k "csc or hybrid or graph or p_invariant or lockstep or full_size or free_running" 2>&1 | tail -2
for args in "--dh-mode csc" "--dh-mode hybrid --hybrid-frac 0.3" "--dh-mode hybrid --hybrid-frac 0.5" "--dh-mode hybrid --hybrid-frac 0.7"; do
  echo "== $args"
  for lib in paper_2306_03725_b200/libfixedfanin.so build/libs/o22.so build/libs/o42.so build/libs/o31.so build/libs/o33.so build/libs/t32.so build/libs/t24.so; do
    FIXEDFANIN_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --train-only --repeats 3 --steps 300 $args 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],4), round(d['row_kernel_ms_per_step'],4))"
  done
  python bench.py --no-cpu-baseline --train-only --repeats 3 --steps 300 $args --flags 16 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('serial', round(d['ms_per_step'],4), round(d['row_kernel_ms_per_step'],4))"
done
