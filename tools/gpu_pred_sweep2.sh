python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
FIXEDFANIN_LIB=$PWD/build/libs/libff_pd2_r2_t128.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k predict 2>&1 | tail -1
for lib in paper_2306_03725_b200/libfixedfanin.so build/libs/*.so; do
  FIXEDFANIN_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --steps 50 --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['predict']['ms_per_batch'])"
done
