# A/B of the working-tree library against build/libs/*.so (bench predict + train step), then
# the parity tests of the touched kernels and one default bench line.
set -u
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "${AB_TESTS:-predict or topk}" 2>&1 | tail -2
for rep in 1 2; do
for lib in paper_2306_03725_b200/libfixedfanin.so build/libs/*.so; do
  FIXEDFANIN_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --steps 300 --e2e-steps 5 ${AB_ARGS:-} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'pred', round(d['predict']['ms_per_batch'],4), 'step', round(d['ms_per_step'],4), 'big', round(d['inference_large_batch']['predict_ms_per_batch'],3), 'redist', json.dumps(d.get('redistribution')), 'model', round(d['model']['ms_per_step'],4), d['clocks']['sm_mhz'])"
done
done
timeout 600 python bench.py > gpurun_out/ab_bench.json 2> gpurun_out/ab_bench.err; tail -c 300 gpurun_out/ab_bench.err
