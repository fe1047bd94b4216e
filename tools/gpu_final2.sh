# Session-3 follow-up: default bench line (with the cuda_graph section), and memcheck over the
# kernels changed in session 3 (vectorized prep / dh_out, redistribution, device step counter,
# host-entry loss store, graph replay).
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default2.json 2> gpurun_out/bench_default2.err; tail -1 gpurun_out/bench_default2.json | cut -c1-200
export PYTHONUNBUFFERED=1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -m gpu -x \
  -k "redistribution or host or graph or tiny or lockstep" > gpurun_out/san_mem_s3.txt 2>&1; tail -3 gpurun_out/san_mem_s3.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -m gpu -x \
  -k "redistribution_all_ties or host_entry_point_loss" > gpurun_out/san_race_s3.txt 2>&1; tail -3 gpurun_out/san_race_s3.txt
