# compute-sanitizer over the small-shape GPU tests: memcheck (dense, predict incl. the per-line ring and
# the two-pass wide kernel, tiny/host/hybrid/pipelined parity), racecheck (dense, ring and wide predict).
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
export PYTHONUNBUFFERED=1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_dense.py -q -m gpu -x -k "not full_size" > gpurun_out/san_mem_dense.txt 2>&1; tail -3 gpurun_out/san_mem_dense.txt
timeout 1500 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "(predict or tiny or host or hybrid or pipelined) and not full_amazon and not 200003" > gpurun_out/san_mem_parity.txt 2>&1; tail -3 gpurun_out/san_mem_parity.txt
timeout 1200 compute-sanitizer --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_dense.py -q -m gpu -x -k "forward_matches or backward_adam_lockstep" > gpurun_out/san_race_dense.txt 2>&1; tail -3 gpurun_out/san_race_dense.txt
timeout 1200 compute-sanitizer --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "predict_topk_bit_exact and (5000 or 2000 or 2500 or 20011 or 37)" > gpurun_out/san_race_pred.txt 2>&1; tail -3 gpurun_out/san_race_pred.txt
