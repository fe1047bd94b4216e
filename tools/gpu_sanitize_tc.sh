python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
export PYTHONUNBUFFERED=1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_dense.py -q -m gpu -x -k "not full_size" > gpurun_out/san_mem_tc.txt 2>&1; grep -E "passed|failed|ERROR SUMMARY" gpurun_out/san_mem_tc.txt | tail -3
timeout 1500 compute-sanitizer --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_dense.py -q -m gpu -x -k "forward_matches and tcgen05" > gpurun_out/san_race_tc.txt 2>&1; grep -E "passed|failed|RACECHECK SUMMARY" gpurun_out/san_race_tc.txt | tail -3
timeout 1500 compute-sanitizer --tool synccheck --print-limit 5 python -m pytest tests/test_gpu_dense.py -q -m gpu -x -k "forward_matches and tcgen05" > gpurun_out/san_sync_tc.txt 2>&1; grep -E "passed|failed|ERROR SUMMARY" gpurun_out/san_sync_tc.txt | tail -3
