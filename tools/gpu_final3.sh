# Session-3 closing run: all GPU tests, smoke, and the default bench line at the final head.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/pytest_gpu3.txt; cat gpurun_out/pytest_gpu3.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default3.json 2> gpurun_out/bench_default3.err; tail -1 gpurun_out/bench_default3.json | cut -c1-300
