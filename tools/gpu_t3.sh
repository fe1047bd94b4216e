python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_dense.py -q -m gpu -x -k "full_size" 2>&1 | tail -30
