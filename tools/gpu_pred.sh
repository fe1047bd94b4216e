# Predict: parity tests of the predict kernels, then the batch sweep.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py -q -m gpu -k "predict or topk or sharded or model" 2>&1 | tail -3
timeout 300 python tools/pred_sweep.py 16 32 33 64 65 96 97 128 256 1024
for v in $(ls build/libs/*.so 2>/dev/null); do echo "== $v"; FIXEDFANIN_LIB=$PWD/$v timeout 300 python tools/pred_sweep.py 32 256 1024; done
