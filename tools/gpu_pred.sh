# Wide predict: parity tests of the predict kernels, then the batch sweep (variants of the wide kernel, generic).
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "predict or graph_replay" 2>&1 | tail -5
timeout 300 python tools/pred_sweep.py
for v in build/libs/*.so; do echo "== $v"; FIXEDFANIN_LIB=$PWD/$v timeout 300 python tools/pred_sweep.py 64 256 1024; done
timeout 300 python tools/pred_sweep.py --no-pipe 64 256 1024
