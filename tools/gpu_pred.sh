# Predict: the batch sweep for the working-tree library and each build/libs/*.so variant.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 300 python tools/pred_sweep.py ${PRED_BS:-32 256 1024}
for v in $(ls build/libs/*.so 2>/dev/null); do echo "== $v"; FIXEDFANIN_LIB=$PWD/$v timeout 300 python tools/pred_sweep.py ${PRED_BS:-32 256 1024}; done
