# Predict variants: the batch sweep for the working-tree library and each build/libs/*.so.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 300 python tools/pred_sweep.py 32 64 256 1024
for v in build/libs/*.so; do echo "== $v"; FIXEDFANIN_LIB=$PWD/$v timeout 300 python tools/pred_sweep.py 32 256 1024; done
