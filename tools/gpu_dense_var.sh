# Dense forward time vs m (tiles per SM: 148 tiles = 18944 columns).
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for m in 9472 18944 28416 32768 37888 56832 75776; do timeout 300 python tools/dense_fwd_time.py $m; done
