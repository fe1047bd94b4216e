python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dense|k_predict_ring" -s 10 -c 3 \
  -o gpurun_out/prof2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu2.log 2>&1; tail -1 gpurun_out/ncu2.log
