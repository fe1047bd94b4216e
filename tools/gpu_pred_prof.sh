python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_predict_wide" -c 1 \
  -o gpurun_out/prof_wide python tools/pred_sweep.py 256 > gpurun_out/ncu_wide.log 2>&1; tail -2 gpurun_out/ncu_wide.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_predict" -c 1 \
  -o gpurun_out/prof_gen python tools/pred_sweep.py --no-pipe 256 > gpurun_out/ncu_gen.log 2>&1; tail -2 gpurun_out/ncu_gen.log
