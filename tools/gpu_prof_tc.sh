python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dense_fwd_tc" -s 2 -c 1 \
  -o gpurun_out/prof_tc python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_tc.log 2>&1; tail -1 gpurun_out/ncu_tc.log
