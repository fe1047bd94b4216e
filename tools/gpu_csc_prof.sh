python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_train_ring|k_dh_csc" -s 12 -c 2 \
  -o gpurun_out/prof_csc python bench.py --steps 3 --warmup 5 --no-cpu-baseline --e2e-steps 2 --dh-mode csc > gpurun_out/ncu_csc.log 2>&1; tail -1 gpurun_out/ncu_csc.log
