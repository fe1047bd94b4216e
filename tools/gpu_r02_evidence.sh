# Round-2 evidence: full-size predict parity, ncu launch list of the default bench command, ncu --set full
# of the dominant kernel (k_train_ring) and of the wide predict kernel, per-shape bench lines.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "full_amazon_670k" 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 20 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 2 > gpurun_out/launches.log 2>&1; tail -1 gpurun_out/launches.log | cut -c1-100
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_train_ring" -s 6 -c 1 \
  -o gpurun_out/prof_train python bench.py --steps 3 --warmup 5 --repeats 1 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_train.log 2>&1; tail -1 gpurun_out/ncu_train.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_predict_wide" -s 1 -c 1 \
  -o gpurun_out/prof_wide python tools/pred_sweep.py 1024 > gpurun_out/ncu_wide.log 2>&1; tail -1 gpurun_out/ncu_wide.log
bash tools/gpu_shapes.sh
