# Round measurement: parity tests, smoke, default bench, reference arm, ncu launch list, ncu --set full of the fused kernel.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt; cat gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json | cut -c1-400
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/launches.log 2>&1; tail -1 gpurun_out/launches.log | cut -c1-100
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_train" -s 6 -c 1 \
  -o gpurun_out/prof_full python bench.py --steps 3 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_predict_reg|k_merge_topk_block" -s 10 -c 2 \
  -o gpurun_out/prof_pred python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_pred.log 2>&1; tail -1 gpurun_out/ncu_pred.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dense_fwd|k_dense_bwd" -s 2 -c 2 \
  -o gpurun_out/prof_dense python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_dense.log 2>&1; tail -1 gpurun_out/ncu_dense.log
FF_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 50 --warmup 5 --repeats 2 --no-cpu-baseline --e2e-steps 10 > gpurun_out/mr.json 2> gpurun_out/mr.err; echo "mr rc=$?"
