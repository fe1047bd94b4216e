# Closing measurement at the head: all GPU tests, smoke, the default bench line, the reference arm, the
# 2-rank gloo N > 1 line, the long run, the ncu launch list.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt; tail -1 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json | cut -c1-200
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json | cut -c1-200
FF_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 50 --warmup 5 --repeats 2 --no-cpu-baseline --e2e-steps 10 > gpurun_out/mr.json 2> gpurun_out/mr.err; echo "mr rc=$?"
timeout 900 python tools/long_run.py 10000 > gpurun_out/long_run.txt 2>&1; tail -2 gpurun_out/long_run.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 20 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 2 > gpurun_out/launches.log 2>&1; echo "ncu rc=$?"
