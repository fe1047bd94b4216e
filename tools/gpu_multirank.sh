python -m pytest tests/ -q -m gpu 2>&1 | tail -1
FF_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/mr.json 2> gpurun_out/mr.err
echo "rc=$?"; python -c "import json; d=json.load(open('gpurun_out/mr.json')); print(d['n_gpus'], d['value'], d['gpu_launches'], d['config']['parallelism'])"; tail -3 gpurun_out/mr.err
timeout 600 python bench.py --steps 1000 --warmup 20 --e2e-steps 200 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['gpu_launches'])"
