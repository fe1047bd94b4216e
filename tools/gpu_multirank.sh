# The N > 1 bench path with 2 ranks sharing one GPU over gloo (FF_BENCH_BACKEND=gloo): the
# contract line with the per-rank breakdown keys, and the reference arm under torchrun.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
FF_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 50 --warmup 5 --repeats 2 --no-cpu-baseline --e2e-steps 10 > gpurun_out/mr.json 2> gpurun_out/mr.err
echo "rc=$?"; tail -1 gpurun_out/mr.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({k: d[k] for k in ('value','ms_per_step','n_gpus','per_rank','comm','host_enqueue_ms_per_step','e2e')}, indent=1))"; tail -3 gpurun_out/mr.err
FF_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err
echo "rc=$?"; tail -1 gpurun_out/mr_ref.json | cut -c1-200
