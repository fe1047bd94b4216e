# ncu --set full capture of one fused row-kernel launch per dh mode (round-1 profiling).
for mode in atomic csc; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_train_ring" -s ${SKIP:-6} -c 1 \
    -o gpurun_out/prof_${mode}_${1:-cur} python bench.py --steps 3 --warmup 5 --no-cpu-baseline --e2e-steps 2 --dh-mode $mode \
    > gpurun_out/ncu_${mode}.log 2>&1; tail -1 gpurun_out/ncu_${mode}.log
done
