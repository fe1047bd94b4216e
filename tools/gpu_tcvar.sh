# dense tcgen05 forward variants: correctness at the full shape (vs the SIMT kernel) and the
# kernel time from an ncu launch list, per library in build/var plus the HEAD build.
for lib in build/var/*.so build/libs/base.so; do
  n=$(basename $lib .so)
  FIXEDFANIN_LIB=$PWD/$lib python tools/dense_fwd_check.py | sed "s/^/$n /"
  FIXEDFANIN_LIB=$PWD/$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dense_fwd_tc" -c 12 --csv \
    --log-file gpurun_out/tcv_$n.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
  python - "$n" <<'PY'
import csv,sys
n=sys.argv[1]
rows=[r for r in csv.reader(open(f"gpurun_out/tcv_{n}.csv")) if len(r)>10]
h=rows[0]; v=h.index('Metric Value')
x=[float(r[v].replace(',','')) for r in rows[1:]]
print(n, 'k_dense_fwd_tc us', round(sum(x)/len(x)/1000,2), len(x))
PY
done
