# per-kernel durations (ncu launch list) of the working tree vs build/libs/base.so
for lib in paper_2306_03725_b200/libfixedfanin.so build/libs/base.so; do
  n=$(basename $lib .so)
  FIXEDFANIN_LIB=$PWD/$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${AB_KERNELS:-k_prep|k_dh_out}" -c 30 --csv \
    --log-file gpurun_out/ab3_$n.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
  python - "$n" <<'PY'
import csv,sys,collections
n=sys.argv[1]
rows=[r for r in csv.reader(open(f"gpurun_out/ab3_{n}.csv")) if len(r)>10]
h=rows[0]; k=h.index('Kernel Name'); v=h.index('Metric Value')
d=collections.defaultdict(list)
for r in rows[1:]:
  try: d[r[k][:40]].append(float(r[v].replace(',','')))
  except: pass
print(n, {a: (round(sum(x)/len(x),2), len(x)) for a,x in d.items()})
PY
done
