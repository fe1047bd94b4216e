# A/B of the working tree against build/libs/base.so: GPU tests (subset), then per-kernel
# times from an ncu launch list of each library and the bench step / e2e.
set -u
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -q -m gpu -x -k "${AB_TESTS:-parity}" 2>&1 | tail -2
for lib in paper_2306_03725_b200/libfixedfanin.so build/libs/base.so; do
  n=$(basename $lib .so)
  FIXEDFANIN_LIB=$PWD/$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_prep|k_dh_out|k_train_ring" -c 30 --csv \
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "
import csv,sys,collections
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; k=h.index('Kernel Name'); v=h.index('Metric Value')
d=collections.defaultdict(list)
for r in rows[1:]:
  try: d[r[k][:30]].append(float(r[v].replace(',','')))
  except: pass
print('$n', {a: round(sum(x)/len(x),2) for a,x in d.items()})"
done
for i in 1 2; do for lib in paper_2306_03725_b200/libfixedfanin.so build/libs/base.so; do FIXEDFANIN_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --steps 500 --e2e-steps 500 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['ms_per_step'], d['e2e']['ms_per_step'], d['model']['ms_per_step'])"; done; done
