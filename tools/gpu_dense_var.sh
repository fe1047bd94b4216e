# Dense forward variants: kernel durations from ncu (the Python loop is host-bound at ~21 us per call).
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for v in $(ls build/libs/*.so); do for m in 18944 32768; do
  FIXEDFANIN_LIB=$PWD/$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dense_fwd|k_dropout" -s 20 -c 20 --csv python tools/dense_fwd_time.py $m 2>/dev/null > /tmp/n.csv
  python - "$v" "$m" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open('/tmp/n.csv')) if len(r) > 10]
hdr = rows[0]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki].split('(')[0]].append(float(r[vi].replace(',', '')))
print(sys.argv[1], 'm=' + sys.argv[2], {k: round(sum(v) / len(v) / 1e3, 2) for k, v in d.items()}, 'us')
PY
done; done
