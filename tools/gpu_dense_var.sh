# Dense forward / backward kernels: durations from ncu (20 launches each after 20 skipped), per variant and m.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for v in paper_2306_03725_b200/libfixedfanin.so $(ls build/libs/*.so 2>/dev/null); do for m in 18944 32768; do for simt in ""; do
  FIXEDFANIN_LIB=$PWD/$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dense|k_dropout" -s 60 -c 60 --csv python tools/dense_fwd_time.py $m $simt 2>/dev/null > /tmp/n.csv
  python - "$v" "$m" "$simt" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open('/tmp/n.csv')) if len(r) > 10]
hdr = rows[0]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki].split('(')[0].replace('void ', '').replace('ff::', '')].append(float(r[vi].replace(',', '')))
print(sys.argv[1].split('/')[-1], 'm=' + sys.argv[2], sys.argv[3] or 'tc', {k: round(sum(v) / len(v) / 1e3, 2) for k, v in d.items()}, 'us')
PY
done; done; done
