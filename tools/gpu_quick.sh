python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for mode in csc; do
  timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --e2e-steps 50 --dh-mode $mode > gpurun_out/q_$mode.json 2>gpurun_out/q_$mode.err
  python -c "import json; d=json.load(open('gpurun_out/q_$mode.json')); print('$mode', round(d['value']), 'ms/step', round(d['ms_per_step'],4), 'row_ms', round(d['roofline']['avg_launch_ms'],4), 'pred', round(d['predict']['value']))" || tail -5 gpurun_out/q_$mode.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -s 80 -c 30 --csv --log-file gpurun_out/launches_csc.csv python bench.py --steps 20 --warmup 20 --no-cpu-baseline --e2e-steps 3 --dh-mode csc > /dev/null 2>&1
python - <<'PY'
import csv
from collections import defaultdict
rows=[r for r in csv.reader(open('gpurun_out/launches_csc.csv')) if len(r)>5]
h=rows[0]; ik=h.index('Kernel Name'); im=h.index('Metric Name'); iv=h.index('Metric Value')
d=defaultdict(lambda: defaultdict(list))
for r in rows[1:]: d[r[ik][:30]][r[im]].append(float(r[iv].replace(',','')))
for k,v in d.items(): print(k, {m: round(sum(x)/len(x),1) for m,x in v.items()})
PY
