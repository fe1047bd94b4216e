python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for sh in tiny wiki10-31k wiki-500k amazon-670k amazon-670k-m16k amazon-670k-k64-m65k amazon-3m; do
  timeout 600 python bench.py --shape $sh --steps 500 --warmup 10 --e2e-steps 100 --no-cpu-baseline > gpurun_out/sh_$sh.json 2>gpurun_out/sh.err
  python -c "
import json; d=json.load(open('gpurun_out/sh_$sh.json')); r=d['roofline']; m=d.get('model') or {}
g=d.get('cuda_graph') or {}; rd=d.get('redistribution') or {}
print('%-22s %9d %8.4f %6.3f %6.3f %9d %9d %9d %6d %9d %7.3f' % ('$sh', d['value'], d['ms_per_step'], r['frac'], d['hbm_step']['frac'], d['e2e']['value'], d['predict']['value'], m.get('value', 0), d['memory']['workspace_bytes_per_gpu']/1e6, g.get('samples_per_s', 0), rd.get('ms_per_call', 0)))" || tail -3 gpurun_out/sh.err
done
