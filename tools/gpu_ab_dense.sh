set -u
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -q -m gpu -x -k "dense or model or smoke" 2>&1 | tail -3
AB_KERNELS="k_dense_fwd_tc|k_dropout" bash tools/gpu_ab3.sh
for i in 1 2; do for lib in paper_2306_03725_b200/libfixedfanin.so build/libs/base.so; do FIXEDFANIN_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --steps 300 --e2e-steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['model']; print('$lib', m['ms_per_step'], m['dense_fwd']['ms'], m['dense_fwd']['frac'])"; done; done
