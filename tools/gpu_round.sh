# parity + quick bench (both dh modes) + one ncu capture per mode of the fused kernel
python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
bash tools/gpu_quick.sh 2>&1 | tail -4
bash tools/gpu_prof.sh ${1:-cur}
