"""tcgen05 dense forward vs the FP32 SIMT kernel at growing m (1 and 2 CTAs per SM) and d
(raw-ring wrap): max |diff| and the count above a crude 1e-4 relative bound (near-zero h
values make that count non-zero even when the kernels agree to ~5e-6)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2306_03725_b200 import synth
from paper_2306_03725_b200 import layer as L
for m in (4096, 16384, 32768):
    for d in (512, 64):
        a = L.DenseLayer(L.DenseConfig(d=d, m=m, max_batch=32, seed=43, dropout=0.0), device="cuda")
        b = L.DenseLayer(L.DenseConfig(d=d, m=m, max_batch=32, seed=43, dropout=0.0, flags=L.FF_FLAG_DENSE_SIMT), device="cuda")
        x = torch.from_numpy(synth.feature_batch(32, d, step=3)).cuda()
        ha = a.forward(x, step=3, train=False); hb = b.forward(x, step=3, train=False)
        torch.cuda.synchronize()
        diff = (ha - hb).abs()
        bad = (diff > 1e-4 * (hb.abs() + 1e-3)).nonzero()
        print(m, d, float(diff.max()), len(bad), bad[:5].tolist() if len(bad) else "", flush=True)
