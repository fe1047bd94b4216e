"""Predict (fused forward + top-K) throughput vs batch size at Amazon-670K: ms per batch,
samples/s and the fraction of the h-line gather floor (128 B per connection and 32-sample
line at the measured 19.9 TB/s gather ceiling).  B <= 96: k_predict_reg (per 32-sample line); B > 96:
k_predict_wide (FF_FLAG_NO_PIPE: the generic k_predict, for comparison).
Usage: python tools/pred_sweep.py [--no-pipe] [B ...]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2306_03725_b200 import synth
from paper_2306_03725_b200.layer import FixedFanInLayer, LayerConfig, FF_FLAG_NO_PIPE

shape = synth.SHAPES["amazon-670k"]
flags = FF_FLAG_NO_PIPE if "--no-pipe" in sys.argv else 0
lay = FixedFanInLayer(LayerConfig(L_global=shape.L, m=shape.m, k=shape.k, max_batch=1024, seed=42, flags=flags))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
Bs = [int(a) for a in sys.argv[1:] if a.isdigit()] or [16, 32, 33, 64, 128, 256, 512, 1024]
for B in Bs:
    h = torch.from_numpy(synth.hidden_batch(B, shape.m, step=5)).cuda()
    lay.predict_topk(h, 5)
    reps = max(3, 2048 // B)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        lay.predict_topk(h, 5)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    floor = 128.0 * shape.L * shape.k * ((B + 31) // 32) / 19.9e12 * 1e3
    print(f"B={B:5d} ms/batch {ms:8.4f} samples/s {B / ms * 1e3:10.0f} gather floor {floor:7.4f} ms frac {floor / ms:.3f}",
          flush=True)
