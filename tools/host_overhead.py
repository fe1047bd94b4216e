"""Host-side cost of one training step call (ctypes + argument marshalling + 3 kernel launches),
measured as the enqueue time of 100 steps while the GPU is still busy (no synchronisation), at
the Amazon-670K shape.  Relevant to multi-GPU scaling: at P = 8 a rank's GPU step is ~0.08 ms."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2306_03725_b200 import synth
from paper_2306_03725_b200.layer import FixedFanInLayer, LayerConfig
shape = synth.SHAPES["amazon-670k"]
B = shape.B
lay = FixedFanInLayer(LayerConfig(L_global=shape.L, m=shape.m, k=shape.k, max_batch=B, seed=42))
h = torch.from_numpy(synth.hidden_batch(B, shape.m)).cuda()
p, i = (torch.from_numpy(a).cuda() for a in synth.label_batch(B, shape.L, shape.avg_pos))
dh = torch.empty((B, shape.m), device="cuda"); loss = torch.zeros(1, device="cuda")
for _ in range(5):
    lay.train_step(h, p, i, 1e-3, dh=dh, loss=loss)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(100):
    lay.train_step(h, p, i, 1e-3, dh=dh, loss=loss)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue per step: {(t1 - t0) * 1e4:.1f} us; GPU time per step: {(t2 - t0) * 1e4:.1f} us")
