"""Cost of the per-launch CUDA-event profiling (fixedfanin_profile_begin) on the device step
time at Amazon-670K: the same 300-step loop with and without it."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2306_03725_b200 import synth
from paper_2306_03725_b200.layer import FixedFanInLayer, LayerConfig
shape = synth.SHAPES["amazon-670k"]
B, N = shape.B, 300
lay = FixedFanInLayer(LayerConfig(L_global=shape.L, m=shape.m, k=shape.k, max_batch=B, seed=42))
hs = [torch.from_numpy(synth.hidden_batch(B, shape.m, step=s)).cuda() for s in range(4)]
lb = [tuple(torch.from_numpy(a).cuda() for a in synth.label_batch(B, shape.L, shape.avg_pos, step=s)) for s in range(4)]
dh = [torch.empty((B, shape.m), device="cuda") for _ in range(2)]; loss = torch.zeros(1, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    for prof in (False, True):
        for s in range(5):
            lay.train_step(hs[s % 4], *lb[s % 4], 1e-3, dh=dh[s & 1], loss=loss)
        torch.cuda.synchronize()
        if prof:
            lay.profile_begin(N * 16)
        e0.record()
        for s in range(N):
            lay.train_step(hs[s % 4], *lb[s % 4], 1e-3, dh=dh[s & 1], loss=loss)
        e1.record()
        torch.cuda.synchronize()
        if prof:
            k_ms, k_n = lay.profile_end()
        print(f"profiling={prof}: {e0.elapsed_time(e1) / N * 1e3:.1f} us/step" + (f" (row kernel {k_ms / k_n * 1e3:.1f} us)" if prof else ""))
