"""Long-run stability check (round 1): N training steps at Amazon-670K (B = 32, atomic and CSC
dh) with the SET redistribution every 1000 steps, then the redistribution invariants on the
GPU state (every row keeps k distinct in-range indices) and finite loss / parameters.
Prints one line per mode."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2306_03725_b200 import synth
from paper_2306_03725_b200.layer import FixedFanInLayer, LayerConfig, FF_DH_ATOMIC, FF_DH_CSC

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
shape = synth.SHAPES["amazon-670k"]
B = shape.B
data = [(torch.from_numpy(synth.hidden_batch(B, shape.m, step=s)).cuda(),
         *(torch.from_numpy(a).cuda() for a in synth.label_batch(B, shape.L, shape.avg_pos, step=s))) for s in range(8)]
for mode, name in ((FF_DH_ATOMIC, "atomic"), (FF_DH_CSC, "csc")):
    lay = FixedFanInLayer(LayerConfig(L_global=shape.L, m=shape.m, k=shape.k, max_batch=B, seed=42, dh_mode=mode))
    loss = torch.zeros(1, device="cuda")
    losses = []
    torch.cuda.synchronize(); t0 = time.time()
    for s in range(steps):
        h, p, i = data[s % 8]
        lay.train_step(h, p, i, 1e-3, loss=loss)
        if (s + 1) % 1000 == 0:
            lay.redistribute(s + 1)
            losses.append(float(loss.item()))
    torch.cuda.synchronize(); dt = time.time() - t0
    st = lay.get_params()
    idx = st["idx"]
    srt = torch.sort(idx, dim=1).values
    distinct = bool((srt[:, 1:] != srt[:, :-1]).all().item())
    in_range = bool(((idx >= 0) & (idx < shape.m)).all().item())
    finite = all(bool(torch.isfinite(st[k]).all().item()) for k in ("W", "bias", "mW", "vW"))
    print(f"{name}: {steps} steps ({steps // 1000} redistributions) in {dt:.2f} s wall = {B * steps / dt:.0f} samples/s; "
          f"rows with k distinct in-range indices: {distinct and in_range}; finite state: {finite}; "
          f"device Adam t = {st['t']} (expected {steps}); "
          f"loss at each redistribution: {[round(x, 2) for x in losses]}")
