"""Where the end-to-end step loses time against the device-resident step (Amazon-670K, B = 32):
device path (inputs resident), host entry point with / without the loss D2H, with a single
staging slot's worth of data reused.  CUDA events on the default stream; 300 steps each."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2306_03725_b200 import synth
from paper_2306_03725_b200.layer import FixedFanInLayer, LayerConfig
shape = synth.SHAPES["amazon-670k"]
B, N = shape.B, 300
lay = FixedFanInLayer(LayerConfig(L_global=shape.L, m=shape.m, k=shape.k, max_batch=B, seed=42))
hs = [torch.from_numpy(synth.hidden_batch(B, shape.m, step=s)).pin_memory() for s in range(4)]
lbl = [synth.label_batch(B, shape.L, shape.avg_pos, step=s) for s in range(4)]
ps = [torch.from_numpy(a[0]).pin_memory() for a in lbl]
ids = [torch.from_numpy(a[1]).pin_memory() for a in lbl]
hd = [h.cuda() for h in hs]; pd = [p.cuda() for p in ps]; idd = [i.cuda() for i in ids]
dh = torch.empty((B, shape.m), device="cuda"); loss = torch.zeros(1, device="cuda")
loss_pin = torch.zeros(1).pin_memory()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def run(name, fn):
    for s in range(10):
        fn(s)
    torch.cuda.synchronize()
    e0.record()
    for s in range(N):
        fn(s)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:40s} {e0.elapsed_time(e1) / N * 1e3:8.1f} us/step")


for rep in range(2):
    run("device (resident inputs, loss on device)", lambda s: lay.train_step(hd[s % 4], pd[s % 4], idd[s % 4], 1e-3, dh=dh, loss=loss))
    run("device + loss D2H on the stream", lambda s: (lay.train_step(hd[s % 4], pd[s % 4], idd[s % 4], 1e-3, dh=dh, loss=loss),
                                                      loss_pin.copy_(loss, non_blocking=True)))
    run("host entry, no loss", lambda s: lay.train_step_host(hs[s % 4], ps[s % 4], ids[s % 4], 1e-3))
    run("host entry, loss D2H", lambda s: lay.train_step_host(hs[s % 4], ps[s % 4], ids[s % 4], 1e-3, loss_host=loss_pin))
