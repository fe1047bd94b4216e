"""Run the intermediate layer's forward (dropout + dense GEMM + bias/ReLU) and backward + Adam
at d = 512, B = 32 (the bench's model config) for a given m, 200 times: a target for ncu
(`gpu__time_duration` per kernel; tools/gpu_dense_var.sh) — the Python loop itself is
host-bound (~21 us per call), so its event time is not the kernels'.  Usage: m [simt]."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2306_03725_b200 import synth
from paper_2306_03725_b200 import layer as L

d, B = 512, 32
m = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
flags = L.FF_FLAG_DENSE_SIMT if "simt" in sys.argv else 0
n = L.DenseLayer(L.DenseConfig(d=d, m=m, max_batch=B, seed=43, dropout=0.1, flags=flags), device="cuda")
x = torch.from_numpy(synth.feature_batch(B, d, step=3)).cuda()
dh = torch.randn(B, m, device="cuda") * 1e-3
for s in range(200):
    n.forward(x, step=s + 1, train=True)
    n.backward_adam(dh, 1e-3)
torch.cuda.synchronize()
print(f"m={m} done", flush=True)
# CUDA-graph replay of 50 forwards (no host cost between launches): dropout + forward per call
s = torch.cuda.Stream()
h = torch.empty(B, m, device="cuda")
with torch.cuda.stream(s):
    n.forward(x, step=1, train=True, h=h)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(50):
            n.forward(x, step=1, train=True, h=h)
    g.replay(); g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        g.replay()
    e1.record(s)
    e1.synchronize()
print(f"m={m} graph-timed forward (dropout + dense): {e0.elapsed_time(e1) / 500 * 1e3:.2f} us per call", flush=True)
# the same for forward + backward/Adam (the backward alone = the difference)
with torch.cuda.stream(s):
    n.forward(x, step=1, train=True, h=h); n.backward_adam(dh, 1e-3)
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=s):
        for i in range(50):
            n.forward(x, step=1, train=True, h=h)
            n.backward_adam(dh, 1e-3)
    g2.replay(); g2.replay()
    e0.record(s)
    for _ in range(10):
        g2.replay()
    e1.record(s)
    e1.synchronize()
fb = e0.elapsed_time(e1) / 500 * 1e3
print(f"m={m} graph-timed forward + backward/Adam: {fb:.2f} us per call", flush=True)
