"""Time the intermediate layer's forward (dropout + tcgen05 3xTF32 GEMM + bias/ReLU) and
backward + Adam at d = 512, m = 32768, B = 32 (the bench's model config): ms per call over
200 calls, CUDA events.  FIXEDFANIN_LIB selects a library variant."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2306_03725_b200 import synth
from paper_2306_03725_b200 import layer as L

d, B = 512, 32
m = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
n = L.DenseLayer(L.DenseConfig(d=d, m=m, max_batch=B, seed=43, dropout=0.1), device="cuda")
x = torch.from_numpy(synth.feature_batch(B, d, step=3)).cuda()
dh = torch.randn(B, m, device="cuda") * 1e-3
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("forward", lambda s: n.forward(x, step=s, train=True)),):
    for s in range(10):
        fn(s)
    torch.cuda.synchronize()
    e0.record()
    for s in range(200):
        fn(s)
    e1.record()
    e1.synchronize()
    print(f"m={m} {name}: {e0.elapsed_time(e1) / 200 * 1e3:.1f} us per call", flush=True)
