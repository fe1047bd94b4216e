"""GPU: the label-sharded training steps captured in one CUDA graph WITH their NCCL
collectives (sharded.GraphedSteps), on a one-rank NCCL process group — the
only multi-process configuration one GPU allows.  The replayed graph (h broadcast, fused
step, async dh all-reduce per step, K steps per graph) must leave the layer in exactly the
state that the same steps run eagerly leave, and produce the same dh (up to the atomic
summation order of the dh scatter)."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"])
from paper_2306_03725_b200 import synth
from paper_2306_03725_b200.layer import FF_DH_CSC, FixedFanInLayer, LayerConfig
from paper_2306_03725_b200.sharded import GraphedSteps, ShardedLayer

dist.init_process_group("nccl", init_method="tcp://127.0.0.1:" + os.environ["PORT"], rank=0, world_size=1)
dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
L, m, k, B, K, ROUNDS, lr = 20000, 1024, 32, 32, 3, 3, 1e-3
csc = os.environ["DH"] == "csc"
mk = lambda: FixedFanInLayer(LayerConfig(L_global=L, m=m, k=k, max_batch=B, seed=7, dh_mode=FF_DH_CSC if csc else 0),
                             device=dev)
a, b = mk(), mk()
h = [torch.from_numpy(synth.hidden_batch(B, m, step=j)).to(dev) for j in range(K)]
lab = [synth.label_batch(B, L, 5.0, step=j) for j in range(K)]
ptr = [torch.from_numpy(p).to(dev) for p, _ in lab]
ids = [torch.from_numpy(i).to(dev) for _, i in lab]
loss_a, loss_b = torch.zeros(1, device=dev), torch.zeros(1, device=dev)
g = GraphedSteps(ShardedLayer(L, m, k, rank=0, world=1, group=dist.group.WORLD, engine=a), h, ptr, ids, lr, B, m,
                 dev, loss=loss_a, collectives=True)            # trains round 0 eagerly, then captures
for _ in range(ROUNDS - 1):
    g.replay()
dh_b = [torch.empty((B, m), device=dev) for _ in range(K)]
for _ in range(ROUNDS):
    for j in range(K):
        b.train_step(h[j], ptr[j], ids[j], lr, dh=dh_b[j], loss=loss_b)
torch.cuda.synchronize()
pa, pb = a.get_params(), b.get_params()
for key in ("W", "idx", "bias", "mW", "vW", "mb", "vb"):
    assert torch.equal(pa[key], pb[key]), key
assert pa["t"] == pb["t"] == ROUNDS * K, (pa["t"], pb["t"])
for j in range(K):
    if csc:                                          # the CSC pull sums in a fixed order: bit-identical
        assert torch.equal(g.dh[j], dh_b[j]), j
    d = (g.dh[j] - dh_b[j]).abs().max().item()
    assert d <= 1e-5 * dh_b[j].abs().max().item(), (j, d)
assert torch.equal(loss_a, loss_b) or abs(loss_a.item() - loss_b.item()) <= 1e-5 * abs(loss_b.item())
dist.destroy_process_group()
print("GRAPH_NCCL_OK")
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("dh", ["atomic", "csc"])
def test_graphed_sharded_steps_with_nccl_match_eager(dh):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__ as g
    g.build_lib()
    env = dict(os.environ, ROOT=ROOT, PORT=str(_free_port()), MASTER_ADDR="127.0.0.1", DH=dh)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "GRAPH_NCCL_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
