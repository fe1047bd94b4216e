"""Single-GPU probes of the label-sharded step (no multi-GPU box this round):

1. shard step time: one rank's step at P = 1, 2, 4, 8 (L_local = L/P rows of Amazon-670K and of
   Amazon-3M, global label ids), eager and replayed from a CUDA graph, i.e. the compute a rank
   does per step under label sharding;
2. contention: the P = 8 shard's eager step with a concurrent stream that moves the traffic of
   the step's two collectives (h broadcast + dh all-reduce, 4.2 MB each: a copy and a
   read-modify-write of dh per step), to bound what overlapping them costs the row kernel.
CUDA events on the launching stream, 500 steps after 20 warm-up."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2306_03725_b200 import synth
from paper_2306_03725_b200.layer import FixedFanInLayer, LayerConfig

N, W = 500, 20
dev = torch.device("cuda")
for name in ("amazon-670k", "amazon-3m"):
    sh = synth.SHAPES[name]
    B, m = sh.B, sh.m
    hs = [torch.from_numpy(synth.hidden_batch(B, m, step=s)).to(dev) for s in range(4)]
    lb = [synth.label_batch(B, sh.L, sh.avg_pos, step=s) for s in range(4)]
    ps = [torch.from_numpy(a).to(dev) for a, _ in lb]
    ids = [torch.from_numpy(b).to(dev) for _, b in lb]
    dh = torch.empty((B, m), device=dev)
    for P in (1, 2, 4, 8):
        Ll = (sh.L + P - 1) // P
        lay = FixedFanInLayer(LayerConfig(L_global=sh.L, m=m, k=sh.k, L_local=Ll, max_batch=B, seed=42), device=dev)
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def run(fn):
            for s in range(W):
                fn(s)
            torch.cuda.synchronize()
            e0.record(st)
            for s in range(N):
                fn(s)
            e1.record(st)
            e1.synchronize()
            return e0.elapsed_time(e1) / N

        eager = run(lambda s: lay.train_step(hs[s % 4], ps[s % 4], ids[s % 4], 1e-3, dh=dh))
        graphs = []
        side = torch.cuda.Stream()
        side.wait_stream(st)
        with torch.cuda.stream(side):
            lay.train_step(hs[0], ps[0], ids[0], 1e-3, dh=dh)
        st.wait_stream(side)
        for i in range(4):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                lay.train_step(hs[i], ps[i], ids[i], 1e-3, dh=dh)
            graphs.append(g)
        graph = run(lambda s: graphs[s % 4].replay())
        line = f"{name:12s} P={P} L_local={Ll:8d} eager {eager * 1e3:7.1f} us  graph {graph * 1e3:7.1f} us"
        if P == 8:
            comm = torch.cuda.Stream()
            hb, acc = torch.empty_like(hs[0]), torch.zeros_like(dh)

            def with_traffic(s):
                lay.train_step(hs[s % 4], ps[s % 4], ids[s % 4], 1e-3, dh=dh)
                ev = torch.cuda.Event()
                ev.record(st)
                with torch.cuda.stream(comm):
                    comm.wait_event(ev)
                    hb.copy_(hs[(s + 1) % 4])          # the next step's h broadcast
                    acc.add_(dh)                       # the dh all-reduce's read-modify-write
            cont = run(with_traffic)
            torch.cuda.synchronize()
            line += f"  eager + concurrent collective traffic {cont * 1e3:7.1f} us"
        print(line, flush=True)
        del lay, graphs
