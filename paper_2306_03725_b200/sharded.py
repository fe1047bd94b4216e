"""Label-sharded multi-GPU driver.

One process per GPU.  Rank r owns the contiguous label rows
[floor(r L / P), floor((r+1) L / P)) of W, idx, bias and the Adam state; labels are
independent in the one-vs-all loss and rows are independent in the uniform
format, so the only exchanges are:

  * h replicated from the producer rank  (NCCL broadcast, B*m*4 bytes)
  * dh = sum over shards of the partial dh (NCCL all_reduce, B*m*4 bytes)
  * per-shard top-K -> all_gather -> exact merge (same total order on every shard)

Redistribution is keyed on the global row id, so it needs no collective and the state
is identical for every P.  The per-shard compute is an ``engine`` (default: the CUDA
``FixedFanInLayer``); CPU multi-process tests substitute an oracle-backed engine to
check the partition/collective logic with the gloo backend.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(L: int, rank: int, world: int):
    """Contiguous row range [begin, end) of `rank` among `world` shards."""
    return L * rank // world, L * (rank + 1) // world


class ShardedLayer:
    def __init__(self, L_global: int, m: int, k: int, rank: int = 0, world: int = 1, group=None,
                 engine=None, merge_fn=None, device=None, **cfg):
        self.L_global, self.m, self.k = L_global, m, k
        self.rank, self.world, self.group = rank, world, group
        self.row_begin, self.row_end = shard_rows(L_global, rank, world)
        if engine is None:
            from .layer import FixedFanInLayer, LayerConfig
            engine = FixedFanInLayer(LayerConfig(L_global=L_global, m=m, k=k, row_begin=self.row_begin,
                                                 L_local=self.row_end - self.row_begin, **cfg), device=device)
        self.engine = engine
        if merge_fn is None:
            from .layer import merge_topk
            merge_fn = merge_topk
        self.merge_fn = merge_fn

    def broadcast_h(self, h: torch.Tensor, src: int = 0) -> torch.Tensor:
        if self.world > 1:
            dist.broadcast(h, src=src, group=self.group)
        return h

    def train_step(self, h, lbl_ptr, lbl_ids, lr, grad_scale=None, dh=None, loss=None, reduce_loss=False,
                   reduce_dh=True):
        """Fused step on this shard, then dh all-reduce (reduce_dh=False: return this shard's
        partial dh, for a caller that reduce-scatters it).  Returns (dh, loss)."""
        dh, loss = self.engine.train_step(h, lbl_ptr, lbl_ids, lr, grad_scale=grad_scale, dh=dh, loss=loss)
        if self.world > 1:
            if reduce_dh:
                dist.all_reduce(dh, op=dist.ReduceOp.SUM, group=self.group)
            if reduce_loss and loss is not None:
                dist.all_reduce(loss, op=dist.ReduceOp.SUM, group=self.group)
        return dh, loss

    def redistribute(self, step: int):
        self.engine.redistribute(step)

    def predict_topk(self, h, K: int):
        s, i = self.engine.predict_topk(h, K)
        if self.world == 1:
            return s, i
        ss = [torch.empty_like(s) for _ in range(self.world)]
        ii = [torch.empty_like(i) for _ in range(self.world)]
        dist.all_gather(ss, s, group=self.group)
        dist.all_gather(ii, i, group=self.group)
        return self.merge_fn(torch.stack(ss), torch.stack(ii))


class OverlappedTrainer:
    """Training loop helper that overlaps the per-step collectives with compute (P > 1):

    * the h broadcast for step s+1 is issued (async) before step s computes;
    * the dh all-reduce of step s runs (async) while step s+1 computes, into one of two
      dh buffers, which is waited on before that buffer is overwritten two steps later.

    ``step(i_cur, i_next)`` runs one step on batch slot ``i_cur`` of the caller's device
    buffers ``h[i]``/``ptr[i]``/``ids[i]`` and prefetches slot ``i_next``; ``finish()`` waits
    for every outstanding collective.  ``dh(s)`` is step s's reduced dh once ``finish()`` (or
    the step two later) has run.  With P = 1 it degenerates to plain ``train_step`` calls.
    """

    def __init__(self, layer: ShardedLayer, h, ptr, ids, lr, B, m, device, loss=None):
        self.layer, self.h, self.ptr, self.ids, self.lr = layer, h, ptr, ids, lr
        self.dh = [torch.empty((B, m), device=device) for _ in range(2)]
        self.loss = loss
        self.bcast = [None] * len(h)
        self.ar = [None, None]
        self.s = 0

    def prefetch(self, i):
        if self.layer.world > 1 and self.bcast[i] is None:
            self.bcast[i] = dist.broadcast(self.h[i], src=0, group=self.layer.group, async_op=True)

    def step(self, i_cur, i_next):
        L = self.layer
        if self.bcast[i_cur] is not None:
            self.bcast[i_cur].wait()
            self.bcast[i_cur] = None
        elif L.world > 1:
            dist.broadcast(self.h[i_cur], src=0, group=L.group)
        if i_next is not None:                          # None: the caller fills the next slot itself
            self.prefetch(i_next)
        slot = self.s & 1
        if self.ar[slot] is not None:
            self.ar[slot].wait()
            self.ar[slot] = None
        L.engine.train_step(self.h[i_cur], self.ptr[i_cur], self.ids[i_cur], self.lr, dh=self.dh[slot], loss=self.loss)
        if L.world > 1:
            self.ar[slot] = dist.all_reduce(self.dh[slot], op=dist.ReduceOp.SUM, group=L.group, async_op=True)
        self.s += 1
        return self.dh[slot]

    def finish(self):
        for k in range(2):
            if self.ar[k] is not None:
                self.ar[k].wait()
                self.ar[k] = None
        for i in range(len(self.bcast)):
            if self.bcast[i] is not None:
                self.bcast[i].wait()
                self.bcast[i] = None


class GraphedSteps:
    """K consecutive label-sharded training steps, collectives included, captured once in one
    CUDA graph and replayed: per step j the h broadcast of slot j, the shard's
    fused step (fixedfanin_train_step) into dh[j], and the async dh all-reduce of dh[j], which
    overlaps the compute of step j + 1 inside the graph (NCCL's stream forks from and joins the
    capture stream); the graph joins every all-reduce at its end.  One graph launch replaces
    K x (broadcast + 3 kernels + all-reduce) host enqueues.

    The caller owns the K static input slots h[j] [B][m], ptr[j] and ids[j] (fixed capacity)
    and refills them between replays; the learning rate is baked in at capture, the Adam step
    counter lives on the device and advances per replayed step.  Construction runs the K steps
    once eagerly (NCCL communicator set-up and lazy allocations must happen outside the
    capture), so it trains K steps.  NCCL collectives are graph-capturable, gloo's are not:
    ``collectives`` defaults to world > 1 and needs the NCCL backend; True with one rank
    exercises the capture path on one GPU."""

    def __init__(self, layer: "ShardedLayer", h, ptr, ids, lr, B, m, device, loss=None, collectives=None):
        self.layer, self.h, self.ptr, self.ids, self.lr, self.loss = layer, h, ptr, ids, lr, loss
        self.K = len(h)
        self.dh = [torch.empty((B, m), device=device) for _ in range(self.K)]
        self.collectives = layer.world > 1 if collectives is None else collectives
        self.stream = torch.cuda.Stream(device=device)
        self.stream.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.stream(self.stream):
            self._steps()                                     # eager pass: communicators, allocations
        torch.cuda.current_stream(device).wait_stream(self.stream)
        torch.cuda.synchronize(device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self._steps()

    def _steps(self):
        L, works = self.layer, []
        for j in range(self.K):
            if self.collectives:
                dist.broadcast(self.h[j], src=0, group=L.group)
            L.engine.train_step(self.h[j], self.ptr[j], self.ids[j], self.lr, dh=self.dh[j], loss=self.loss)
            if self.collectives:
                works.append(dist.all_reduce(self.dh[j], op=dist.ReduceOp.SUM, group=L.group, async_op=True))
        for w in works:
            w.wait()

    def replay(self):
        """Run the K captured steps (on the current stream's device; ordered after prior work)."""
        self.graph.replay()


class ShardedModel:
    """The whole proposed architecture (Fig. 2) under label sharding (NEXT-2,
    SURVEY §8(f)2): rank r owns one label shard of the fixed fan-in layer AND the column shard
    [m r / P, m (r+1) / P) of the dense intermediate layer (Wd, bd and their Adam state), so
    the dense layer's bytes per rank fall as 1/P like the sparse layer's.

    Per step (x replicated, broadcast from rank 0):
      1. dropout + dense forward of this rank's columns: h_r = ReLU(dropout(x) Wd[:, cols] + bd)
         — the dropout mask is keyed on (seed, step, sample, feature) (R25), identical on
         every rank;
      2. all_gather of the column shards -> the full h [B][m];
      3. the label shard's fused step -> this shard's partial dh [B][m];
      4. reduce_scatter of the partial dh -> dh[:, cols] summed over the label shards;
      5. dense backward + Adam of this rank's columns (dWd[:, cols] = xt^T (dh_r [h_r > 0])).
    Bytes on the wire per step: 4 B m (P-1)/P for each of the all-gather and the
    reduce-scatter (the same as the dh all-reduce they replace)."""

    def __init__(self, layer: ShardedLayer, dense=None, d: int | None = None, device=None, **dense_cfg):
        self.layer = layer
        m, P, r = layer.m, layer.world, layer.rank
        self.cols = [shard_rows(m, q, P) for q in range(P)]
        self.col_begin, self.col_end = self.cols[r]
        self.mc = max(e - b for b, e in self.cols)            # padded shard width of the collectives
        if dense is None:
            from .layer import DenseConfig, DenseLayer
            dense = DenseLayer(DenseConfig(d=d, m=self.col_end - self.col_begin, col_begin=self.col_begin,
                                           m_global=m, **dense_cfg), device=device)
        self.dense = dense

    def broadcast_x(self, x: torch.Tensor, src: int = 0) -> torch.Tensor:
        if self.layer.world > 1:
            dist.broadcast(x, src=src, group=self.layer.group)
        return x

    def gather_h(self, h_r: torch.Tensor) -> torch.Tensor:
        """[B][m_r] column shards of every rank -> the full h [B][m] (all_gather)."""
        L = self.layer
        if L.world == 1:
            return h_r
        B, mr = h_r.shape
        send = h_r
        if mr < self.mc:
            send = torch.zeros((B, self.mc), dtype=h_r.dtype, device=h_r.device)
            send[:, :mr] = h_r
        out = torch.empty((L.world * B, self.mc), dtype=h_r.dtype, device=h_r.device)
        dist.all_gather_into_tensor(out, send.contiguous(), group=L.group)
        out = out.view(L.world, B, self.mc)
        return torch.cat([out[q, :, :e - b] for q, (b, e) in enumerate(self.cols)], dim=1)

    def scatter_dh(self, dh: torch.Tensor) -> torch.Tensor:
        """This label shard's partial dh [B][m] -> dh[:, own columns] summed over the label
        shards (reduce_scatter)."""
        L = self.layer
        if L.world == 1:
            return dh
        B = dh.shape[0]
        inp = torch.zeros((L.world, B, self.mc), dtype=dh.dtype, device=dh.device)
        for q, (b, e) in enumerate(self.cols):
            inp[q, :, :e - b] = dh[:, b:e]
        out = torch.empty((B, self.mc), dtype=dh.dtype, device=dh.device)
        dist.reduce_scatter_tensor(out, inp.view(L.world * B, self.mc), op=dist.ReduceOp.SUM, group=L.group)
        return out[:, :self.col_end - self.col_begin].contiguous()

    def train_step(self, x, step, lbl_ptr, lbl_ids, lr, grad_scale=None, loss=None, reduce_loss=False):
        """One step (1-5 above).  Returns (dh of this rank's columns, loss)."""
        h = self.gather_h(self.dense.forward(x, step=step, train=True))
        dh, loss = self.layer.train_step(h, lbl_ptr, lbl_ids, lr, grad_scale=grad_scale, loss=loss,
                                         reduce_loss=reduce_loss, reduce_dh=False)
        dh_r = self.scatter_dh(dh)
        self.dense.backward_adam(dh_r, lr)
        return dh_r, loss

    def predict_topk(self, x, K: int):
        return self.layer.predict_topk(self.gather_h(self.dense.forward(x, train=False)), K)
