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

    def train_step(self, h, lbl_ptr, lbl_ids, lr, grad_scale=None, dh=None, loss=None, reduce_loss=False):
        """Fused step on this shard, then dh all-reduce.  Returns (dh, loss)."""
        dh, loss = self.engine.train_step(h, lbl_ptr, lbl_ids, lr, grad_scale=grad_scale, dh=dh, loss=loss)
        if self.world > 1:
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


class ShardedModel:
    """The whole proposed architecture (Fig. 2) under label sharding (NEXT-2):
    every rank holds a replica of the dense intermediate layer (``dense``: the CUDA
    ``DenseLayer`` by default) and one label shard of the fixed fan-in layer.

    Per step: the features x (replicated; broadcast from rank 0) go through the replica's
    dropout + dense forward — identical on every rank, because the dropout mask is keyed on
    (seed, step, sample) (reading R25) — the shard's fused step yields its partial dh, the
    dh all-reduce sums the shards, and every replica applies the same dense backward + Adam
    to the same summed dh, so the replicas stay identical without another collective."""

    def __init__(self, layer: ShardedLayer, dense=None, d: int | None = None, device=None, **dense_cfg):
        self.layer = layer
        if dense is None:
            from .layer import DenseConfig, DenseLayer
            dense = DenseLayer(DenseConfig(d=d, m=layer.m, **dense_cfg), device=device)
        self.dense = dense

    def broadcast_x(self, x: torch.Tensor, src: int = 0) -> torch.Tensor:
        if self.layer.world > 1:
            dist.broadcast(x, src=src, group=self.layer.group)
        return x

    def train_step(self, x, step, lbl_ptr, lbl_ids, lr, grad_scale=None, dh=None, loss=None, reduce_loss=False):
        h = self.dense.forward(x, step=step, train=True)
        dh, loss = self.layer.train_step(h, lbl_ptr, lbl_ids, lr, grad_scale=grad_scale, dh=dh, loss=loss,
                                         reduce_loss=reduce_loss)
        self.dense.backward_adam(dh, lr)
        return dh, loss

    def predict_topk(self, x, K: int):
        return self.layer.predict_topk(self.dense.forward(x, train=False), K)
