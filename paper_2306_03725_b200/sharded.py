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
