"""Multi-process (world size 2, gloo, CPU) test of the label-sharded driver's partition and
collective logic (paper_2306_03725_b200/sharded.py).

The per-shard compute is an oracle-backed engine (tests may use the oracle); the driver's
own code paths — row partition, h broadcast, dh all-reduce, top-K all-gather + merge,
collective-free redistribution keyed on global rows — are exercised as in production and
compared with the single-process, unsharded oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2306_03725_b200 import synth
from paper_2306_03725_b200.sharded import ShardedLayer, shard_rows

L, M, K_FAN, B, SEED = 203, 40, 8, 6, 17


class OracleEngine:
    """CPU stand-in for FixedFanInLayer on one shard (same method signatures)."""

    def __init__(self, L_global, m, k, row_begin, row_end, seed):
        self.row_begin = row_begin
        self.m = m
        self.st = oracle.State.create(row_end - row_begin, m, k, seed, row_begin=row_begin)

    def train_step(self, h, lbl_ptr, lbl_ids, lr, grad_scale=None, dh=None, loss=None):
        gs = 1.0 / h.shape[0] if grad_scale is None else grad_scale
        r = oracle.train_step(self.st, h.numpy(), lbl_ptr.numpy(), lbl_ids.numpy(), gs, lr, row_begin=self.row_begin)
        out = torch.from_numpy(r.dh.copy())
        if dh is not None:
            dh.copy_(out)
            out = dh
        lt = torch.tensor([r.loss], dtype=torch.float64)
        if loss is not None:
            loss.copy_(lt)
            lt = loss
        return out, lt

    def predict_topk(self, h, K):
        y, _ = oracle.forward(self.st.W, self.st.idx, self.st.bias, h.numpy())
        s, i = oracle.topk(y, K, row_begin=self.row_begin)
        return torch.from_numpy(s), torch.from_numpy(i)

    def redistribute(self, step):
        p = int(np.floor(np.float32(0.25) * K_FAN))
        st = self.st
        st.W, st.idx, st.mW, st.vW = oracle.redistribute(st.W, st.idx, st.mW, st.vW, self.m, p, SEED, step,
                                                         row_begin=self.row_begin)


def cpu_merge(scores, ids):
    """Exact merge of per-shard lists [P][B][K] under (score desc, id asc)."""
    P, Bn, K = scores.shape
    out_s = torch.empty((Bn, K), dtype=scores.dtype)
    out_i = torch.empty((Bn, K), dtype=ids.dtype)
    for b in range(Bn):
        s = scores[:, b, :].reshape(-1).numpy()
        i = ids[:, b, :].reshape(-1).numpy()
        order = np.lexsort((i, -s))[:K]
        out_s[b] = torch.from_numpy(s[order])
        out_i[b] = torch.from_numpy(i[order])
    return out_s, out_i


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rb, re_ = shard_rows(L, rank, world)
        eng = OracleEngine(L, M, K_FAN, rb, re_, SEED)
        lay = ShardedLayer(L, M, K_FAN, rank=rank, world=world, engine=eng, merge_fn=cpu_merge)
        out = {}
        for step in range(2):
            # only rank 0 holds the real batch: the driver must broadcast it
            h = torch.from_numpy(synth.hidden_batch(B, M, step=step).astype(np.float64))
            if rank != 0:
                h = torch.zeros_like(h)
            lay.broadcast_h(h)
            ptr, ids = synth.label_batch(B, L, 3.0, step=step)
            dh, loss = lay.train_step(h, torch.from_numpy(ptr), torch.from_numpy(ids), 1e-2, reduce_loss=True,
                                      loss=torch.zeros(1, dtype=torch.float64))
            out[f"dh{step}"] = dh.numpy().copy()
            out[f"loss{step}"] = float(loss.item())
        lay.redistribute(1000)
        h = torch.from_numpy(synth.hidden_batch(B, M, step=9).astype(np.float64))
        s, i = lay.predict_topk(h, 5)
        out["top_s"], out["top_i"] = s.numpy(), i.numpy()
        out["W"], out["idx"] = eng.st.W, eng.st.idx
        out["rows"] = (rb, re_)
        results[rank] = out
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_rows_partition():
    for world in (1, 2, 3, 8):
        bounds = [shard_rows(1000003, r, world) for r in range(world)]
        assert bounds[0][0] == 0 and bounds[-1][1] == 1000003
        assert all(bounds[r][1] == bounds[r + 1][0] for r in range(world - 1))
        sizes = [e - b for b, e in bounds]
        assert max(sizes) - min(sizes) <= 1


def test_two_rank_gloo_matches_unsharded_oracle():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    # unsharded reference
    st = oracle.State.create(L, M, K_FAN, SEED)
    for step in range(2):
        h = synth.hidden_batch(B, M, step=step).astype(np.float64)
        ptr, ids = synth.label_batch(B, L, 3.0, step=step)
        r = oracle.train_step(st, h, ptr, ids, 1.0 / B, 1e-2)
        for rank in range(world):
            np.testing.assert_allclose(results[rank][f"dh{step}"], r.dh, rtol=1e-12, atol=1e-14)
            assert results[rank][f"loss{step}"] == pytest.approx(r.loss, rel=1e-12)
    p = int(np.floor(np.float32(0.25) * K_FAN))
    st.W, st.idx, st.mW, st.vW = oracle.redistribute(st.W, st.idx, st.mW, st.vW, M, p, SEED, 1000)
    W = np.concatenate([results[r]["W"] for r in range(world)])
    idx = np.concatenate([results[r]["idx"] for r in range(world)])
    assert (idx == st.idx).all()                              # P-invariant redistribution
    np.testing.assert_allclose(W, st.W, rtol=0, atol=0)
    h = synth.hidden_batch(B, M, step=9).astype(np.float64)
    y, _ = oracle.forward(st.W, st.idx, st.bias, h)
    s_ref, i_ref = oracle.topk(y, 5)
    for rank in range(world):
        assert (results[rank]["top_i"] == i_ref).all()
        np.testing.assert_array_equal(results[rank]["top_s"], s_ref)


def _worker_overlap(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2306_03725_b200.sharded import OverlappedTrainer
        rb, re_ = shard_rows(L, rank, world)
        eng = OracleEngine(L, M, K_FAN, rb, re_, SEED)
        lay = ShardedLayer(L, M, K_FAN, rank=rank, world=world, engine=eng, merge_fn=cpu_merge)
        nb = 3
        hs, ptrs, idss = [], [], []
        for s in range(nb):
            h = torch.from_numpy(synth.hidden_batch(B, M, step=s).astype(np.float64))
            if rank != 0:
                h = torch.zeros_like(h)                 # only the producer rank has the data
            p_, i_ = synth.label_batch(B, L, 3.0, step=s)
            hs.append(h); ptrs.append(torch.from_numpy(p_)); idss.append(torch.from_numpy(i_))
        tr = OverlappedTrainer(lay, hs, ptrs, idss, 1e-2, B, M, "cpu")
        tr.dh = [torch.empty((B, M), dtype=torch.float64) for _ in range(2)]
        out = []
        for s in range(nb):
            out.append(tr.step(s, (s + 1) % nb))
        tr.finish()
        results[rank] = [d.numpy().copy() for d in out[-2:]]
    finally:
        dist.destroy_process_group()


def test_overlapped_trainer_two_ranks():
    """Async h broadcast / dh all-reduce pipeline: after finish(), the last two steps' dh
    buffers equal the unsharded oracle's dh of those steps."""
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker_overlap, args=(world, _free_port(), results), nprocs=world, join=True)
    st = oracle.State.create(L, M, K_FAN, SEED)
    ref = []
    for s in range(3):
        h = synth.hidden_batch(B, M, step=s).astype(np.float64)
        ptr, ids = synth.label_batch(B, L, 3.0, step=s)
        ref.append(oracle.train_step(st, h, ptr, ids, 1.0 / B, 1e-2).dh)
    for rank in range(world):
        np.testing.assert_allclose(results[rank][0], ref[1], rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(results[rank][1], ref[2], rtol=1e-12, atol=1e-14)


# ------------------------------------------------ NEXT-2: the whole architecture, sharded
D_FEAT, P_DROP, DSEED = 12, 0.2, 5


class OracleDense:
    """CPU stand-in for DenseLayer (same method signatures) backed by the oracle: the column
    shard [c0, c1) of the dense layer (its columns of the whole layer's Glorot init; the
    oracle's dense arithmetic is per column, so a slice of its inputs is the shard)."""

    def __init__(self, c0=0, c1=M):
        full = oracle.DenseState.create(D_FEAT, M, DSEED)
        sl = slice(c0, c1)
        self.ds = oracle.DenseState(full.Wd[:, sl].copy(), full.bd[sl].copy(), full.mWd[:, sl].copy(),
                                    full.vWd[:, sl].copy(), full.mbd[sl].copy(), full.vbd[sl].copy(), 0)
        self.xt = self.z = None

    def forward(self, x, step=0, train=True):
        xt = oracle.dropout(x.numpy(), P_DROP, DSEED, step)[0] if train else x.numpy()
        z, _, h = oracle.dense_forward(self.ds.Wd, self.ds.bd, xt)
        self.xt, self.z = xt, z
        return torch.from_numpy(h)

    def backward_adam(self, dh, lr):
        dWd, _, dbd, _ = oracle.dense_backward(self.xt, self.z, dh.numpy())
        ds = self.ds
        ds.t += 1
        ds.Wd, ds.mWd, ds.vWd = oracle.adam(ds.Wd, dWd, ds.mWd, ds.vWd, ds.t, lr)
        ds.bd, ds.mbd, ds.vbd = oracle.adam(ds.bd, dbd, ds.mbd, ds.vbd, ds.t, lr)


def _worker_model(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2306_03725_b200.sharded import ShardedModel
        rb, re_ = shard_rows(L, rank, world)
        eng = OracleEngine(L, M, K_FAN, rb, re_, SEED)
        c0, c1 = shard_rows(M, rank, world)                 # this rank's dense columns
        model = ShardedModel(ShardedLayer(L, M, K_FAN, rank=rank, world=world, engine=eng, merge_fn=cpu_merge),
                             dense=OracleDense(c0, c1))
        assert (model.col_begin, model.col_end) == (c0, c1)
        out = {}
        for step in range(3):
            x = torch.from_numpy(synth.feature_batch(B, D_FEAT, step=step).astype(np.float64))
            if rank != 0:
                x = torch.zeros_like(x)                 # only the producer rank has the features
            model.broadcast_x(x)
            ptr, ids = synth.label_batch(B, L, 3.0, step=step)
            _, loss = model.train_step(x, step, torch.from_numpy(ptr), torch.from_numpy(ids), 1e-2,
                                       loss=torch.zeros(1, dtype=torch.float64), reduce_loss=True)
            out[f"loss{step}"] = float(loss.item())
        x = torch.from_numpy(synth.feature_batch(B, D_FEAT, step=9).astype(np.float64))
        s, i = model.predict_topk(x, 5)
        out["top_i"] = i.numpy()
        out["Wd"] = model.dense.ds.Wd
        out["W"] = eng.st.W
        results[rank] = out
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_model_matches_unsharded_oracle(world):
    """ShardedModel over 2 and 3 gloo ranks (dense layer column-sharded, h
    all-gathered, dh reduce-scattered; fixed fan-in layer label-sharded) == the unsharded
    oracle.model_train_step: the ranks' Wd column shards concatenate to the unsharded Wd,
    their label rows to W; identical losses and merged top-K."""
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker_model, args=(world, _free_port(), results), nprocs=world, join=True)
    st = oracle.State.create(L, M, K_FAN, SEED)
    ds = oracle.DenseState.create(D_FEAT, M, DSEED)
    for step in range(3):
        x = synth.feature_batch(B, D_FEAT, step=step).astype(np.float64)
        ptr, ids = synth.label_batch(B, L, 3.0, step=step)
        r = oracle.model_train_step(ds, st, x, step, P_DROP, DSEED, ptr, ids, 1.0 / B, 1e-2)
        for rank in range(world):
            assert results[rank][f"loss{step}"] == pytest.approx(r.sparse.loss, rel=1e-12)
    Wd_cat = np.concatenate([results[r]["Wd"] for r in range(world)], axis=1)
    assert Wd_cat.shape == ds.Wd.shape and results[0]["Wd"].shape[1] == shard_rows(M, 0, world)[1]
    np.testing.assert_allclose(Wd_cat, ds.Wd, rtol=0, atol=1e-12)
    np.testing.assert_allclose(np.concatenate([results[r]["W"] for r in range(world)]), st.W, rtol=0, atol=1e-12)
    _, _, h = oracle.dense_forward(ds.Wd, ds.bd, synth.feature_batch(B, D_FEAT, step=9).astype(np.float64))
    y, _ = oracle.forward(st.W, st.idx, st.bias, h)
    _, i_ref = oracle.topk(y, 5)
    for rank in range(world):
        assert (results[rank]["top_i"] == i_ref).all()
