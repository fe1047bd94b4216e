"""GPU parity of NEXT-2: the intermediate layer of the proposed architecture
(input dropout P:686-689 -> dense Wd P:594-603 -> ReLU) and the whole-architecture step,
through the C ABI, against the fp64 oracle.

Tolerances as in test_gpu_parity.py (R19): err = |x - x_ref| / max(|x_ref|, A_ref) <= 1e-4.
Bit-exact: the Philox init of Wd, the dropout keep mask.  Where a float decides an integer
(the ReLU mask of the backward) the oracle takes the GPU's decision (lockstep, R20).
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2306_03725_b200 import synth
from test_gpu_parity import ADAM, F32, adam_A, assert_close, dev, make, state_of, tens

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__ as g
    g.build_lib()


def L_():
    from paper_2306_03725_b200 import layer
    return layer


def make_dense(d, m, B=32, **kw):
    layer = L_()
    return layer.DenseLayer(layer.DenseConfig(d=d, m=m, max_batch=B, **kw), device=dev())


def dstate(dn):
    return {k: (v.cpu().numpy() if torch.is_tensor(v) else v) for k, v in dn.get_params().items()}


SHAPES = [(32, 512, 1000), (7, 37, 203), (70, 64, 300), (1, 5, 3), (32, 130, 4096),
          (32, 100, 37988)]   # > one column tile per SM (persistent TMA forward, backward ranges across tiles)


@pytest.mark.parametrize("d,m,seed", [(512, 1000, 7), (37, 203, 3), (5, 3, 1), (768, 4096, 42)])
def test_dense_init_bit_exact(d, m, seed):
    dn = make_dense(d, m, seed=seed)
    s = dstate(dn)
    ref = oracle.dense_init(d, m, seed)
    assert (s["Wd"].view(np.uint32) == ref.view(np.uint32)).all()
    assert (s["bd"] == 0).all() and (s["mWd"] == 0).all() and (s["vWd"] == 0).all() and s["t"] == 0


@pytest.mark.parametrize("B,d,p,step", [(32, 64, 0.1, 5), (7, 37, 0.2, 0), (70, 16, 0.5, 123456)])
@pytest.mark.parametrize("simt", [True, False], ids=["simt", "tcgen05"])
def test_dropout_mask_bit_exact(B, d, p, step, simt):
    """Wd = I, bd = 0, x > 0: h = xt, so h exposes the keep mask (bit-exact) and the scaled
    values: fp32 x*s exactly through the FP32 forward; within 3xTF32 rounding (the lo part is
    truncated to tf32 by the tensor core, ~2^-22 relative) through the tcgen05 forward."""
    layer = L_()
    dn = make_dense(d, d, B=B, seed=99, dropout=p, flags=layer.FF_FLAG_DENSE_SIMT if simt else 0)
    dn.set_params(Wd=tens(np.eye(d, dtype=np.float32)))
    x = np.abs(synth.feature_batch(B, d, step=3)) + np.float32(0.1)
    h = dn.forward(tens(x), step=step, train=True).cpu().numpy()
    xt, keep, s = oracle.dropout(x, p, seed=99, step=step)
    assert ((h != 0) == (keep == 1)).all()
    assert_close(h, xt, 0, "dropped-out features")
    h0 = dn.forward(tens(x), step=step, train=False).cpu().numpy()      # inference: no dropout
    if simt or B > 32:
        assert (h[keep == 1].astype(np.float32) == (x[keep == 1] * np.float32(s)).astype(np.float32)).all()
        assert (h0 == x).all()
    else:
        assert_close(h0, x.astype(np.float64), 0, "no-dropout features", rtol=1e-6)


@pytest.mark.parametrize("B,d,m", SHAPES)
@pytest.mark.parametrize("train", [False, True])
@pytest.mark.parametrize("simt", [False, True], ids=["tcgen05", "simt"])
def test_dense_forward_matches_oracle(B, d, m, train, simt):
    """B <= 32 runs the tcgen05 3xTF32 kernel unless FF_FLAG_DENSE_SIMT; B > 32 the FP32 one."""
    layer = L_()
    dn = make_dense(d, m, B=B, seed=5, dropout=0.1, flags=layer.FF_FLAG_DENSE_SIMT if simt else 0)
    bd = (np.random.default_rng(2).random(m, dtype=np.float32) - np.float32(0.5)) * np.float32(0.2)
    dn.set_params(bd=tens(bd))
    s = dstate(dn)
    x = synth.feature_batch(B, d, step=1)
    h = dn.forward(tens(x), step=11, train=train).cpu().numpy()
    xt = oracle.dropout(x, 0.1, seed=5, step=11)[0] if train else x.astype(np.float64)
    z, Az, href = oracle.dense_forward(s["Wd"], s["bd"], xt)
    assert_close(h, href, Az, "h = ReLU(z)")


@pytest.mark.parametrize("B,d,m", SHAPES)
def test_dense_backward_adam_lockstep(B, d, m):
    layer = L_()
    dn = make_dense(d, m, B=B, seed=8, dropout=0.1, flags=layer.FF_FLAG_STORE_GRADS)
    rng = np.random.default_rng(4)
    mWd = (rng.random((d, m), dtype=np.float32) * np.float32(1e-3))
    vWd = (rng.random((d, m), dtype=np.float32) * np.float32(1e-6))
    dn.set_params(mWd=tens(mWd), vWd=tens(vWd), t=3)
    s0 = dstate(dn)
    x = synth.feature_batch(B, d, step=2)
    h = dn.forward(tens(x), step=4, train=True).cpu().numpy()
    dh = synth.feature_batch(B, m, step=9) * np.float32(0.01)
    lr = F32(1e-3)
    dn.backward_adam(tens(dh), lr)
    dWd, dbd = (t.cpu().numpy() for t in dn.get_grads())
    s1 = dstate(dn)
    xt = oracle.dropout(x, 0.1, seed=8, step=4)[0]
    # the ReLU mask is the GPU's decision (h > 0 <=> z > 0): feed h as z (R20)
    rW, AW, rb, Ab = oracle.dense_backward(xt, h.astype(np.float64), dh)
    assert_close(dWd, rW, AW, "dWd")
    assert_close(dbd, rb, Ab, "dbd")
    assert s1["t"] == 4
    Wr, mr, vr = oracle.adam(s0["Wd"], dWd, s0["mWd"], s0["vWd"], 4, lr, **ADAM)
    assert_close(s1["Wd"], Wr, adam_A(s0["Wd"], Wr), "Wd'")
    # m' = b1 m + (1 - b1) q: R19 companion = the two terms' magnitudes (they can cancel)
    Am = np.abs(ADAM["beta1"] * s0["mWd"].astype(np.float64)) + np.abs((1 - ADAM["beta1"]) * dWd.astype(np.float64))
    assert_close(s1["mWd"], mr, Am, "mWd'"); assert_close(s1["vWd"], vr, 1e-30, "vWd'")
    br, mbr, vbr = oracle.adam(s0["bd"], dbd, s0["mbd"], s0["vbd"], 4, lr, **ADAM)
    assert_close(s1["bd"], br, adam_A(s0["bd"], br), "bd'")


def test_dense_backward_requires_forward_and_same_batch():
    layer = L_()
    dn = make_dense(8, 16, B=4)
    with pytest.raises(layer.FFError) as e:
        dn.backward_adam(tens(np.zeros((4, 16), np.float32)), 1e-3)
    assert e.value.status == layer.FF_ERR_STATE
    dn.forward(tens(synth.feature_batch(4, 8)), train=True)
    with pytest.raises(layer.FFError):
        dn.backward_adam(tens(np.zeros((3, 16), np.float32)), 1e-3)


def _model(L, m, k, d, B, dh_mode, p, flags=0):
    layer = L_()
    lay = make(L, m, k, B=B, seed=42, dh_mode=dh_mode, flags=flags)
    dn = make_dense(d, m, B=B, seed=17, dropout=p, flags=flags)
    return lay, dn


@pytest.mark.parametrize("dh_mode", [0, 1])
def test_model_step_equals_composed_calls(dh_mode):
    """fixedfanin_model_train_step (h, dh stay in the layer's column lines) == dense_forward ->
    train_step -> dense_backward_adam through [B][m] buffers.  CSC dh is deterministic, so
    the two paths are bit-identical there; atomic dh within rounding of its sum order."""
    layer = L_()
    L, m, k, d, B = 3000, 1024, 32, 96, 32
    lay1, dn1 = _model(L, m, k, d, B, dh_mode, 0.1)
    lay2, dn2 = _model(L, m, k, d, B, dh_mode, 0.1)
    loss1 = torch.zeros(1, device=dev()); loss2 = torch.zeros(1, device=dev())
    for step in range(3):
        x = tens(synth.feature_batch(B, d, step=step))
        ptr, ids = (tens(a) for a in synth.label_batch(B, L, 5.0, step=step))
        layer.model_train_step(dn1, lay1, x, step, ptr, ids, F32(1e-3), loss=loss1)
        h = dn2.forward(x, step=step, train=True)
        dh, _ = lay2.train_step(h, ptr, ids, F32(1e-3), loss=loss2)
        dn2.backward_adam(dh, F32(1e-3))
    s1, s2, d1, d2 = state_of(lay1), state_of(lay2), dstate(dn1), dstate(dn2)
    if dh_mode == 1:
        for kk in ("W", "idx", "bias", "mW", "vW"):
            assert (s1[kk] == s2[kk]).all(), kk
        for kk in ("Wd", "bd", "mWd", "vWd"):
            assert (d1[kk] == d2[kk]).all(), kk
        # the loss is summed across CTAs with atomics: equal up to that order
        assert abs(loss1.item() - loss2.item()) <= 1e-6 * abs(loss2.item())
    else:
        assert (s1["idx"] == s2["idx"]).all()
        assert np.allclose(s1["W"], s2["W"], rtol=1e-5, atol=1e-6)
        assert np.allclose(d1["Wd"], d2["Wd"], rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("dh_mode,B,k", [(0, 32, 16), (1, 32, 16), (2, 32, 16), (0, 70, 32), (1, 45, 32), (0, 32, 32)])
def test_model_step_lockstep_vs_oracle(dh_mode, B, k):
    """One whole-architecture step vs oracle.model_train_step from the GPU's state: loss, the
    sparse layer's and the dense layer's gradients (R19), then Adam on those gradients.
    B > 32 runs the 32-sample chunk paths of every kernel; k = 32, B <= 32 the pipelined one."""
    layer = L_()
    L, m, d = 2000, 512, 64
    lay, dn = _model(L, m, k, d, B, dh_mode, 0.1, flags=layer.FF_FLAG_STORE_GRADS)
    s0, d0 = state_of(lay), dstate(dn)
    x = synth.feature_batch(B, d, step=5)
    ptr, ids = synth.label_batch(B, L, 5.0, step=5)
    loss = torch.zeros(1, device=dev())
    lr = F32(1e-3)
    # the GPU's h of this step (a standalone forward of the same state, dropout mask and batch):
    # its ReLU mask is the GPU's decision, which the oracle's backward takes (R20)
    h_gpu = dn.forward(tens(x), step=5, train=True).cpu().numpy().astype(np.float64)
    layer.model_train_step(dn, lay, tens(x), 5, tens(ptr), tens(ids), lr, loss=loss)
    dW, db = (t.cpu().numpy() for t in lay.get_grads())
    dWd, dbd = (t.cpu().numpy() for t in dn.get_grads())
    s1, d1 = state_of(lay), dstate(dn)
    st = oracle.State(s0["W"].astype(np.float64), s0["idx"], s0["bias"].astype(np.float64),
                      s0["mW"].astype(np.float64), s0["vW"].astype(np.float64), s0["mb"].astype(np.float64),
                      s0["vb"].astype(np.float64), s0["t"])
    ds = oracle.DenseState(d0["Wd"].astype(np.float64), d0["bd"].astype(np.float64), d0["mWd"].astype(np.float64),
                           d0["vWd"].astype(np.float64), d0["mbd"].astype(np.float64), d0["vbd"].astype(np.float64),
                           d0["t"])
    r = oracle.model_train_step(ds, st, x, 5, 0.1, 17, ptr, ids, F32(1.0 / B), lr, **ADAM)
    assert abs(loss.item() - r.sparse.loss) <= 1e-4 * abs(r.sparse.loss)
    assert_close(dW, r.sparse.dW, r.sparse.AdW, "sparse dW")
    assert_close(db, r.sparse.db, r.sparse.Adb, "sparse db")
    assert_close(h_gpu, r.h, r.Az, "h")
    rWd, AWd, rbd, Abd = oracle.dense_backward(r.xt, h_gpu, r.sparse.dh)
    assert_close(dWd, rWd, AWd, "dense dWd")
    assert_close(dbd, rbd, Abd, "dense dbd")
    assert ((h_gpu > 0) == (r.z > 0)).mean() > 0.999     # the masks differ only at rounding-level |z|
    assert s1["t"] == 1 and d1["t"] == 1
    Wr, _, _ = oracle.adam(d0["Wd"], dWd, d0["mWd"], d0["vWd"], 1, lr, **ADAM)
    assert_close(d1["Wd"], Wr, adam_A(d0["Wd"], Wr), "Wd'")


@pytest.mark.parametrize("dh_mode", [0, 1])
def test_model_free_running_tiny_matches_oracle(dh_mode):
    """tiny config + the intermediate layer (d = 32): 5 whole-architecture steps, then one
    redistribution and a model prediction, the oracle evolving its own fp64 state."""
    layer = L_()
    L, m, k, d, B = 1000, 256, 16, 32, 32
    lay, dn = _model(L, m, k, d, B, dh_mode, 0.1)
    st = oracle.State.create(L, m, k, seed=42)
    ds = oracle.DenseState.create(d, m, seed=17)
    lr = F32(1e-3)
    for step in range(5):
        x = synth.feature_batch(B, d, step=step)
        ptr, ids = synth.label_batch(B, L, 5.0, step=step)
        layer.model_train_step(dn, lay, tens(x), step, tens(ptr), tens(ids), lr)
        oracle.model_train_step(ds, st, x, step, 0.1, 17, ptr, ids, F32(1.0 / B), lr, **ADAM)
    s, dd = state_of(lay), dstate(dn)
    assert_close(s["W"], st.W, np.abs(st.W) + 5 * lr, "W after 5 model steps")
    assert_close(dd["Wd"], ds.Wd, np.abs(ds.Wd) + 5 * lr, "Wd after 5 model steps")
    assert_close(s["bias"], st.bias, np.abs(st.bias) + 5 * lr, "bias after 5 model steps")
    lay.redistribute(5)
    x = synth.feature_batch(B, d, step=50)
    sc, ids_ = layer.model_predict_topk(dn, lay, tens(x), 5)
    h = dn.forward(tens(x), train=False)
    y = lay.forward(h).cpu().numpy().astype(np.float64)
    rs, rid = oracle.topk(y, 5)
    assert (ids_.cpu().numpy() == rid).all() and (sc.cpu().numpy() == rs).all()


@pytest.mark.parametrize("dh_mode", [0, 1])
def test_model_full_size_amazon_670k_sampled(dh_mode):
    """The bench's `model` configuration (Amazon-670K, 512-d features, 10% dropout, B = 32):
    the dense forward h against the oracle over the full [B][m]; one whole-architecture step
    checked on sampled label rows (sparse dW, db, W') and sampled dense columns (dWd, Wd'),
    lockstep (R20: the oracle takes the GPU's h, its ReLU mask and the GPU's dh)."""
    layer = L_()
    shape = synth.SHAPES["amazon-670k"]
    L, m, k, B, d = shape.L, shape.m, shape.k, shape.B, 512
    lay = make(L, m, k, B=B, seed=42, flags=layer.FF_FLAG_STORE_GRADS, dh_mode=dh_mode)
    dn = make_dense(d, m, B=B, seed=43, dropout=0.1, flags=layer.FF_FLAG_STORE_GRADS)
    s0, d0 = state_of(lay), dstate(dn)
    x = synth.feature_batch(B, d, step=3)
    ptr, ids = synth.label_batch(B, L, shape.avg_pos, step=3)
    h_gpu = dn.forward(tens(x), step=3, train=True)
    y = lay.forward(h_gpu).cpu().numpy().astype(np.float64)
    h_gpu = h_gpu.cpu().numpy().astype(np.float64)
    xt = oracle.dropout(x, 0.1, seed=43, step=3)[0]
    z, Az, href = oracle.dense_forward(d0["Wd"], d0["bd"], xt)
    assert_close(h_gpu, href, Az, "h (full)")
    loss = torch.zeros(1, device=dev())
    layer.model_train_step(dn, lay, tens(x), 3, tens(ptr), tens(ids), F32(1e-3), loss=loss)
    dW, db = (t.cpu().numpy() for t in lay.get_grads())
    dWd, dbd = (t.cpu().numpy() for t in dn.get_grads())
    s1, d1 = state_of(lay), dstate(dn)
    rng = np.random.default_rng(9)
    rows = np.sort(rng.choice(L, 256, replace=False))
    g, lref = oracle.bce_grad(y, ptr, ids, F32(1.0 / B))
    assert abs(loss.item() - lref) <= 1e-4 * abs(lref)
    dWr, AdW, dbr, Adb = oracle.weight_grad(s0["idx"][rows], h_gpu, g[:, rows])
    assert_close(dW[rows], dWr, AdW, "sparse dW rows")
    assert_close(db[rows], dbr, Adb, "sparse db rows")
    Wr, _, _ = oracle.adam(s0["W"][rows], dW[rows], s0["mW"][rows], s0["vW"][rows], 1, F32(1e-3), **ADAM)
    assert_close(s1["W"][rows], Wr, adam_A(s0["W"][rows], Wr), "W' rows")
    # dense gradients on sampled columns, from the oracle's Alg. 2 dh over every connection
    dhr, _ = oracle.input_grad(s0["W"], s0["idx"], g, m)
    cols = np.sort(rng.choice(m, 512, replace=False))
    rWd, AWd, rbd, Abd = oracle.dense_backward(xt, h_gpu[:, cols], dhr[:, cols])
    assert_close(dWd[:, cols], rWd, AWd, "dense dWd cols")
    assert_close(dbd[cols], rbd, Abd, "dense dbd cols")
    Wdr, _, _ = oracle.adam(d0["Wd"][:, cols], dWd[:, cols], d0["mWd"][:, cols], d0["vWd"][:, cols], 1, F32(1e-3), **ADAM)
    assert_close(d1["Wd"][:, cols], Wdr, adam_A(d0["Wd"][:, cols], Wdr), "Wd' cols")


@pytest.mark.parametrize("dh_mode", [1, 0])
def test_model_step_cuda_graph_replay(dh_mode):
    """The whole-architecture step is capturable with step = FF_STEP_AUTO: both Adam counters
    and the dropout step key live on the device, so replays of one captured step equal eager
    steps with explicit steps 1, 2, ... (CSC: bit-identical; atomic: dh rounding order)."""
    layer = L_()
    L, m, k, B, d = 2000, 1024, 32, 32, 64
    runs = []
    for graph in (True, False):
        lay = make(L, m, k, B=B, seed=42, dh_mode=dh_mode)
        dn = make_dense(d, m, B=B, seed=43, dropout=0.1)
        xs = [tens(synth.feature_batch(B, d, step=s)) for s in range(5)]
        lb = [synth.label_batch(B, L, 5.0, step=s) for s in range(5)]
        nnz = max(int(p_[-1]) for p_, _ in lb)
        sx = torch.zeros((B, d), device=dev()); sp = torch.zeros(B + 1, dtype=torch.int32, device=dev())
        si = torch.zeros(nnz, dtype=torch.int32, device=dev()); loss = torch.zeros(1, device=dev())

        def load(s):
            sx.copy_(xs[s]); sp.copy_(tens(lb[s][0])); si[:len(lb[s][1])].copy_(tens(lb[s][1]))
        if graph:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                load(0)
                layer.model_train_step(dn, lay, sx, layer.FF_STEP_AUTO, sp, si, F32(1e-3), loss=loss)
            torch.cuda.current_stream().wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                layer.model_train_step(dn, lay, sx, layer.FF_STEP_AUTO, sp, si, F32(1e-3), loss=loss)
            for s in range(1, 5):
                load(s)
                g.replay()
        else:
            for s in range(5):
                load(s)
                layer.model_train_step(dn, lay, sx, s + 1, sp, si, F32(1e-3), loss=loss)
        torch.cuda.synchronize()
        runs.append((state_of(lay), dstate(dn), float(loss.item())))
    (sa, da, la), (sb, db_, lb_) = runs
    assert sa["t"] == sb["t"] == 5 and da["t"] == db_["t"] == 5
    if dh_mode == 1:
        for key in ("W", "bias", "mW", "vW", "idx"):
            assert (sa[key] == sb[key]).all(), key
        for key in ("Wd", "bd", "mWd", "vWd"):
            assert (da[key] == db_[key]).all(), key
        # the loss is an fp32 atomicAdd of per-CTA partial sums (B L = 64,000 terms) in arrival
        # order: the two runs agree to fp32 summation-order rounding, ~1e-6 relative
        assert abs(la - lb_) <= 1e-5 * abs(lb_)
    else:
        for key in ("Wd", "W"):
            ref = (db_ if key == "Wd" else sb)[key]
            got = (da if key == "Wd" else sa)[key]
            assert np.allclose(got, ref, rtol=1e-4, atol=1e-6), key
        assert abs(la - lb_) <= 1e-5 * abs(lb_)


def test_dense_auto_step_equals_explicit_steps():
    """Standalone dense layer: forward(step = FF_STEP_AUTO) keys the dropout on the device
    counter + 1 and backward_adam advances it (k_step_t), so three AUTO steps equal three
    steps with explicit keys 1, 2, 3: same h, same Wd / moments, t = 3."""
    layer = L_()
    d, m, B = 64, 512, 32
    a = make_dense(d, m, B=B, seed=21, dropout=0.2)
    b = make_dense(d, m, B=B, seed=21, dropout=0.2)
    for s in range(3):
        x = tens(synth.feature_batch(B, d, step=s))
        dh = tens(synth.feature_batch(B, m, step=10 + s) * np.float32(0.01))
        ha = a.forward(x, step=layer.FF_STEP_AUTO, train=True)
        hb = b.forward(x, step=s + 1, train=True)
        assert torch.equal(ha, hb), s
        a.backward_adam(dh, F32(1e-3))
        b.backward_adam(dh, F32(1e-3))
    torch.cuda.synchronize()
    da, db_ = dstate(a), dstate(b)
    assert da["t"] == db_["t"] == 3
    for key in ("Wd", "bd", "mWd", "vWd"):
        assert (da[key] == db_[key]).all(), key


@pytest.mark.parametrize("P,d,m,B", [(2, 64, 512, 32), (3, 37, 203, 7), (4, 512, 4100, 32), (3, 48, 1000, 70)])
def test_column_shards_concatenate_to_the_unsharded_layer(P, d, m, B):
    """SURVEY §8(f)2 on one GPU: P virtual column shards [m r / P, m (r+1) / P) of the dense
    layer (col_begin, m_global): their Philox init, training forward (same dropout mask) and
    backward + Adam on the dh columns are bit-identical to the unsharded layer's columns (the
    arithmetic of a column does not depend on the others), over two steps."""
    layer = L_()
    full = make_dense(d, m, B=B, seed=23, dropout=0.1)
    cols = [(m * r // P, m * (r + 1) // P) for r in range(P)]
    shards = [make_dense(d, e - b, B=B, seed=23, dropout=0.1, col_begin=b, m_global=m) for b, e in cols]
    sf = dstate(full)
    assert (np.concatenate([dstate(s)["Wd"] for s in shards], axis=1).view(np.uint32) == sf["Wd"].view(np.uint32)).all()
    for step in (1, 2):
        x = tens(synth.feature_batch(B, d, step=step))
        hf = full.forward(x, step=step, train=True)
        hs = [s.forward(x, step=step, train=True) for s in shards]
        assert torch.equal(torch.cat(hs, dim=1), hf), step
        dh = tens(synth.signed_hidden_batch(B, m, step=20 + step, scale=0.01))
        full.backward_adam(dh, F32(1e-3))
        for s, (b, e) in zip(shards, cols):
            s.backward_adam(dh[:, b:e].contiguous(), F32(1e-3))
    torch.cuda.synchronize()
    sf = dstate(full)
    cat = [dstate(s) for s in shards]
    for key, ax in (("Wd", 1), ("mWd", 1), ("vWd", 1), ("bd", 0), ("mbd", 0), ("vbd", 0)):
        assert (np.concatenate([c[key] for c in cat], axis=ax) == sf[key]).all(), key


def test_sharded_model_world1_equals_model_step_composition():
    """ShardedModel with one rank runs the unsharded layer through the standalone calls:
    its state after two steps equals forward + train_step + backward_adam composed by hand,
    bit for bit (CSC dh: deterministic summation order)."""
    from paper_2306_03725_b200.sharded import ShardedLayer, ShardedModel
    L, m, k, d, B = 3000, 512, 32, 64, 32
    sm = ShardedModel(ShardedLayer(L, m, k, device=dev(), max_batch=B, seed=9, dh_mode=1), d=d, device=dev(), seed=3,
                      dropout=0.1, max_batch=B)
    lay = make(L, m, k, B=B, seed=9, dh_mode=1)
    dn = make_dense(d, m, B=B, seed=3, dropout=0.1)
    for step in (1, 2):
        x = tens(synth.feature_batch(B, d, step=step))
        ptr, ids = synth.label_batch(B, L, 5.0, step=step)
        sm.train_step(x, step, tens(ptr), tens(ids), F32(1e-3))
        h = dn.forward(x, step=step, train=True)
        dh, _ = lay.train_step(h, tens(ptr), tens(ids), F32(1e-3))
        dn.backward_adam(dh, F32(1e-3))
    torch.cuda.synchronize()
    a, b = dstate(sm.dense), dstate(dn)
    for key in ("Wd", "bd", "mWd", "vWd"):
        assert (a[key] == b[key]).all(), key
    sa, sb = state_of(sm.layer.engine), state_of(lay)
    for key in ("W", "idx", "bias", "mW", "vW"):
        assert (sa[key] == sb[key]).all(), key
