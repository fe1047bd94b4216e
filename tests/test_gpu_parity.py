"""GPU parity: the sm_100a kernels (through the C ABI) against the fp64 oracle.

Tolerances (R19/R20): floats compare with
    err = |x_gpu - x_ref| / max(|x_ref|, A_ref)  <= 1e-4
where A_ref is the oracle's sum of |terms| of that output; indices, redistribution and
top-K label sets are bit-exact.  Lockstep protocol: the oracle step is evaluated on the
GPU's state (fp32 widened exactly to fp64), so |W| orders and scores are comparable.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2306_03725_b200 import synth

pytestmark = pytest.mark.gpu

RTOL = 1e-4
F32 = lambda x: float(np.float32(x))       # the GPU's fp32 hyper-parameters, widened exactly


@pytest.fixture(scope="module", autouse=True)
def built():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__ as g
    g.build_lib()


def L_():
    from paper_2306_03725_b200 import layer
    return layer


def dev():
    return torch.device("cuda:0")


def make(L, m, k, B=32, **kw):
    layer = L_()
    return layer.FixedFanInLayer(layer.LayerConfig(L_global=kw.pop("L_global", L), m=m, k=k, max_batch=B, **kw),
                                 device=dev())


def tens(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev())


def rel_err(x, ref, A):
    x = np.asarray(x, dtype=np.float64)
    return np.abs(x - ref) / np.maximum(np.maximum(np.abs(ref), A), 1e-300)


def assert_close(x, ref, A, what, rtol=RTOL):
    e = rel_err(x, ref, A)
    assert e.max() <= rtol, f"{what}: max err {e.max():.3e} at {np.unravel_index(e.argmax(), e.shape)}"


def dh_close(a, b):
    """Two GPU dh results whose fp32 sums ran in different (atomic) orders: equal up to
    rounding relative to the dh scale (R19/R21; elements with cancellation have no
    meaningful plain relative error)."""
    scale = float(torch.maximum(a.abs().max(), b.abs().max()))
    return torch.allclose(a, b, rtol=1e-5, atol=1e-5 * scale + 1e-30)


def adam_A(W_old, W_new_ref):
    """R19 companion of p' = p - lr*mhat/(sqrt(vhat)+eps): |p| + |update| (the subtraction's terms)."""
    W_old = np.asarray(W_old, dtype=np.float64)
    return np.abs(W_old) + np.abs(np.asarray(W_new_ref) - W_old)


def assert_adam_update(W_old, W_new, W_ref, what):
    """Direct check of the Adam update u = p - p' itself (not only of p' = p - u at the scale
    of |p| + |u|): |(p'_gpu - p) - (p'_ref - p)| <= 1e-4 |u_ref| + 2 ulp_fp32(p, p'), the last
    term being the fp32 rounding of the subtraction p - u on the GPU."""
    W_old = np.asarray(W_old, dtype=np.float32)
    W_new = np.asarray(W_new, dtype=np.float32)
    d_gpu = W_new.astype(np.float64) - W_old.astype(np.float64)      # exact in fp64
    u_ref = np.asarray(W_ref, dtype=np.float64) - W_old.astype(np.float64)
    ulp = np.maximum(np.spacing(np.abs(W_old)), np.spacing(np.abs(W_new))).astype(np.float64)
    err = np.abs(d_gpu - u_ref)
    bound = 1e-4 * np.abs(u_ref) + 2 * ulp
    bad = err > bound
    assert not bad.any(), (f"{what}: {bad.sum()} updates off, worst err {err[bad].max():.3e} "
                           f"vs bound {bound[bad][err[bad].argmax()]:.3e}")


def state_of(lay):
    p = lay.get_params()
    return {k: (v.cpu().numpy() if torch.is_tensor(v) else v) for k, v in p.items()}


ADAM = dict(beta1=F32(0.9), beta2=F32(0.999), eps=F32(1e-8))


# ------------------------------------------------------------------ init (bit-exact)
@pytest.mark.parametrize("L,m,k,row_begin,Lg", [(1000, 256, 16, 0, 1000), (777, 4096, 32, 123, 5000),
                                                  (50, 37, 13, 0, 50), (40, 5, 5, 10, 50), (3, 1, 1, 0, 3),
                                                  (300, 65536, 64, 7, 400), (90, 70, 47, 0, 90), (20, 64, 64, 0, 20)])
def test_init_bit_exact(L, m, k, row_begin, Lg):
    lay = make(L, m, k, L_global=Lg, row_begin=row_begin, L_local=L, seed=42)
    s = state_of(lay)
    idx, W = oracle.init(L, m, k, seed=42, row_begin=row_begin)
    assert (s["idx"] == idx).all()
    assert (s["W"].view(np.uint32) == W.view(np.uint32)).all()
    assert (s["bias"] == 0).all() and (s["mW"] == 0).all() and (s["vW"] == 0).all() and s["t"] == 0


def test_init_full_amazon_670k_sampled_rows():
    L, m, k = 670091, 32768, 32
    lay = make(L, m, k, seed=42)
    s = state_of(lay)
    rng = np.random.default_rng(0)
    for j in list(rng.choice(L, 64, replace=False)) + [0, L - 1]:
        idx, W = oracle.init(1, m, k, seed=42, row_begin=int(j))
        assert (s["idx"][j] == idx[0]).all() and (s["W"][j].view(np.uint32) == W[0].view(np.uint32)).all()
    assert all(len(set(r)) == k for r in s["idx"][::997])


# --------------------------------------------------------------- forward / backward
CASES = [(1000, 256, 16, 32), (1000, 256, 16, 5), (333, 100, 13, 37), (2000, 512, 32, 100), (97, 64, 1, 1),
         (64, 32, 32, 128), (1500, 2048, 64, 32), (400, 300, 50, 40), (130, 64, 64, 7), (700, 512, 32, 300),
         (300, 256, 32, 1024)]                       # FF_MAX_BATCH: 32 sample chunks


@pytest.mark.parametrize("L,m,k,B", CASES)
def test_forward_parity(L, m, k, B):
    lay = make(L, m, k, B=B, seed=7)
    W, idx, bias = synth.random_params(L, m, k, seed=L + B)
    lay.set_params(W=tens(W), idx=tens(idx), bias=tens(bias))
    h = synth.hidden_batch(B, m, step=3)
    y = lay.forward(tens(h)).cpu().numpy()
    yr, Ay = oracle.forward(W, idx, bias, h)
    assert_close(y, yr, Ay, "y")


DH = pytest.mark.parametrize("dh_mode", [0, 1, 2], ids=["atomic", "csc", "hybrid"])


@pytest.mark.parametrize("m,offset", [(257, 0), (258, 0), (256, 1), (256, 0)])
def test_transpose_kernels_scalar_and_vector_paths(m, offset):
    """k_prep / k_dh_out take 16-B vector paths only when m % 4 == 0 and h / dh are 16-B
    aligned: odd widths and a misaligned (offset) h / dh view run the scalar paths.  Forward
    y and backward dh against the oracle either way."""
    L, k, B = 500, 16, 32
    lay = make(L, m, k, B=B, seed=9)
    W, idx, bias = synth.random_params(L, m, k, seed=m + offset)
    lay.set_params(W=tens(W), idx=tens(idx), bias=tens(bias))
    h = synth.hidden_batch(B, m, step=5)
    ptr, ids = synth.label_batch(B, L, 5.0, step=5)
    hb = torch.zeros(B * m + offset, device=dev())
    hb[offset:].copy_(tens(h).reshape(-1))
    hv = hb[offset:].view(B, m)                        # data_ptr() % 16 != 0 when offset = 1
    y = lay.forward(hv)
    yr, Ay = oracle.forward(W, idx, bias, h)
    assert_close(y.cpu().numpy(), yr, Ay, "y")
    db_ = torch.zeros(B * m + offset, device=dev())
    dh = db_[offset:].view(B, m)
    lay.backward(hv, y, tens(ptr), tens(ids), dh=dh)
    g, _ = oracle.loss_grad("bce", y.cpu().numpy().astype(np.float64), ptr, ids, F32(1.0 / B))
    dhr, Adh = oracle.input_grad(W, idx, g, m)
    assert_close(dh.cpu().numpy(), dhr, Adh, "dh")


LOSS = pytest.mark.parametrize("loss", ["bce", "sqh"])


def loss_id(loss):
    return L_().FF_LOSS_SQH if loss == "sqh" else L_().FF_LOSS_BCE


@LOSS
@DH
@pytest.mark.parametrize("L,m,k,B", CASES)
def test_backward_and_adam_parity(L, m, k, B, dh_mode, loss):
    lay = make(L, m, k, B=B, seed=8, dh_mode=dh_mode, loss=loss_id(loss))
    W, idx, bias = synth.random_params(L, m, k, seed=L + 2 * B, scale=0.5)
    lay.set_params(W=tens(W), idx=tens(idx), bias=tens(bias))
    h = synth.hidden_batch(B, m, step=4)
    ptr, ids = synth.label_batch(B, L, 5.0, step=4)
    y = lay.forward(tens(h))
    loss_t = torch.zeros(1, device=dev())
    dh, _ = lay.backward(tens(h), y, tens(ptr), tens(ids), loss=loss_t)
    dW, db = lay.get_grads()
    yn = y.cpu().numpy().astype(np.float64)
    g, lr_ = oracle.loss_grad(loss, yn, ptr, ids, F32(1.0 / B))
    dWr, AdW, dbr, Adb = oracle.weight_grad(idx, h, g)
    dhr, Adh = oracle.input_grad(W, idx, g, m)
    assert_close(dW.cpu().numpy(), dWr, AdW, "dW")
    assert_close(db.cpu().numpy(), dbr, Adb, "db")
    assert_close(dh.cpu().numpy(), dhr, Adh, "dh")
    assert abs(loss_t.item() - lr_) <= RTOL * abs(lr_)
    # Adam on the GPU's gradients (lockstep): elementwise fp32 vs fp64
    lay.adam_step(1e-3)
    s = state_of(lay)
    dWg, dbg = dW.cpu().numpy(), db.cpu().numpy()
    lr32 = F32(1e-3)
    Wr, mr, vr = oracle.adam(W, dWg, np.zeros_like(dWg), np.zeros_like(dWg), 1, lr32, **ADAM)
    br, mbr, vbr = oracle.adam(bias, dbg, np.zeros(L), np.zeros(L), 1, lr32, **ADAM)
    assert_close(s["W"], Wr, adam_A(W, Wr), "W'")
    assert_close(s["mW"], mr, 0, "mW'")
    assert_close(s["vW"], vr, 1e-30, "vW'")
    assert_close(s["bias"], br, adam_A(bias, br), "bias'")
    assert_adam_update(W, s["W"], Wr, "W update")
    assert_adam_update(bias, s["bias"], br, "bias update")
    assert s["t"] == 1


@DH
@pytest.mark.parametrize("L,m,k,B", [(1000, 256, 16, 32), (333, 100, 13, 37), (2000, 512, 32, 100),
                                     (3000, 512, 32, 32), (777, 300, 32, 7), (65, 40, 32, 1)])
def test_fused_step_equals_unfused_path(L, m, k, B, dh_mode):
    """train_step (one fused kernel) = forward + backward + adam_step: dW, db and the
    updated state are bit-identical (same device arithmetic), dh equal up to atomic order."""
    layer = L_()
    W, idx, bias = synth.random_params(L, m, k, seed=5, scale=0.5)
    a = make(L, m, k, B=B, flags=layer.FF_FLAG_STORE_GRADS, dh_mode=dh_mode)
    b = make(L, m, k, B=B, dh_mode=dh_mode)
    for x in (a, b):
        x.set_params(W=tens(W), idx=tens(idx), bias=tens(bias))
    for step in range(3):
        h = tens(synth.hidden_batch(B, m, step=step))
        ptr, ids = synth.label_batch(B, L, 5.0, step=step)
        la, lb = torch.zeros(1, device=dev()), torch.zeros(1, device=dev())
        dha, _ = a.train_step(h, tens(ptr), tens(ids), 1e-2, loss=la)
        dWa, dba = a.get_grads()
        y = b.forward(h)
        dhb, _ = b.backward(h, y, tens(ptr), tens(ids), loss=lb)
        dWb, dbb = b.get_grads()
        b.adam_step(1e-2)
        assert torch.equal(dWa, dWb) and torch.equal(dba, dbb)
        sa, sb = state_of(a), state_of(b)
        for key in ("W", "mW", "vW", "bias", "mb", "vb", "idx"):
            assert (sa[key] == sb[key]).all(), key
        if dh_mode == 1:
            assert torch.equal(dha, dhb)          # CSC pull: fixed summation order
        else:
            assert dh_close(dha, dhb)
        assert abs(la.item() - lb.item()) <= 1e-5 * abs(lb.item())


@LOSS
@DH
@pytest.mark.parametrize("k,B", [(16, 32), (32, 32), (64, 32), (32, 16), (32, 5)])
def test_fused_step_lockstep_vs_oracle(dh_mode, loss, k, B):
    L, m = 1000, 256
    layer = L_()
    lay = make(L, m, k, B=B, flags=layer.FF_FLAG_STORE_GRADS, seed=42, dh_mode=dh_mode, loss=loss_id(loss))
    for step in range(5):
        s0 = state_of(lay)
        st = oracle.State(s0["W"].astype(np.float64), s0["idx"], s0["bias"].astype(np.float64),
                          s0["mW"].astype(np.float64), s0["vW"].astype(np.float64), s0["mb"].astype(np.float64),
                          s0["vb"].astype(np.float64), s0["t"])
        h = synth.hidden_batch(B, m, step=step)
        ptr, ids = synth.label_batch(B, L, 5.0, step=step)
        y_gpu = lay.forward(tens(h)).cpu().numpy().astype(np.float64)     # = the fused step's y
        loss_t = torch.zeros(1, device=dev())
        dh, _ = lay.train_step(tens(h), tens(ptr), tens(ids), F32(1e-3), loss=loss_t)
        dW, db = lay.get_grads()
        r = oracle.train_step(st, h, ptr, ids, F32(1.0 / B), F32(1e-3), loss=loss, **ADAM)
        assert_close(y_gpu, r.y, r.Ay, f"y step {step}")
        if loss == "sqh":
            # the hinge's zero/non-zero decision max(0, 1 - t'y) is taken on the kernel's y
            # (fp32) on both sides; it may differ from the fp64 decision only at a margin tie
            g2, _ = oracle.loss_grad(loss, y_gpu, ptr, ids, F32(1.0 / B))
            flip = (g2 != 0) != (r.g != 0)
            tp = -np.ones((B, L))                                       # t' = +-1
            for b_ in range(B):
                tp[b_, ids[ptr[b_]:ptr[b_ + 1]]] = 1.0
            assert (np.abs(1 - tp * r.y)[flip] <= RTOL * r.Ay[flip]).all(), "hinge decision away from a tie"
            dWr, AdWr, dbr, Adbr = oracle.weight_grad(s0["idx"], h, g2)
            dhr, Adhr = oracle.input_grad(s0["W"], s0["idx"], g2, m)
        else:
            dWr, AdWr, dbr, Adbr, dhr, Adhr = r.dW, r.AdW, r.db, r.Adb, r.dh, r.Adh
        assert_close(dh.cpu().numpy(), dhr, Adhr, f"dh step {step}")
        assert_close(dW.cpu().numpy(), dWr, AdWr, f"dW step {step}")
        assert_close(db.cpu().numpy(), dbr, Adbr, f"db step {step}")
        assert abs(loss_t.item() - r.loss) <= RTOL * r.loss
        # Adam applied by the oracle to the GPU's gradient: tight elementwise parity
        s1 = state_of(lay)
        Wr, mr, vr = oracle.adam(s0["W"], dW.cpu().numpy(), s0["mW"], s0["vW"], s0["t"] + 1, F32(1e-3), **ADAM)
        assert_close(s1["W"], Wr, adam_A(s0["W"], Wr), "W'")
        assert_close(s1["mW"], mr, 0, "m'"); assert_close(s1["vW"], vr, 1e-30, "v'")
        assert_adam_update(s0["W"], s1["W"], Wr, f"W update step {step}")
        br, _, _ = oracle.adam(s0["bias"], db.cpu().numpy(), s0["mb"], s0["vb"], s0["t"] + 1, F32(1e-3), **ADAM)
        assert_adam_update(s0["bias"], s1["bias"], br, f"bias update step {step}")
        assert s1["t"] == step + 1


@pytest.mark.parametrize("t0", [41, 999, 123456])
def test_set_params_t_drives_the_device_step_counter(t0):
    """set_params(t) reaches the device counter: the next fused step and the next unfused
    adam_step use the bias corrections of t0 + 1 and t0 + 2 (R6, R7), and get_params reads
    the counter back."""
    L, m, k, B = 800, 256, 32, 32
    layer = L_()
    lay = make(L, m, k, B=B, flags=layer.FF_FLAG_STORE_GRADS, seed=5)
    rng = np.random.default_rng(t0)
    mW = (rng.random((L, k)) * 1e-3).astype(np.float32); vW = (rng.random((L, k)) * 1e-6).astype(np.float32)
    lay.set_params(mW=tens(mW), vW=tens(vW), t=t0)
    assert state_of(lay)["t"] == t0
    s0 = state_of(lay)
    h = synth.hidden_batch(B, m, step=1)
    ptr, ids = synth.label_batch(B, L, 5.0, step=1)
    lay.train_step(tens(h), tens(ptr), tens(ids), F32(1e-3))
    dW, _ = lay.get_grads()
    s1 = state_of(lay)
    assert s1["t"] == t0 + 1
    Wr, mr, vr = oracle.adam(s0["W"], dW.cpu().numpy(), s0["mW"], s0["vW"], t0 + 1, F32(1e-3), **ADAM)
    assert_close(s1["W"], Wr, adam_A(s0["W"], Wr), "W' (fused)")
    assert_adam_update(s0["W"], s1["W"], Wr, "W update (fused, t0 + 1)")
    y = lay.forward(tens(h))
    lay.backward(tens(h), y, tens(ptr), tens(ids))
    dW2, _ = lay.get_grads()
    lay.adam_step(F32(1e-3))
    s2 = state_of(lay)
    assert s2["t"] == t0 + 2
    Wr2, _, _ = oracle.adam(s1["W"], dW2.cpu().numpy(), s1["mW"], s1["vW"], t0 + 2, F32(1e-3), **ADAM)
    assert_close(s2["W"], Wr2, adam_A(s1["W"], Wr2), "W' (unfused)")
    assert_adam_update(s1["W"], s2["W"], Wr2, "W update (unfused, t0 + 2)")


@DH
def test_free_running_tiny_run_matches_oracle(dh_mode):
    """tiny config of BASELINE.json: 5 Adam steps + 1 redistribution, then predict K = 5.
    The oracle evolves its own fp64 state from the same Philox init."""
    L, m, k, B = 1000, 256, 16, 32
    lay = make(L, m, k, B=B, seed=42, dh_mode=dh_mode)
    st = oracle.State.create(L, m, k, seed=42)
    for step in range(5):
        h = synth.hidden_batch(B, m, step=step)
        ptr, ids = synth.label_batch(B, L, 5.0, step=step)
        lay.train_step(tens(h), tens(ptr), tens(ids), F32(1e-3))
        oracle.train_step(st, h, ptr, ids, F32(1.0 / B), F32(1e-3), **ADAM)
    s = state_of(lay)
    A = np.abs(st.W) + 5 * F32(1e-3)            # 5 steps of at most ~lr each
    assert_close(s["W"], st.W, A, "W after 5 steps")
    lay.redistribute(5)
    p = int(np.floor(F32(0.1) * k))
    # redistribution is bit-exact given the state: run the oracle on the GPU's pre-call state
    W2, idx2, m2, v2 = oracle.redistribute(s["W"], s["idx"], s["mW"], s["vW"], m, p, seed=42, step=5)
    s2 = state_of(lay)
    assert (s2["idx"] == idx2).all() and (s2["W"] == W2).all() and (s2["mW"] == m2).all() and (s2["vW"] == v2).all()
    # and the free-running oracle (its own fp64 state) agrees except at near-ties of |W|
    # (SURVEY §8(c).4): the regrow draws and the pre-call sets are identical (same Philox key,
    # same idx), so a row can only differ if the p-th and (p+1)-th smallest |W| swap places
    # between the fp32 and fp64 runs, i.e. if their fp64 gap is within the two elements'
    # R19 error bound after 5 steps: 1e-4 (|W| + 5 lr) each.
    Wf, idxf, _, _ = oracle.redistribute(st.W, st.idx, st.mW, st.vW, m, p, seed=42, step=5)
    rows = np.where((idxf != s2["idx"]).any(axis=1))[0]
    lr5 = 5 * F32(1e-3)
    for j in rows:
        a = np.sort(np.abs(st.W[j]))
        gap = a[p] - a[p - 1]
        tol = 1e-4 * (a[p] + lr5) + 1e-4 * (a[p - 1] + lr5)
        assert gap <= tol, f"row {j}: pruned set differs without a near-tie (gap {gap:.3e} > {tol:.3e})"
    print(f"free-running redistribution: {len(rows)} of {L} rows differ, all at near-ties of |W|")
    # one more step after the redistribution: dh must use the new connections (CSC rebuilt)
    s2 = state_of(lay)
    st2 = oracle.State(s2["W"].astype(np.float64), s2["idx"], s2["bias"].astype(np.float64),
                       s2["mW"].astype(np.float64), s2["vW"].astype(np.float64), s2["mb"].astype(np.float64),
                       s2["vb"].astype(np.float64), s2["t"])
    h = synth.hidden_batch(B, m, step=6)
    ptr, ids = synth.label_batch(B, L, 5.0, step=6)
    dh, _ = lay.train_step(tens(h), tens(ptr), tens(ids), F32(1e-3))
    r = oracle.train_step(st2, h, ptr, ids, F32(1.0 / B), F32(1e-3), **ADAM)
    assert_close(dh.cpu().numpy(), r.dh, r.Adh, "dh after redistribution")
    h = synth.hidden_batch(B, m, step=99)
    sc, ids_ = lay.predict_topk(tens(h), 5)
    y = lay.forward(tens(h)).cpu().numpy().astype(np.float64)
    _, oid = oracle.topk(y, 5)
    assert (ids_.cpu().numpy() == oid).all()


# ------------------------------------------------------------------- redistribution
@pytest.mark.parametrize("L,m,k,frac,step", [(1000, 256, 16, 0.1, 1000), (3000, 4096, 32, 0.1, 7),
                                              (500, 40, 32, 0.25, 3), (64, 3, 2, 0.5, 1), (800, 65536, 64, 0.1, 1000),
                                              (300, 120, 48, 0.3, 11), (50, 70, 64, 0.05, 2)])
def test_redistribution_bit_exact(L, m, k, frac, step):
    lay = make(L, m, k, seed=11, prune_frac=frac)
    W, idx, _ = synth.random_params(L, m, k, seed=3)
    W[::3, 1] = W[::3, 0]            # ties
    W[::4, 2 % k] = -W[::4, 0]       # ties across sign
    W[::5, 0] = 0.0
    rng = np.random.default_rng(1)
    mW, vW = rng.random((L, k)).astype(np.float32), rng.random((L, k)).astype(np.float32)
    lay.set_params(W=tens(W), idx=tens(idx), mW=tens(mW), vW=tens(vW))
    lay.redistribute(step)
    s = state_of(lay)
    p = int(np.floor(F32(frac) * k))
    W2, idx2, m2, v2 = oracle.redistribute(W, idx, mW, vW, m, p, seed=11, step=step)
    assert (s["idx"] == idx2).all()
    assert (s["W"] == W2).all() and (s["mW"] == m2).all() and (s["vW"] == v2).all()
    assert all(len(set(r)) == k for r in s["idx"])


@pytest.mark.parametrize("k,frac", [(16, 0.1), (32, 0.1), (32, 0.25)])
def test_hundred_train_redistribute_cycles(k, frac):
    """SPEC acceptance criterion 3 on the GPU: 100 interleaved train / redistribute
    cycles.  Every redistribution is checked in lockstep against the oracle's on the GPU's
    pre-call state (bit-exact W, idx, moments), and afterwards every row still has k distinct
    in-range indices, the regrown slots have zero weight and moments, the untouched slots are
    bitwise unchanged, and the pruned slots were the row's p smallest (|W|, slot) keys (R9)."""
    L, m, B = 300, 256, 16
    lay = make(L, m, k, B=B, seed=23, prune_frac=frac)
    p = int(np.floor(F32(frac) * k))
    for cyc in range(100):
        h = synth.hidden_batch(B, m, step=cyc)
        ptr, ids = synth.label_batch(B, L, 5.0, step=cyc)
        lay.train_step(tens(h), tens(ptr), tens(ids), F32(1e-2))
        s0 = state_of(lay)
        lay.redistribute(1000 * (cyc + 1))
        s1 = state_of(lay)
        W2, idx2, m2, v2 = oracle.redistribute(s0["W"], s0["idx"], s0["mW"], s0["vW"], m, p, seed=23,
                                               step=1000 * (cyc + 1))
        assert (s1["idx"] == idx2).all() and (s1["W"] == W2).all(), cyc
        assert (s1["mW"] == m2).all() and (s1["vW"] == v2).all(), cyc
        changed = s1["idx"] != s0["idx"]
        assert (changed.sum(axis=1) == p).all(), cyc                          # exactly p regrown per row
        assert ((s1["idx"] >= 0) & (s1["idx"] < m)).all()
        assert all(len(set(r)) == k for r in s1["idx"])                       # k distinct
        assert (s1["W"][changed] == 0).all() and (s1["mW"][changed] == 0).all() and (s1["vW"][changed] == 0).all()
        keep = ~changed
        assert (s1["W"][keep].view(np.uint32) == s0["W"][keep].view(np.uint32)).all()   # survivors untouched
        for j in range(0, L, 7):                                              # sort-oracle check of the pruned set
            keys = sorted(range(k), key=lambda i: (np.float32(abs(s0["W"][j, i])), i))
            assert set(np.nonzero(changed[j])[0]) == set(keys[:p]), (cyc, j)
        # freshness (R10): a regrown index was not in the row before the call
        for j in range(0, L, 11):
            assert not (set(s1["idx"][j][changed[j]]) & set(s0["idx"][j])), (cyc, j)


def test_column_independence():
    """changing one label row's weights and indices changes that label's scores only
    (bit-exact for every other label), in the forward and in the fused step's state."""
    L, m, k, B = 2000, 512, 32, 32
    a = make(L, m, k, B=B, seed=31)
    b = make(L, m, k, B=B, seed=31)
    s = state_of(b)
    j0 = 777
    W, idx = s["W"].copy(), s["idx"].copy()
    W[j0] = -W[j0] * np.float32(1.5)
    idx[j0] = np.random.default_rng(3).choice(m, size=k, replace=False).astype(np.int32)
    b.set_params(W=tens(W), idx=tens(idx))
    h = tens(synth.hidden_batch(B, m, step=1))
    ya, yb = a.forward(h).cpu().numpy(), b.forward(h).cpu().numpy()
    other = np.arange(L) != j0
    assert (ya[:, other].view(np.uint32) == yb[:, other].view(np.uint32)).all()
    assert (ya[:, j0] != yb[:, j0]).any()
    ptr, ids = synth.label_batch(B, L, 5.0, step=1)
    a.train_step(h, tens(ptr), tens(ids), F32(1e-3))
    b.train_step(h, tens(ptr), tens(ids), F32(1e-3))
    sa, sb = state_of(a), state_of(b)
    for key in ("W", "mW", "vW", "bias", "mb", "vb"):
        assert (sa[key][other] == sb[key][other]).all(), key


@pytest.mark.parametrize("k", [16, 32, 48])
def test_redistribution_all_ties(k):
    """Rows whose |W| are all equal (incl. +-0): the p lowest slots are pruned (R9)."""
    L, m = 600, 1024
    lay = make(L, m, k, seed=5, prune_frac=0.1)
    W, idx, _ = synth.random_params(L, m, k, seed=4)
    W[::2, :] = 0.0
    W[1::4, :] = np.where(np.arange(k) % 2 == 0, 0.5, -0.5).astype(np.float32)
    W[3::8, ::3] = -0.0
    lay.set_params(W=tens(W), idx=tens(idx))
    lay.redistribute(1000)
    s = state_of(lay)
    z = np.zeros_like(W)
    p = int(np.floor(F32(0.1) * k))
    W2, idx2, _, _ = oracle.redistribute(W, idx, z, z, m, p, seed=5, step=1000)
    assert (s["idx"] == idx2).all() and (s["W"] == W2).all()
    pruned = (s["idx"] != idx)
    assert (pruned[::2].sum(axis=1) == p).all() and pruned[::2, :p].all()


def test_redistribution_config_errors():
    layer = L_()
    lay = make(100, 64, 8, prune_frac=0.05)          # floor(0.05*8) = 0
    with pytest.raises(layer.FFError) as e:
        lay.redistribute(1)
    assert e.value.status == layer.FF_ERR_CONFIG
    lay = make(100, 10, 10, prune_frac=0.2)          # m - k = 0 < p = 2
    with pytest.raises(layer.FFError):
        lay.redistribute(1)


# ------------------------------------------------------------------------- top-K
@pytest.mark.parametrize("L,m,k,B,K", [(1000, 256, 16, 32, 5), (5000, 512, 32, 70, 8), (9, 16, 4, 3, 1),
                                        (8, 16, 4, 3, 8), (3000, 4096, 64, 32, 5), (700, 500, 40, 50, 3),
                                        (4000, 1024, 32, 1024, 5),
                                        # k = 32, B <= 32: the pipelined predict kernel
                                        (5000, 512, 32, 32, 5), (3001, 300, 32, 7, 8), (40, 64, 32, 32, 8),
                                        (200003, 4096, 32, 32, 5),
                                        # k = 32, B > 32: the chunked wide kernel (ragged lines and chunks)
                                        (3001, 300, 32, 33, 8), (2000, 512, 32, 129, 5), (2500, 700, 32, 300, 3),
                                        (20011, 2048, 32, 1000, 8), (37, 64, 32, 64, 8)])
def test_predict_topk_bit_exact(L, m, k, B, K):
    lay = make(L, m, k, B=B, seed=3)
    h = tens(synth.hidden_batch(B, m, step=1))
    sc, ids = lay.predict_topk(h, K)
    y = lay.forward(h).cpu().numpy().astype(np.float64)
    rs, rid = oracle.topk(y, K)
    assert (ids.cpu().numpy() == rid).all()
    assert (sc.cpu().numpy() == rs).all()


def test_predict_topk_ties_resolved_by_lower_id():
    L, m, k, B = 300, 64, 8, 4
    lay = make(L, m, k, B=B)
    W = np.zeros((L, k), np.float32)
    bias = np.zeros(L, np.float32); bias[[17, 5, 250, 100]] = 1.0
    lay.set_params(W=tens(W), bias=tens(bias))
    sc, ids = lay.predict_topk(tens(synth.hidden_batch(B, m)), 6)
    assert (ids.cpu().numpy() == np.array([5, 17, 100, 250, 0, 1])).all()


def test_predict_topk_ties_resolved_by_lower_id_pipelined():
    L, m, k, B = 5000, 64, 32, 32          # k = 32, B <= 32: k_predict_ring + block merge
    lay = make(L, m, k, B=B)
    W = np.zeros((L, k), np.float32)
    bias = np.zeros(L, np.float32); bias[[4999, 17, 5, 2500, 100]] = 1.0
    lay.set_params(W=tens(W), bias=tens(bias))
    sc, ids = lay.predict_topk(tens(synth.hidden_batch(B, m)), 8)
    assert (ids.cpu().numpy() == np.array([5, 17, 100, 2500, 4999, 0, 1, 2])).all()


def test_predict_shared_thresholds_rearm_between_calls():
    """The ring kernel's shared per-sample thresholds are re-armed by each call's merge: calls
    with different batches and inputs in any order (B = 64, 16, 64 on other data, 300 on the
    wide path) give exactly the top-K of a fresh layer."""
    L, m, k, K = 6000, 512, 32, 5
    lay = make(L, m, k, B=300, seed=27)
    for B, step in ((64, 1), (16, 2), (64, 3), (300, 4), (32, 1)):
        h = tens(synth.hidden_batch(B, m, step=step))
        fresh = make(L, m, k, B=300, seed=27)
        s1, i1 = lay.predict_topk(h, K)
        s2, i2 = fresh.predict_topk(h, K)
        assert torch.equal(i1, i2) and torch.equal(s1, s2), (B, step)
        rs, rid = oracle.topk(lay.forward(h).cpu().numpy(), K)
        assert (i1.cpu().numpy() == rid).all(), (B, step)


@pytest.mark.parametrize("B", [70, 300])
def test_predict_topk_ties_resolved_by_lower_id_wide(B):
    L, m, k = 5000, 64, 32                 # k = 32, B > 32: k_predict_wide + block merge
    lay = make(L, m, k, B=B)
    W = np.zeros((L, k), np.float32)
    bias = np.zeros(L, np.float32); bias[[4999, 17, 5, 2500, 100]] = 1.0
    lay.set_params(W=tens(W), bias=tens(bias))
    sc, ids = lay.predict_topk(tens(synth.hidden_batch(B, m)), 8)
    assert (ids.cpu().numpy() == np.array([5, 17, 100, 2500, 4999, 0, 1, 2])).all()


@DH
@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_sharded_layers_are_p_invariant(P, dh_mode):
    """Virtual sharding on one GPU: P handles with row offsets reproduce the unsharded
    state, scores and (after merge) top-K bit-exactly (rows are independent)."""
    layer = L_()
    L, m, k, B, K = 2003, 512, 32, 32, 5
    full = make(L, m, k, B=B, seed=9, dh_mode=dh_mode)
    bounds = [L * r // P for r in range(P + 1)]
    shards = [make(bounds[r + 1] - bounds[r], m, k, B=B, seed=9, L_global=L, row_begin=bounds[r],
                   L_local=bounds[r + 1] - bounds[r], dh_mode=dh_mode) for r in range(P)]
    for step in range(2):
        h = tens(synth.hidden_batch(B, m, step=step))
        ptr, ids = synth.label_batch(B, L, 5.0, step=step)
        dh_full, _ = full.train_step(h, tens(ptr), tens(ids), 1e-3)
        dh_sum = sum(s.train_step(h, tens(ptr), tens(ids), 1e-3)[0] for s in shards)
        assert dh_close(dh_full, dh_sum)
    full.redistribute(1000)
    for s in shards:
        s.redistribute(1000)
    sf = state_of(full)
    cat = [state_of(s) for s in shards]
    for key in ("W", "idx", "bias", "mW", "vW"):
        assert (np.concatenate([c[key] for c in cat]) == sf[key]).all(), key
    h = tens(synth.hidden_batch(B, m, step=5))
    fs, fi = full.predict_topk(h, K)
    parts = [s.predict_topk(h, K) for s in shards]
    ms, mi = layer.merge_topk(torch.stack([p[0] for p in parts]), torch.stack([p[1] for p in parts]))
    assert torch.equal(mi, fi) and torch.equal(ms, fs)


@pytest.mark.parametrize("P,B", [(2, 64), (3, 100), (8, 300)])
def test_sharded_predict_is_p_invariant_large_batch(P, B):
    """Label shards (row_begin > 0) through the per-line ring (B <= 96) and the two-pass wide
    kernel (B > 96): merged shard top-K == the unsharded top-K, bit for bit."""
    layer = L_()
    L, m, k, K = 4001, 512, 32, 8
    full = make(L, m, k, B=B, seed=19)
    bounds = [L * r // P for r in range(P + 1)]
    shards = [make(bounds[r + 1] - bounds[r], m, k, B=B, seed=19, L_global=L, row_begin=bounds[r],
                   L_local=bounds[r + 1] - bounds[r]) for r in range(P)]
    h = tens(synth.hidden_batch(B, m, step=6))
    fs, fi = full.predict_topk(h, K)
    parts = [s.predict_topk(h, K) for s in shards]
    ms, mi = layer.merge_topk(torch.stack([p[0] for p in parts]), torch.stack([p[1] for p in parts]))
    assert torch.equal(mi, fi) and torch.equal(ms, fs)


# ------------------------------------------------------------------- edge cases
def test_label_id_out_of_range_reported():
    layer = L_()
    lay = make(100, 64, 8, B=2)
    h = tens(synth.hidden_batch(2, 64))
    ptr = np.array([0, 1, 2], np.int32); ids = np.array([5, 100], np.int32)
    lay.train_step(h, tens(ptr), tens(ids), 1e-3)
    with pytest.raises(layer.FFError) as e:
        lay.check()
    assert e.value.status == layer.FF_ERR_RANGE
    lay.check()                                           # cleared


def test_set_params_rejects_bad_idx():
    layer = L_()
    lay = make(10, 64, 4)
    idx = np.tile(np.arange(4, dtype=np.int32), (10, 1)); idx[3, 2] = idx[3, 0]
    with pytest.raises(layer.FFError) as e:
        lay.set_params(idx=tens(idx))
    assert e.value.status == layer.FF_ERR_RANGE
    idx[3, 2] = 64
    with pytest.raises(layer.FFError):
        lay.set_params(idx=tens(idx))


@DH
def test_empty_batch_and_empty_shard(dh_mode):
    L, m, k = 50, 32, 4
    lay = make(L, m, k, B=8, seed=1, dh_mode=dh_mode)
    s0 = state_of(lay)
    h = torch.zeros((0, m), device=dev())
    y = lay.forward(h)
    assert y.shape == (0, L)
    ptr = tens(np.zeros(1, np.int32)); ids = tens(np.zeros(1, np.int32))
    lay.train_step(h, ptr, ids, 1e-3)                     # no samples: zero gradients, Adam still steps
    s1 = state_of(lay)
    Wr, _, _ = oracle.adam(s0["W"], np.zeros((L, k)), s0["mW"], s0["vW"], 1, F32(1e-3), **ADAM)
    assert_close(s1["W"], Wr, adam_A(s0["W"], Wr), "W' with B=0")
    assert s1["t"] == 1
    empty = make(0, m, k, B=8, L_global=10, row_begin=10, L_local=0, dh_mode=dh_mode)
    hb = tens(synth.hidden_batch(3, m))
    dh, _ = empty.train_step(hb, tens(np.array([0, 0, 0, 0], np.int32)), ids, 1e-3)
    assert (dh == 0).all()


def test_full_fan_in_is_dense():
    L, m, B = 40, 16, 8
    lay = make(L, m, m, B=B)
    rng = np.random.default_rng(0)
    idx = np.stack([rng.permutation(m) for _ in range(L)]).astype(np.int32)
    Wd = rng.standard_normal((m, L)).astype(np.float32)
    W = np.take_along_axis(Wd.T, idx, axis=1)
    lay.set_params(W=tens(np.ascontiguousarray(W)), idx=tens(idx), bias=tens(np.zeros(L, np.float32)))
    h = synth.hidden_batch(B, m)
    y = lay.forward(tens(h)).cpu().numpy()
    ref = h.astype(np.float64) @ Wd.astype(np.float64)
    assert np.abs(y - ref).max() <= 1e-4 * np.abs(h).sum(1).max() * np.abs(Wd).max()


@DH
def test_host_entry_point_equals_device_entry_point(dh_mode):
    L, m, k, B = 1000, 256, 16, 32
    a, b = make(L, m, k, B=B, seed=4, dh_mode=dh_mode), make(L, m, k, B=B, seed=4, dh_mode=dh_mode)
    h = synth.hidden_batch(B, m, step=2)
    ptr, ids = synth.label_batch(B, L, 5.0, step=2)
    dh_host = torch.empty((B, m)).pin_memory(); loss_host = torch.empty(1).pin_memory()
    a.train_step_host(torch.from_numpy(h).pin_memory(), torch.from_numpy(ptr), torch.from_numpy(ids), 1e-3,
                      dh_host=dh_host, loss_host=loss_host)
    loss = torch.zeros(1, device=dev())
    dh, _ = b.train_step(tens(h), tens(ptr), tens(ids), 1e-3, loss=loss)
    torch.cuda.synchronize()
    assert dh_close(dh_host, dh.cpu())
    assert abs(loss_host.item() - loss.item()) <= 1e-5 * loss.item()
    sa, sb = state_of(a), state_of(b)
    assert (sa["W"] == sb["W"]).all() and (sa["bias"] == sb["bias"]).all()


@DH
def test_host_entry_point_double_buffering_over_many_steps(dh_mode):
    """train_step_host stages into two alternating slots on its own copy stream: a run of
    host-entry steps with different batches (no synchronisation in between) leaves exactly
    the state of the same run through the device entry point."""
    L, m, k, B = 3000, 512, 32, 32
    a, b = make(L, m, k, B=B, seed=6, dh_mode=dh_mode), make(L, m, k, B=B, seed=6, dh_mode=dh_mode)
    hs = [torch.from_numpy(synth.hidden_batch(B, m, step=s)).pin_memory() for s in range(5)]
    lb = [synth.label_batch(B, L, 5.0, step=s) for s in range(5)]
    loss_host = torch.empty(1).pin_memory()
    for s in range(5):
        a.train_step_host(hs[s], torch.from_numpy(lb[s][0]), torch.from_numpy(lb[s][1]), 1e-3, loss_host=loss_host)
    for s in range(5):
        b.train_step(hs[s].to(dev()), tens(lb[s][0]), tens(lb[s][1]), 1e-3)
    torch.cuda.synchronize()
    sa, sb = state_of(a), state_of(b)
    for key in ("W", "bias", "mW", "vW", "idx"):
        assert (sa[key] == sb[key]).all(), key


@pytest.mark.parametrize("pinned", [True, False])
def test_host_entry_point_loss_output(pinned):
    """The loss of every host-entry step reaches host memory: page-locked (kernel store into
    mapped memory) or pageable (cudaMemcpyAsync); dh_host = None skips only the copy-out."""
    L, m, k, B = 2000, 512, 32, 32
    a, b = make(L, m, k, B=B, seed=8), make(L, m, k, B=B, seed=8)
    loss_host = torch.empty(1).pin_memory() if pinned else torch.empty(1)
    loss = torch.zeros(1, device=dev())
    for s in range(4):
        h = synth.hidden_batch(B, m, step=s)
        ptr, ids = synth.label_batch(B, L, 5.0, step=s)
        loss_host.fill_(-1.0)
        a.train_step_host(torch.from_numpy(h).pin_memory(), torch.from_numpy(ptr), torch.from_numpy(ids), 1e-3,
                          loss_host=loss_host)
        b.train_step(tens(h), tens(ptr), tens(ids), 1e-3, loss=loss)
        torch.cuda.synchronize()
        assert abs(loss_host.item() - loss.item()) <= 1e-5 * loss.item(), s
    sa, sb = state_of(a), state_of(b)
    assert (sa["W"] == sb["W"]).all() and (sa["vW"] == sb["vW"]).all()


@DH
def test_train_step_cuda_graph_replay(dh_mode):
    """The fused step is capturable: it only enqueues kernels on the caller's stream, and the
    Adam step counter lives on the device (k_prep advances it), so N replays of one captured
    step (inputs copied into static buffers) equal N eager steps bit for bit, t included, with
    a redistribution between replays."""
    L, m, k, B = 3000, 512, 32, 32
    a, b = make(L, m, k, B=B, seed=6, dh_mode=dh_mode), make(L, m, k, B=B, seed=6, dh_mode=dh_mode)
    batches = [synth.label_batch(B, L, 5.0, step=s) for s in range(6)]
    hs = [tens(synth.hidden_batch(B, m, step=s)) for s in range(6)]
    nnz_max = max(int(p_[-1]) for p_, _ in batches)
    sh, sp = torch.zeros((B, m), device=dev()), torch.zeros(B + 1, dtype=torch.int32, device=dev())
    si = torch.zeros(nnz_max, dtype=torch.int32, device=dev())
    sdh, sloss = torch.empty((B, m), device=dev()), torch.zeros(1, device=dev())

    def load(s):
        sh.copy_(hs[s]); sp.copy_(tens(batches[s][0])); si[:len(batches[s][1])].copy_(tens(batches[s][1]))

    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):                      # one eager step before capture (torch's rule)
        load(0)
        a.train_step(sh, sp, si, 1e-3, dh=sdh, loss=sloss)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        a.train_step(sh, sp, si, 1e-3, dh=sdh, loss=sloss)
    # the capture did not run the step: a has taken exactly one step (t = 1)
    losses_g = []
    for s in range(1, 6):
        load(s)
        g.replay()
        losses_g.append(sloss.clone())
        if s == 3:
            a.redistribute(1000)
    loss_e = torch.zeros(1, device=dev())
    losses_e = []
    for s in range(6):
        dh_e, _ = b.train_step(hs[s], tens(batches[s][0]), tens(batches[s][1]), 1e-3, loss=loss_e)
        if s > 0:
            losses_e.append(loss_e.clone())
        if s == 3:
            b.redistribute(1000)
    torch.cuda.synchronize()
    sa, sb = state_of(a), state_of(b)
    assert sa["t"] == sb["t"] == 6
    for key in ("W", "bias", "mW", "vW", "idx", "mb", "vb"):
        assert (sa[key] == sb[key]).all(), key
    if dh_mode == 1:                                   # CSC: deterministic dh order
        assert torch.equal(sdh, dh_e)
    else:                                              # atomic reductions: order-dependent rounding
        assert dh_close(sdh.cpu(), dh_e.cpu())
    # the loss is an fp32 sum of per-block partials added by atomics in arrival order (every
    # dh mode): replay and eager agree to summation-order rounding, bounded well inside R19
    assert all(abs(x.item() - y.item()) <= 1e-5 * abs(y.item()) for x, y in zip(losses_g, losses_e))


def test_csc_dh_is_deterministic_and_matches_atomic():
    L, m, k, B = 3000, 1024, 32, 32
    a, b = make(L, m, k, B=B, seed=2, dh_mode=1), make(L, m, k, B=B, seed=2, dh_mode=0)
    h = tens(synth.hidden_batch(B, m, step=1))
    ptr, ids = synth.label_batch(B, L, 5.0, step=1)
    W, idx, bias = synth.random_params(L, m, k, seed=3)
    for x in (a, b):
        x.set_params(W=tens(W), idx=tens(idx), bias=tens(bias))
    y = a.forward(h)
    d1, _ = a.backward(h, y, tens(ptr), tens(ids))
    d2, _ = a.backward(h, y, tens(ptr), tens(ids))
    assert torch.equal(d1, d2)
    d3, _ = b.backward(h, y, tens(ptr), tens(ids))
    assert dh_close(d1, d3)


@pytest.mark.parametrize("shape_name,dh_modes,loss", [("wiki10-31k", (0,), "bce"), ("wiki-500k", (0,), "bce"),
                                                       ("amazon-670k", (1, 0, 2), "bce"), ("amazon-3m", (1, 0), "bce"),
                                                       ("amazon-670k-k64-m65k", (0, 1), "bce"),
                                                       ("amazon-670k", (0, 1), "sqh")])
def test_full_size_sampled_parity(shape_name, dh_modes, loss):
    """BASELINE.json's shapes in the bench's launch configuration: one fused step checked on
    sampled label rows (y, dW, db, W') and on the full dh (the oracle's Alg. 2 over every
    connection), lockstep (R20); the squared hinge (the paper's loss, with its exact-zero
    skips) at Amazon-670K as well, its margin decisions taken on the kernel's y."""
    layer = L_()
    shape = synth.SHAPES[shape_name]
    L, m, k, B = shape.L, shape.m, shape.k, shape.B
    h = synth.hidden_batch(B, m, step=0)
    ptr, ids = synth.label_batch(B, L, shape.avg_pos, step=0)
    rng = np.random.default_rng(5)
    rows = np.sort(rng.choice(L, 256, replace=False))
    for dh_mode in dh_modes:
        lay = make(L, m, k, B=B, seed=42, flags=layer.FF_FLAG_STORE_GRADS, dh_mode=dh_mode, loss=loss_id(loss))
        s0 = state_of(lay)
        y = lay.forward(tens(h)).cpu().numpy().astype(np.float64)
        dh, _ = lay.train_step(tens(h), tens(ptr), tens(ids), F32(1e-3))
        dW, db = (x.cpu().numpy() for x in lay.get_grads())
        s1 = state_of(lay)
        yr, Ay = oracle.forward(s0["W"][rows], s0["idx"][rows], s0["bias"][rows], h)
        assert_close(y[:, rows], yr, Ay, "y rows")
        g, _ = oracle.loss_grad(loss, y, ptr, ids, F32(1.0 / B))
        dWr, AdW, dbr, Adb = oracle.weight_grad(s0["idx"][rows], h, g[:, rows])
        assert_close(dW[rows], dWr, AdW, "dW rows")
        assert_close(db[rows], dbr, Adb, "db rows")
        Wr, mr, vr = oracle.adam(s0["W"][rows], dW[rows], s0["mW"][rows], s0["vW"][rows], 1, F32(1e-3), **ADAM)
        assert_close(s1["W"][rows], Wr, adam_A(s0["W"][rows], Wr), "W' rows")
        dhr, Adh = oracle.input_grad(s0["W"], s0["idx"], g, m)
        assert_close(dh.cpu().numpy(), dhr, Adh, f"dh full (mode {dh_mode})")
        del lay
        torch.cuda.empty_cache()


def test_csc_multi_tile_dh_and_grads():
    """CSC mode with several label tiles (B = 100 -> 4 sample chunks -> 65,536-row tiles):
    the per-tile column passes accumulate dh across tiles; compared with the oracle."""
    layer = L_()
    L, m, k, B = 140000, 2048, 32, 100
    lay = make(L, m, k, B=128, seed=6, dh_mode=1, flags=layer.FF_FLAG_STORE_GRADS)
    s0 = state_of(lay)
    h = synth.hidden_batch(B, m, step=2)
    ptr, ids = synth.label_batch(B, L, 5.0, step=2)
    y = lay.forward(tens(h)).cpu().numpy().astype(np.float64)
    dh, _ = lay.train_step(tens(h), tens(ptr), tens(ids), F32(1e-3))
    dW, db = (x.cpu().numpy() for x in lay.get_grads())
    g, _ = oracle.bce_grad(y, ptr, ids, F32(1.0 / B))
    dhr, Adh = oracle.input_grad(s0["W"], s0["idx"], g, m)
    assert_close(dh.cpu().numpy(), dhr, Adh, "dh (3 tiles)")
    rows = np.arange(0, L, 997)
    dWr, AdW, dbr, Adb = oracle.weight_grad(s0["idx"][rows], h, g[:, rows])
    assert_close(dW[rows], dWr, AdW, "dW rows")
    assert_close(db[rows], dbr, Adb, "db rows")


@LOSS
@DH
@pytest.mark.parametrize("L,m,B", [(5000, 1024, 32), (1234, 700, 19), (31, 64, 32), (70000, 4096, 32),
                                   # B <= 16: padded samples in every line
                                   (5000, 1024, 16), (1234, 700, 9), (33, 64, 1), (70000, 4096, 13)])
def test_pipelined_step_equals_generic_step(L, m, B, dh_mode, loss):
    """k = 32, B <= 32 runs the software-pipelined fused kernel (cp.async shared-memory ring);
    FF_FLAG_NO_PIPE forces the generic one.  Both implement the same arithmetic: state and
    gradients bit-identical."""
    layer = L_()
    k = 32
    flags = layer.FF_FLAG_STORE_GRADS
    a = make(L, m, k, B=B, seed=12, flags=flags, dh_mode=dh_mode, loss=loss_id(loss))
    b = make(L, m, k, B=B, seed=12, flags=flags | layer.FF_FLAG_NO_PIPE, dh_mode=dh_mode, loss=loss_id(loss))
    for step in range(3):
        h = tens(synth.hidden_batch(B, m, step=step))
        ptr, ids = synth.label_batch(B, L, 5.0, step=step)
        la, lb = torch.zeros(1, device=dev()), torch.zeros(1, device=dev())
        dha, _ = a.train_step(h, tens(ptr), tens(ids), 1e-2, loss=la)
        dhb, _ = b.train_step(h, tens(ptr), tens(ids), 1e-2, loss=lb)
        ga, gb = a.get_grads(), b.get_grads()
        assert torch.equal(ga[0], gb[0]) and torch.equal(ga[1], gb[1])
        sa, sb = state_of(a), state_of(b)
        for key in ("W", "mW", "vW", "bias", "mb", "vb", "idx"):
            assert (sa[key] == sb[key]).all(), key
        if dh_mode == 1:
            assert torch.equal(dha, dhb)
        else:
            assert dh_close(dha, dhb)
        assert abs(la.item() - lb.item()) <= 1e-5 * abs(lb.item())



@DH
@pytest.mark.parametrize("k,B", [(32, 32), (32, 20), (16, 32), (13, 40)])
def test_sqh_implicit_negative_mining_skips_are_exact(dh_mode, k, B):
    """Engineered margins (bias = -3): most negatives meet the margin, so most of the
    squared-hinge gradient is exactly zero and the kernels skip that work.
    Skipping must not change anything: dW rows whose gradient column is all zero are
    exactly 0, and dh / dW / W' match the oracle, which never skips."""
    layer = L_()
    L, m = 4000, 1024
    lay = make(L, m, k, B=max(B, 32), seed=31, dh_mode=dh_mode, loss=layer.FF_LOSS_SQH,
               flags=layer.FF_FLAG_STORE_GRADS)
    W, idx, _ = synth.random_params(L, m, k, seed=4, scale=0.3)
    bias = np.full(L, -3.0, np.float32)
    lay.set_params(W=tens(W), idx=tens(idx), bias=tens(bias))
    h = synth.hidden_batch(B, m, step=7)
    ptr, ids = synth.label_batch(B, L, 5.0, step=7)
    y = lay.forward(tens(h)).cpu().numpy().astype(np.float64)
    loss = torch.zeros(1, device=dev())
    dh, _ = lay.train_step(tens(h), tens(ptr), tens(ids), F32(1e-3), loss=loss)
    dW, db = (x.cpu().numpy() for x in lay.get_grads())
    g, lref = oracle.sqh_grad(y, ptr, ids, F32(1.0 / B))
    zero_cols = (g == 0).all(axis=0)
    assert zero_cols.mean() > 0.5                      # the skip really happens
    assert (dW[zero_cols] == 0).all() and (db[zero_cols] == 0).all()
    dWr, AdW, dbr, Adb = oracle.weight_grad(idx, h, g)
    dhr, Adh = oracle.input_grad(W, idx, g, m)
    assert_close(dW, dWr, AdW, "dW")
    assert_close(db, dbr, Adb, "db")
    assert_close(dh.cpu().numpy(), dhr, Adh, "dh")
    assert abs(loss.item() - lref) <= RTOL * lref


# ---------------------------------------------------------- shortlist scoring (NEXT-3)
def _shortlist(B, L_global, n, seed):
    """CSR shortlist: n candidates per instance (some repeated), sorted per instance."""
    r = np.random.default_rng(seed)
    ptr = np.arange(B + 1, dtype=np.int32) * n
    ids = np.concatenate([np.sort(r.integers(0, L_global, size=n)) for _ in range(B)]).astype(np.int32) \
        if B * n else np.zeros(0, np.int32)
    return ptr, ids


@pytest.mark.parametrize("L,m,k,B,n", [(1000, 256, 16, 32, 40), (5000, 1024, 32, 70, 100), (400, 300, 50, 9, 33),
                                        (3000, 4096, 64, 32, 17), (333, 100, 13, 5, 200), (97, 64, 1, 3, 5)])
def test_shortlist_scores_parity_and_bit_exact_vs_forward(L, m, k, B, n):
    """P:1057-1059 (R24): shortlist scores match the oracle within R19 and equal the
    forward's score of the same (instance, label) bit for bit."""
    lay = make(L, m, k, B=min(B, 128), seed=5)
    W, idx, bias = synth.random_params(L, m, k, seed=L + k)
    lay.set_params(W=tens(W), idx=tens(idx), bias=tens(bias))
    h = synth.hidden_batch(B, m, step=2)
    ptr, ids = _shortlist(B, L, n, seed=L + n)
    sc = lay.score_shortlist(tens(h), tens(ptr), tens(ids)).cpu().numpy()
    p = state_of(lay)
    yr, Ay = oracle.score_shortlist(p["W"], p["idx"], p["bias"], h, ptr, ids)
    assert_close(sc, yr, Ay, "shortlist")
    y = lay.forward(tens(h)).cpu().numpy()
    b_of = np.repeat(np.arange(B), np.diff(ptr))
    assert np.array_equal(sc.view(np.uint32), y[b_of, ids].view(np.uint32))


def test_shortlist_sharded_sum_and_errors():
    """Labels owned by another shard score +0, so the shards' outputs sum to the unsharded
    result; an id outside [0, L_global) is NaN and reported by check(); empty lists."""
    layer = L_()
    L, m, k, B = 1000, 256, 16, 6
    full = make(L, m, k, B=B, seed=9)
    sh = [make(500, m, k, B=B, seed=9, L_global=L, row_begin=r, L_local=500) for r in (0, 500)]
    p = full.get_params()
    for r, s in zip((0, 500), sh):
        s.set_params(**{key: v[r:r + 500] for key, v in p.items() if torch.is_tensor(v) and v.shape[0] == L})
    h = tens(synth.hidden_batch(B, m, step=4))
    ptr = np.array([0, 3, 3, 5, 9, 9, 12], np.int32)
    ids = np.array([0, 499, 500, 7, 999, 1, 2, 3, 4, 998, 500, 501], np.int32)
    ref = full.score_shortlist(h, tens(ptr), tens(ids))
    parts = [s.score_shortlist(h, tens(ptr), tens(ids)) for s in sh]
    assert torch.equal(parts[0] + parts[1], ref)
    assert (parts[0][torch.from_numpy(ids >= 500).to(dev())] == 0).all()
    bad = np.array([0, 1, 1, 1, 1, 1, 1], np.int32)
    out = full.score_shortlist(h, tens(bad), tens(np.array([L], np.int32)))
    assert torch.isnan(out).all()
    with pytest.raises(layer.FFError) as e:
        full.check()
    assert e.value.status == layer.FF_ERR_RANGE
    empty = full.score_shortlist(h, tens(np.zeros(B + 1, np.int32)), tens(np.zeros(0, np.int32)))
    assert empty.numel() == 0
    full.check()


@pytest.mark.parametrize("B,K,npos", [(32, 5, 5.0), (7, 1, 1.0), (100, 8, 40.0), (0, 3, 2.0)])
def test_precision_at_k_matches_oracle(B, K, npos):
    """Eq. (1) on the GPU: per-instance hits bit-exact, the mean within fp32
    rounding, for top-K lists that mix positives and negatives (and > 32 positives)."""
    layer = L_()
    L, m, k = 3000, 256, 16
    if B == 0:
        hits, mean = layer.precision_at_k(torch.empty((0, K), dtype=torch.int32, device=dev()),
                                          torch.zeros(1, dtype=torch.int32, device=dev()),
                                          torch.zeros(1, dtype=torch.int32, device=dev()))
        assert mean.item() == 0.0
        return
    lay = make(L, m, k, B=min(B, 1024), seed=5)
    ptr, ids = synth.label_batch(B, L, npos, step=2)
    h = synth.hidden_batch(B, m, step=2)
    _, top = lay.predict_topk(tens(h), K)
    top = top.cpu().numpy()
    # plant some positives into the predictions so that hits are not all zero
    for b in range(0, B, 2):
        pos = ids[ptr[b]:ptr[b + 1]]
        top[b, : min(len(pos), K) // 2 + 1] = pos[: min(len(pos), K) // 2 + 1]
    hits, mean = layer.precision_at_k(tens(top.astype(np.int32)), tens(ptr), tens(ids))
    ref_h = np.array([sum(int(t in set(ids[ptr[b]:ptr[b + 1]].tolist())) for t in top[b]) for b in range(B)])
    assert (hits.cpu().numpy() == ref_h).all()
    ref = oracle.precision_at_k(top.astype(np.int64), ptr, ids)
    assert abs(mean.item() - ref) <= 1e-6 * max(ref, 1e-30)


# ------------------------------------------- top-K against the fp64 oracle (gap-guarded)
def _topk_gap_guarded(ids_gpu, y64, Ay, K):
    """SURVEY §8(c).2 #20 against the fp64 scores.  With s_0 >= s_1 >= ... the oracle's
    ordered scores of a sample and tol_r = 1e-4 (A_r + A_{r+1}) the R19 bound of two
    neighbours: where the K-th / (K+1)-th gap exceeds tol the GPU's top-K id SET equals the
    oracle's top-K of the fp64 y, and every rank r whose gaps to both neighbours exceed their
    tol holds the oracle's id exactly.  A sample where any of these gaps is within tol is a
    near-tie: counted, and its ids must still be a valid top-K (every returned score within
    the bound of the oracle's K-th, K distinct ids).  Returns the number of near-tie samples."""
    _, oid = oracle.topk(y64, K + 1)
    near = 0
    for b in range(y64.shape[0]):
        o = oid[b]
        s = y64[b, o]
        sep = s[:-1] - s[1:] > 1e-4 * (Ay[b, o[:-1]] + Ay[b, o[1:]])      # gap r / r+1 is unambiguous
        if sep[K - 1]:
            assert set(ids_gpu[b].tolist()) == set(o[:K].tolist()), f"sample {b}: {ids_gpu[b]} vs {o[:K]}"
        for r in range(K):
            if sep[r] and (r == 0 or sep[r - 1]):
                assert ids_gpu[b, r] == o[r], f"sample {b} rank {r}: {ids_gpu[b]} vs fp64 top-K {o[:K]}"
        if not sep.all():
            near += 1
            kth = s[K - 1] - 1e-4 * Ay[b, o[K - 1]]
            assert (y64[b, ids_gpu[b]] + 1e-4 * Ay[b, ids_gpu[b]] >= kth).all(), f"sample {b}: invalid top-K"
            assert len(set(ids_gpu[b].tolist())) == K
    return near


@pytest.mark.parametrize("L,m,k,B,K", [(5000, 512, 32, 32, 5), (3001, 300, 32, 7, 8), (4000, 1024, 16, 70, 5),
                                        (2000, 4096, 64, 32, 3), (200003, 4096, 32, 32, 5), (3000, 1024, 32, 1024, 5)])
def test_predict_topk_vs_fp64_oracle_gap_guarded(L, m, k, B, K):
    lay = make(L, m, k, B=B, seed=13)
    h = synth.hidden_batch(B, m, step=11)
    _, ids = lay.predict_topk(tens(h), K)
    s = state_of(lay)
    y64, Ay = oracle.forward(s["W"], s["idx"], s["bias"], h)      # fp64 scores of the GPU's params
    near = _topk_gap_guarded(ids.cpu().numpy(), y64, Ay, K)
    print(f"top-{K} vs fp64 oracle: {B - near} of {B} samples without a near-tie, {near} near-ties")
    assert near <= max(2, B // 4)           # sanity: ties within the 1e-4 bound stay a minority


@pytest.mark.parametrize("B", [32, 64, 160])
def test_predict_topk_vs_fp64_oracle_full_amazon_670k(B):
    """BASELINE.json's Amazon-670K shape in the bench's predict configuration (k = 32, the
    ring kernel at B = 32 and, per 32-sample line, at B = 64; the two-pass wide kernel at
    B = 160: one full 128-sample chunk and a ragged one), after one training step so that bias
    and W are not at init.  Checked against the fp64 oracle (gap-guarded) and bit-exactly
    against the oracle's top-K of the GPU's own forward scores."""
    shape = synth.SHAPES["amazon-670k"]
    L, m, k = shape.L, shape.m, shape.k
    lay = make(L, m, k, B=max(B, shape.B), seed=42)
    ptr, lid = synth.label_batch(B, L, shape.avg_pos, step=0)
    lay.train_step(tens(synth.hidden_batch(B, m, step=0)), tens(ptr), tens(lid), F32(1e-3))
    h = synth.hidden_batch(B, m, step=3)
    sc, ids = lay.predict_topk(tens(h), 5)
    rs, rid = oracle.topk(lay.forward(tens(h)).cpu().numpy(), 5)            # bit-exact: same fp32 y
    assert (ids.cpu().numpy() == rid).all() and (sc.cpu().numpy() == rs).all()
    s = state_of(lay)
    y64, Ay = oracle.forward(s["W"], s["idx"], s["bias"], h)
    near = _topk_gap_guarded(ids.cpu().numpy(), y64, Ay, 5)
    print(f"Amazon-670K top-5 vs fp64 oracle: {B - near} of {B} samples without a near-tie, {near} near-ties")
    assert near <= B // 4


# ------------------------------------------- saturated-logit BCE regime, signed h (R5)
SAT_BIAS = np.array([-60.0, -25.0, 0.0, 25.0, 60.0], np.float32)


@LOSS
@DH
@pytest.mark.parametrize("k,B", [(32, 32), (16, 32), (32, 20), (13, 40), (32, 12)])
def test_saturated_logits_and_signed_h_lockstep(dh_mode, loss, k, B):
    """biases of +-25 and +-60 with positives and negatives on each, W scale 2
    and signed (non-ReLU) h, so that y reaches |y| ~ 65.  For a positive with y >~ 17 the naive
    fp32 sigma(y) - 1 is exactly 0 while the true gradient is -s sigma(-y) ~ 1e-26 (R5): dW,
    db (sums of such terms) and the loss are compared with the oracle at R19, the Adam state
    in lockstep, the update directly.  Runs the pipelined (k = 32, B <= 32) and generic kernels."""
    layer = L_()
    L, m = 1500, 512
    lay = make(L, m, k, B=max(B, 32), seed=17, dh_mode=dh_mode, loss=loss_id(loss), flags=layer.FF_FLAG_STORE_GRADS)
    W, idx, _ = synth.random_params(L, m, k, seed=21, scale=2.0)
    bias = SAT_BIAS[np.arange(L) % len(SAT_BIAS)]
    lay.set_params(W=tens(W), idx=tens(idx), bias=tens(bias))
    h = synth.signed_hidden_batch(B, m, step=3)
    ptr, ids = synth.random_labels_uniform(B, L, 60, seed=5)      # ~60 positives per sample: every bias class
    st = oracle.State(W.astype(np.float64), idx, bias.astype(np.float64), np.zeros((L, k)), np.zeros((L, k)),
                      np.zeros(L), np.zeros(L), 0)
    y = lay.forward(tens(h)).cpu().numpy()
    loss_t = torch.zeros(1, device=dev())
    dh, _ = lay.train_step(tens(h), tens(ptr), tens(ids), F32(1e-3), loss=loss_t)
    dW, db = (x.cpu().numpy() for x in lay.get_grads())
    r = oracle.train_step(st, h, ptr, ids, F32(1.0 / B), F32(1e-3), loss=loss, **ADAM)
    assert np.abs(r.y).max() > 40                                  # the saturated regime is reached
    posmask = np.zeros((B, L), bool)
    for b in range(B):
        posmask[b, ids[ptr[b]:ptr[b + 1]]] = True
    if loss == "bce":
        sat_pos = posmask & (r.y > 17)                             # sigma(y) - 1 == 0 in fp32 here
        assert sat_pos.sum() > 50 and (r.g[sat_pos] != 0).all()
    assert_close(y, r.y, r.Ay, "y")
    assert_close(dW, r.dW, r.AdW, "dW")
    assert_close(db, r.db, r.Adb, "db")
    assert_close(dh.cpu().numpy(), r.dh, r.Adh, "dh")
    assert abs(loss_t.item() - r.loss) <= RTOL * abs(r.loss)
    s1 = state_of(lay)
    Wr, mr, vr = oracle.adam(W, dW, np.zeros((L, k)), np.zeros((L, k)), 1, F32(1e-3), **ADAM)
    br, mbr, vbr = oracle.adam(bias, db, np.zeros(L), np.zeros(L), 1, F32(1e-3), **ADAM)
    assert_close(s1["W"], Wr, adam_A(W, Wr), "W'")
    assert_close(s1["mW"], mr, 0, "mW'")
    assert_close(s1["vW"], vr, 1e-30, "vW'")
    assert_close(s1["bias"], br, adam_A(bias, br), "bias'")
    assert_adam_update(W, s1["W"], Wr, "W update")
    assert_adam_update(bias, s1["bias"], br, "bias update")


# ------------------------------------------------------------ FF_FLAG_CHECK_FINITE
@DH
@pytest.mark.parametrize("k,B", [(32, 32), (16, 32), (32, 100), (32, 8)])
@pytest.mark.parametrize("bad", [np.inf, -np.inf, np.nan])
def test_check_finite_reports_nonfinite_scores(dh_mode, k, B, bad):
    """with FF_FLAG_CHECK_FINITE a non-finite score (an inf / NaN in h reaches
    every label connected to that column) raises FF_ERR_NONFINITE at the next check(), which
    clears it; without the flag the same step reports nothing."""
    layer = L_()
    L, m = 2000, 256
    h = synth.hidden_batch(B, m, step=1)
    h[B // 2, 17] = bad
    ptr, ids = synth.label_batch(B, L, 5.0, step=1)
    flagged = make(L, m, k, B=B, seed=3, dh_mode=dh_mode, flags=layer.FF_FLAG_CHECK_FINITE)
    plain = make(L, m, k, B=B, seed=3, dh_mode=dh_mode)
    flagged.train_step(tens(h), tens(ptr), tens(ids), F32(1e-3))
    with pytest.raises(layer.FFError) as e:
        flagged.check()
    assert e.value.status == layer.FF_ERR_NONFINITE
    flagged.check()                                                # cleared
    plain.train_step(tens(h), tens(ptr), tens(ids), F32(1e-3))
    plain.check()
    hf = synth.hidden_batch(B, m, step=2)                          # finite input: no report
    flagged.train_step(tens(hf), tens(ptr), tens(ids), F32(1e-3))
    # (the previous step left non-finite weights in the rows that saw the inf: fresh layer)
    fresh = make(L, m, k, B=B, seed=3, dh_mode=dh_mode, flags=layer.FF_FLAG_CHECK_FINITE)
    fresh.train_step(tens(hf), tens(ptr), tens(ids), F32(1e-3))
    fresh.check()
    y = fresh.forward(tens(hf))
    fresh.backward(tens(h), y, tens(ptr), tens(ids))              # unfused backward: y finite, h not
    fresh.check()                                                  # scores are checked, finite here
    y[B // 2, 5] = bad
    fresh.backward(tens(hf), y, tens(ptr), tens(ids))
    with pytest.raises(layer.FFError) as e:
        fresh.check()
    assert e.value.status == layer.FF_ERR_NONFINITE


@pytest.mark.parametrize("B", [32, 64, 300])
def test_check_finite_reports_nonfinite_predict_scores(B):
    """R15 / SURVEY c.2 #15: with FF_FLAG_CHECK_FINITE a NaN score seen by the predict kernels
    (ring, per-line ring, wide) raises FF_ERR_NONFINITE at the next check(); the NaN label never
    enters the top K, and without the flag nothing is reported."""
    layer = L_()
    L, m, k = 3000, 256, 32
    flagged = make(L, m, k, B=B, seed=4, flags=layer.FF_FLAG_CHECK_FINITE)
    plain = make(L, m, k, B=B, seed=4)
    bias = np.zeros(L, np.float32); bias[1234] = np.nan
    for lay in (flagged, plain):
        lay.set_params(bias=tens(bias))
    h = tens(synth.hidden_batch(B, m, step=2))
    _, ids = flagged.predict_topk(h, 5)
    with pytest.raises(layer.FFError) as e:
        flagged.check()
    assert e.value.status == layer.FF_ERR_NONFINITE
    assert not (ids.cpu().numpy() == 1234).any()
    plain.predict_topk(h, 5)
    plain.check()


# ------------------------------------------- redistribution with more than 32 pruned slots
@pytest.mark.parametrize("L,m,k,frac", [(500, 4096, 64, 0.6), (300, 200, 64, 0.99), (400, 1000, 48, 0.8)])
def test_redistribution_more_than_32_pruned_slots(L, m, k, frac):
    """p = floor(frac k) up to 63 (k = 64): the regrow draws beyond the 32nd are held
    in a second register per lane; bit-exact vs the oracle and k distinct indices per row."""
    lay = make(L, m, k, seed=19, prune_frac=frac)
    W, idx, _ = synth.random_params(L, m, k, seed=8)
    rng = np.random.default_rng(2)
    mW, vW = rng.random((L, k)).astype(np.float32), rng.random((L, k)).astype(np.float32)
    lay.set_params(W=tens(W), idx=tens(idx), mW=tens(mW), vW=tens(vW))
    lay.redistribute(1000)
    s = state_of(lay)
    p = int(np.floor(F32(frac) * k))
    assert p > 32
    W2, idx2, m2, v2 = oracle.redistribute(W, idx, mW, vW, m, p, seed=19, step=1000)
    assert (s["idx"] == idx2).all()
    assert (s["W"] == W2).all() and (s["mW"] == m2).all() and (s["vW"] == v2).all()
    assert all(len(set(r)) == k for r in s["idx"])
    lay.set_params(idx=tens(s["idx"]))                              # round trip: no duplicate rejected


def test_redistribute_invalidates_stored_gradients():
    """backward -> redistribute -> adam_step must not apply the old connections'
    gradients to the regrown slots: the Adam step after a redistribution is refused."""
    layer = L_()
    L, m, k, B = 300, 256, 16, 32
    lay = make(L, m, k, B=B, seed=4)
    h = tens(synth.hidden_batch(B, m, step=1))
    ptr, ids = synth.label_batch(B, L, 5.0, step=1)
    y = lay.forward(h)
    lay.backward(h, y, tens(ptr), tens(ids))
    lay.redistribute(1000)
    with pytest.raises(layer.FFError) as e:
        lay.adam_step(1e-3)
    assert e.value.status == layer.FF_ERR_STATE
