"""Pins for the fp64 oracle against things other than itself (CPU only, -m "not gpu").

Each test names what fixes the expected value: a worked example printed in the paper
or SPEC (tests/golden/), a closed form, a textbook/library routine the operation
reduces to (dense matmul with a mask, a full sort), central finite differences, or an
invariant of the method.  Plausible oracle bugs (dropped bias, transposed idx, wrong
sign of the BCE gradient, using post-update W in dh, wrong Adam bias correction,
wrong tie rule, off-by-one in the Philox round/bump order) each fail at least one.
"""
import math

import numpy as np
import pytest

import oracle
from conftest import fig1c, read_golden
from paper_2306_03725_b200 import synth


def dense_equivalent(W, idx, m):
    """D[c][j] = sum_i W[j][i] [idx[j][i] = c] — the scatter-to-dense matrix."""
    L, k = W.shape
    D = np.zeros((m, L))
    for j in range(L):
        for i in range(k):
            D[idx[j, i], j] += W[j, i]
    return D


# ----------------------------------------------------------------- Fig. 1c (paper)
def test_fig1c_forward_ones_and_1234():
    f = fig1c()
    bias = np.zeros(5)
    y, _ = oracle.forward(f["W"], f["idx"], bias, np.ones((1, f["m"])))
    np.testing.assert_allclose(y[0], f["forward ones"], rtol=0, atol=1e-12)
    y, _ = oracle.forward(f["W"], f["idx"], bias, np.array([[1.0, 2.0, 3.0, 4.0]]))
    np.testing.assert_allclose(y[0], f["forward 1234"], rtol=0, atol=1e-12)
    _, ids = oracle.topk(y, 3)
    assert list(ids[0]) == [int(x) for x in f["top3 1234"]]


def test_fig1c_bias_is_added():
    f = fig1c()
    bias = np.array([1.0, -2.0, 0.5, 0.0, 3.0])
    y, Ay = oracle.forward(f["W"], f["idx"], bias, np.ones((1, 4)))
    np.testing.assert_allclose(y[0], np.array(f["forward ones"]) + bias, atol=1e-12)
    # companion: |bias| + sum |terms| with h = 1 -> |bias| + sum_i |W|
    np.testing.assert_allclose(Ay[0], np.abs(bias) + np.abs(f["W"]).sum(1), atol=1e-12)


def test_fig1c_onehot_input_grad_and_weight_grad():
    f = fig1c()
    g = np.zeros((1, 5)); g[0, 2] = 1.0
    dh, _ = oracle.input_grad(f["W"], f["idx"], g, 4)
    np.testing.assert_allclose(dh[0], f["dh onehot02"], atol=1e-12)
    h = np.array([[1.0, 2.0, 3.0, 4.0]])
    dW, _, db, _ = oracle.weight_grad(f["idx"], h, g)
    # only label 2 receives gradient: dW[2] = h[0][idx[2]] = h[0][{0,1}] = [1, 2]
    expect = np.zeros((5, 2)); expect[2] = [1.0, 2.0]
    np.testing.assert_allclose(dW, expect, atol=1e-12)
    np.testing.assert_allclose(db, [0, 0, 1, 0, 0], atol=1e-12)


def test_fig1c_redistribution_alpha_half():
    f = fig1c()
    z = np.zeros((5, 2))
    W2, idx2, m2, v2 = oracle.redistribute(f["W"], f["idx"], z + 0.5, z + 0.25, m=4, p=1, seed=7, step=1000)
    pruned = [int(x) for x in f["pruned p1"]]
    for j in range(5):
        s = pruned[j]
        other = 1 - s
        assert idx2[j, other] == f["idx"][j, other] and W2[j, other] == f["W"][j, other]
        assert idx2[j, s] in f["candidates"][j]
        assert W2[j, s] == 0.0 and m2[j, s] == 0.0 and v2[j, s] == 0.0
        assert m2[j, other] == 0.5 and v2[j, other] == 0.25


# ------------------------------------------------ dense-with-mask equivalence
@pytest.mark.parametrize("L,m,k,B", [(29, 13, 4, 7), (64, 64, 8, 3), (50, 200, 16, 32)])
def test_dense_mask_equivalence(L, m, k, B):
    W, idx, bias = synth.random_params(L, m, k, seed=L + m)
    W = W.astype(np.float64); bias = bias.astype(np.float64)
    rng = np.random.default_rng(5)
    h = rng.standard_normal((B, m))
    g = rng.standard_normal((B, L))
    D = dense_equivalent(W, idx, m)
    y, Ay = oracle.forward(W, idx, bias, h)
    np.testing.assert_allclose(y, h @ D + bias, rtol=0, atol=1e-12 * Ay.max())
    dh, Adh = oracle.input_grad(W, idx, g, m)
    np.testing.assert_allclose(dh, g @ D.T, rtol=0, atol=1e-12 * max(Adh.max(), 1))
    dW, AdW, db, _ = oracle.weight_grad(idx, h, g)
    G = h.T @ g                              # dense weight gradient [m][L]
    np.testing.assert_allclose(dW, G[idx, np.arange(L)[:, None]], rtol=0, atol=1e-12 * AdW.max())
    np.testing.assert_allclose(db, g.sum(0), atol=1e-12)


@pytest.mark.parametrize("row_begin", [0, 11])
def test_shortlist_is_a_slice_of_the_dense_layer(row_begin):
    """P:1057-1059 (R24): shortlist scores are the entries (b, j) of h @ D + bias for the
    listed pairs (dense matmul with the scatter matrix, a route independent of Alg. 1's
    loop), 0 for labels outside this shard; an empty list scores nothing."""
    L, m, k, B = 40, 30, 6, 5
    W, idx, bias = synth.random_params(L, m, k, seed=77)
    W = W.astype(np.float64); bias = bias.astype(np.float64)
    h = np.random.default_rng(3).standard_normal((B, m))
    Yd = h @ dense_equivalent(W, idx, m) + bias
    ptr = np.array([0, 4, 4, 7, 12, 13], np.int32)
    ids = np.array([11, 50, 12, 11, 0, 39 + 11, 20, 30, 31, 51, 10, 13, 25], np.int32)
    y, Ay = oracle.score_shortlist(W, idx, bias, h, ptr, ids, row_begin=row_begin)
    b_of = np.repeat(np.arange(B), np.diff(ptr))
    j = ids.astype(np.int64) - row_begin
    own = (j >= 0) & (j < L)
    np.testing.assert_allclose(y[own], Yd[b_of[own], j[own]], rtol=0, atol=1e-12 * Ay.max())
    assert (y[~own] == 0).all() and (~own).any() and own.any()
    y0, _ = oracle.score_shortlist(W, idx, bias, h, np.zeros(B + 1, np.int32), np.zeros(0, np.int32))
    assert y0.shape == (0,)


def test_full_fan_in_equals_dense_layer():
    """k = m: every label connects to every feature -> a dense layer."""
    L, m, B = 12, 8, 5
    rng = np.random.default_rng(1)
    idx = np.stack([rng.permutation(m) for _ in range(L)]).astype(np.int32)
    Wd = rng.standard_normal((m, L))                      # dense decoder W in R^{m x L}
    W = np.take_along_axis(Wd.T, idx, axis=1)             # the same weights in fixed fan-in form
    h = rng.standard_normal((B, m))
    y, _ = oracle.forward(W, idx, np.zeros(L), h)
    np.testing.assert_allclose(y, h @ Wd, atol=1e-12)


# ---------------------------------------------------------- finite differences
def _loss(W, idx, bias, h, ptr, ids, s):
    y, _ = oracle.forward(W, idx, bias, h)
    return oracle.bce_grad(y, ptr, ids, s)[1]


def test_gradients_match_central_finite_differences():
    L, m, k, B = 9, 11, 3, 4
    W, idx, bias = synth.random_params(L, m, k, seed=3, scale=0.8)
    W = W.astype(np.float64); bias = bias.astype(np.float64)
    h = np.random.default_rng(2).standard_normal((B, m))
    ptr, ids = synth.random_labels_uniform(B, L, 2, seed=9)
    s = 1.0 / B
    y, _ = oracle.forward(W, idx, bias, h)
    g, _ = oracle.bce_grad(y, ptr, ids, s)
    dW, _, db, _ = oracle.weight_grad(idx, h, g)
    dh, _ = oracle.input_grad(W, idx, g, m)
    eps = 1e-6

    def fd(arr, pos, fn):
        a = arr.copy(); a[pos] += eps; up = fn(a)
        a = arr.copy(); a[pos] -= eps; dn = fn(a)
        return (up - dn) / (2 * eps)

    for pos in [(0, 0), (3, 2), (8, 1), (5, 0)]:
        num = fd(W, pos, lambda a: _loss(a, idx, bias, h, ptr, ids, s))
        assert abs(num - dW[pos]) <= 1e-4 * max(abs(dW[pos]), 1e-3)
    for j in [0, 4, 8]:
        num = fd(bias, (j,), lambda a: _loss(W, idx, a, h, ptr, ids, s))
        assert abs(num - db[j]) <= 1e-4 * max(abs(db[j]), 1e-3)
    for pos in [(0, idx[0, 0]), (2, idx[3, 1]), (3, 10), (1, 5)]:
        num = fd(h, pos, lambda a: _loss(W, idx, bias, a, ptr, ids, s))
        assert abs(num - dh[pos]) <= 1e-4 * max(abs(dh[pos]), 1e-3)


# ----------------------------------------------------------------- BCE closed forms
def test_bce_closed_forms():
    rows = [ln for ln in read_golden("spec_examples.txt") if ln.startswith("bce:")]
    yv, t, loss_e, g_e = [p.strip() for p in rows[0].split(":", 1)[1].split("|")]
    ptr = np.array([0, 1], np.int32); ids = np.array([0], np.int32)
    g, loss = oracle.bce_grad(np.array([[float(yv)]]), ptr, ids, 1.0)
    assert int(t) == 1
    assert abs(loss - float(loss_e)) < 1e-15 and abs(g[0, 0] - float(g_e)) < 1e-15
    # grad_scale multiplies both (R4)
    g, loss = oracle.bce_grad(np.array([[0.0]]), ptr, ids, 0.25)
    assert abs(loss - 0.25 * math.log(2)) < 1e-15 and abs(g[0, 0] + 0.125) < 1e-15
    # y = +40, t = 1: loss = log1p(e^-40) ~ 4.25e-18, grad = -sigma(-40), stable and non-zero (R5)
    g, loss = oracle.bce_grad(np.array([[40.0]]), ptr, ids, 1.0)
    assert loss == pytest.approx(math.exp(-40), rel=1e-12) and g[0, 0] == pytest.approx(-math.exp(-40), rel=1e-12)
    # y = +40, t = 0: loss = 40 + log1p(e^-40), grad = sigma(40) ~ 1
    g, loss = oracle.bce_grad(np.array([[40.0]]), np.array([0, 0], np.int32), np.zeros(0, np.int32), 1.0)
    assert loss == pytest.approx(40.0, rel=1e-15) and g[0, 0] == pytest.approx(1.0, rel=1e-15)
    # y = -800, t = 1: no overflow, loss = 800
    g, loss = oracle.bce_grad(np.array([[-800.0]]), ptr, ids, 1.0)
    assert loss == pytest.approx(800.0) and g[0, 0] == pytest.approx(-1.0)


def test_bce_labels_outside_shard_are_negatives_and_row_begin_offsets():
    # instance 0 has positive global label 7; a shard with rows [5, 10) sees it at local 2
    y = np.zeros((1, 5))
    ptr = np.array([0, 1], np.int32); ids = np.array([7], np.int32)
    g, _ = oracle.bce_grad(y, ptr, ids, 1.0, row_begin=5)
    np.testing.assert_allclose(g[0], [0.5, 0.5, -0.5, 0.5, 0.5])
    g, _ = oracle.bce_grad(y, ptr, ids, 1.0, row_begin=0)
    np.testing.assert_allclose(g[0], [0.5] * 5)


def test_bce_grad_is_loss_derivative():
    rng = np.random.default_rng(4)
    y = rng.standard_normal((3, 6)) * 5
    ptr, ids = synth.random_labels_uniform(3, 6, 2, seed=1)
    g, _ = oracle.bce_grad(y, ptr, ids, 0.5)
    for pos in [(0, 0), (1, 3), (2, 5)]:
        e = 1e-6
        yp = y.copy(); yp[pos] += e
        ym = y.copy(); ym[pos] -= e
        num = (oracle.bce_grad(yp, ptr, ids, 0.5)[1] - oracle.bce_grad(ym, ptr, ids, 0.5)[1]) / (2 * e)
        assert num == pytest.approx(g[pos], rel=1e-6)


# ----------------------------------------------------------------------- Adam
def test_adam_first_step_is_sign_step():
    """t = 1 from zero state: m_hat = q, v_hat = q^2 -> dp = -lr q/(|q| + eps)."""
    q = np.array([1.0, -3.0, 1e-3, 0.0])
    p, m, v = oracle.adam(np.zeros(4), q, np.zeros(4), np.zeros(4), t=1, lr=1e-3)
    np.testing.assert_allclose(p, -1e-3 * q / (np.abs(q) + 1e-8), rtol=1e-12, atol=0)
    np.testing.assert_allclose(m, 0.1 * q, rtol=1e-14)
    np.testing.assert_allclose(v, 0.001 * q * q, rtol=1e-13)
    assert p[3] == 0.0          # g = 0 from zero state -> unchanged


def test_adam_constant_gradient_closed_form():
    """Constant q: m_t = (1-b1^t) q and v_t = (1-b2^t) q^2 exactly in real arithmetic, so
    every bias-corrected step is -lr q/(|q|+eps); after T steps p = p0 - T lr q/(|q|+eps)."""
    q = np.array([0.7, -2.0, 5e-5])
    p, m, v = np.ones(3), np.zeros(3), np.zeros(3)
    for t in range(1, 11):
        p, m, v = oracle.adam(p, q, m, v, t=t, lr=1e-2)
        np.testing.assert_allclose(m, (1 - 0.9 ** t) * q, rtol=1e-13)
        np.testing.assert_allclose(v, (1 - 0.999 ** t) * q * q, rtol=1e-12)
    np.testing.assert_allclose(p, 1.0 - 10 * 1e-2 * q / (np.abs(q) + 1e-8), rtol=1e-12)


def test_adam_uses_global_t_for_bias_correction():
    # step 2 with fresh (zero) moments: m = 0.1 q, v = 0.001 q^2, bias corrections 1-.81, 1-.998001
    q = np.array([2.0])
    p, _, _ = oracle.adam(np.zeros(1), q, np.zeros(1), np.zeros(1), t=2, lr=1.0)
    mhat = 0.1 * 2 / (1 - 0.81); vhat = 0.001 * 4 / (1 - 0.998001)
    assert p[0] == pytest.approx(-mhat / (math.sqrt(vhat) + 1e-8), rel=1e-14)


# ---------------------------------------------------------------------- Philox
def test_philox_known_answer_vectors():
    for ln in read_golden("philox_kat.txt"):
        a, b = ln.split("->")
        w = [int(x, 16) for x in a.split()]
        out = [int(x, 16) for x in b.split()]
        assert list(oracle.philox4x32_10(w[:4], w[4:6])) == out


# ------------------------------------------------------------------------ init
def test_init_rows_distinct_in_range_deterministic_and_key_dependent():
    idx, W = oracle.init(500, 64, 16, seed=42)
    assert idx.min() >= 0 and idx.max() < 64
    assert all(len(set(r)) == 16 for r in idx)
    idx2, W2 = oracle.init(500, 64, 16, seed=42)
    assert (idx == idx2).all() and (W.view(np.uint32) == W2.view(np.uint32)).all()
    idx3, _ = oracle.init(500, 64, 16, seed=43)
    assert (idx3 != idx).any()
    a = np.float32(1 / np.sqrt(16))
    assert np.abs(W).max() <= a and W.dtype == np.float32


def test_init_sharding_is_row_keyed():
    """A shard [row_begin, row_begin+L) initializes exactly the corresponding rows (R13)."""
    idx, W = oracle.init(100, 50, 8, seed=5)
    idx_s, W_s = oracle.init(30, 50, 8, seed=5, row_begin=40)
    assert (idx_s == idx[40:70]).all() and (W_s == W[40:70]).all()


def test_init_is_uniform():
    """chi-square of index frequencies at L = 10^4, m = 128 (S:337 style); W ~ U(-a, a)."""
    L, m, k = 10000, 128, 16
    idx, W = oracle.init(L, m, k, seed=11)
    cnt = np.bincount(idx.ravel(), minlength=m)
    exp = L * k / m
    chi2 = ((cnt - exp) ** 2 / exp).sum()
    assert chi2 < 127 + 5 * math.sqrt(2 * 127)         # dof = 127, 5 sigma
    a = 1 / math.sqrt(k)
    assert abs(W.mean()) < 5 * a / math.sqrt(3 * W.size)
    assert W.var() == pytest.approx(a * a / 3, rel=0.02)


# --------------------------------------------------------------- redistribution
def test_prune_count_examples():
    for ln in read_golden("spec_examples.txt"):
        if ln.startswith("prune_count:"):
            k, alpha, p = ln.split(":")[1].split()
            assert math.floor(float(np.float32(alpha)) * int(k)) == int(p)


def _check_redistribution(W, idx, mW, vW, W2, idx2, m2, v2, m, p):
    L, k = W.shape
    for j in range(L):
        # brute-force sort oracle: stable order by (|W|, slot) via lexsort
        order = np.lexsort((np.arange(k), np.abs(W[j])))
        pruned = set(order[:p].tolist())
        survivors = [i for i in range(k) if i not in pruned]
        assert len(set(idx2[j])) == k and idx2[j].min() >= 0 and idx2[j].max() < m       # fan-in
        for i in survivors:                                                                # untouched
            assert idx2[j, i] == idx[j, i] and W2[j, i] == W[j, i] and m2[j, i] == mW[j, i] and v2[j, i] == vW[j, i]
        old = set(idx[j].tolist())
        for i in sorted(pruned):
            assert idx2[j, i] not in old                                                   # freshness
            assert W2[j, i] == 0 and m2[j, i] == 0 and v2[j, i] == 0                      # hygiene
        if survivors and pruned:                                                           # dominance
            assert min(abs(W[j, i]) for i in survivors) >= max(abs(W[j, i]) for i in pruned)


@pytest.mark.parametrize("L,m,k,p", [(300, 40, 16, 1), (200, 64, 32, 3), (100, 35, 32, 3), (50, 12, 4, 2)])
def test_redistribution_invariants_vs_sort(L, m, k, p):
    W, idx, _ = synth.random_params(L, m, k, seed=p + k)
    W = W.astype(np.float64)
    rng = np.random.default_rng(0)
    W[::7, 1] = W[::7, 0]          # exact ties in |W| -> lower slot pruned first
    W[::5, 2] = -W[::5, 3]
    mW, vW = rng.random((L, k)), rng.random((L, k))
    W2, idx2, m2, v2 = oracle.redistribute(W, idx, mW, vW, m, p, seed=3, step=1000)
    _check_redistribution(W, idx, mW, vW, W2, idx2, m2, v2, m, p)


def test_hundred_train_redistribute_cycles_keep_the_invariants():
    """SPEC acceptance criterion 3 on the oracle: 100 interleaved train / prune-and-
    regrow cycles on a random model; after every cycle each row has k distinct in-range
    indices, regrown slots have zero weight and moments, survivors are untouched and dominate
    the pruned slots in |W| (the sort-oracle check)."""
    L, m, k, B = 60, 48, 8, 4
    p = 2
    st = oracle.State.create(L, m, k, seed=7)
    for cyc in range(100):
        h = synth.hidden_batch(B, m, step=cyc)
        ptr, ids = synth.label_batch(B, L, 2.0, step=cyc)
        oracle.train_step(st, h, ptr, ids, 1.0 / B, 1e-2)
        W, idx, mW, vW = st.W.copy(), st.idx.copy(), st.mW.copy(), st.vW.copy()
        st.W, st.idx, st.mW, st.vW = oracle.redistribute(W, idx, mW, vW, m, p, seed=7, step=1000 * (cyc + 1))
        _check_redistribution(W, idx, mW, vW, st.W, st.idx, st.mW, st.vW, m, p)


def test_redistribution_all_equal_prunes_lowest_slots_and_single_zero():
    W = np.ones((4, 8)); W[1] = -1; W[2, 5] = 0.0   # row 2: the single zero-magnitude entry
    idx = np.tile(np.arange(8, dtype=np.int32), (4, 1))
    z = np.zeros((4, 8))
    W2, idx2, _, _ = oracle.redistribute(W, idx, z, z, m=20, p=2, seed=1, step=5)
    for j in (0, 1, 3):
        assert (W2[j, :2] == 0).all() and (idx2[j, 2:] == np.arange(2, 8)).all()
    assert W2[2, 5] == 0 and W2[2, 0] == 0 and (W2[2, 1:5] == 1).all()
    _, idx3, _, _ = oracle.redistribute(W, idx, z, z, m=20, p=1, seed=1, step=5)
    assert idx3[2, 5] >= 8 and (idx3[2, :5] == np.arange(5)).all()


def test_redistribution_is_uniform_and_step_keyed():
    """Regrown indices are uniform over the structural zeros (chi-square), and different
    steps draw different streams while the same step reproduces bit-exactly."""
    L, m, k, p = 20000, 40, 8, 1
    idx = np.tile(np.arange(k, dtype=np.int32), (L, 1))         # all rows use columns 0..7
    W = np.tile(np.arange(1, k + 1, dtype=np.float64), (L, 1))  # slot 0 always pruned
    z = np.zeros((L, k))
    _, idx2, _, _ = oracle.redistribute(W, idx, z, z, m, p, seed=9, step=1000)
    new = idx2[:, 0]
    assert new.min() >= k
    cnt = np.bincount(new - k, minlength=m - k)
    exp = L / (m - k)
    chi2 = ((cnt - exp) ** 2 / exp).sum()
    dof = m - k - 1
    assert chi2 < dof + 5 * math.sqrt(2 * dof)
    _, idx3, _, _ = oracle.redistribute(W, idx, z, z, m, p, seed=9, step=1000)
    assert (idx3 == idx2).all()
    _, idx4, _, _ = oracle.redistribute(W, idx, z, z, m, p, seed=9, step=2000)
    assert (idx4 != idx2).any()


# ------------------------------------------------------------------ top-k / P@k
def test_topk_spec_examples_and_full_sort():
    for ln in read_golden("spec_examples.txt"):
        if ln.startswith("topk:"):
            sc, K, out = [p.strip() for p in ln.split(":", 1)[1].split("|")]
            y = np.array([[float(x) for x in sc.split()]])
            _, ids = oracle.topk(y, int(K))
            assert list(ids[0]) == [int(x) for x in out.split()]
    rng = np.random.default_rng(8)
    y = np.round(rng.standard_normal((5, 1000)), 1)      # many exact ties
    s, ids = oracle.topk(y, 7, row_begin=100)
    for b in range(5):
        order = np.lexsort((np.arange(1000), -y[b]))[:7]  # full sort (score desc, id asc)
        assert list(ids[b]) == list(order + 100)
        np.testing.assert_array_equal(s[b], y[b, order])


def test_precision_at_k_example():
    ln = [l for l in read_golden("spec_examples.txt") if l.startswith("patk:")][0]
    pos, top, val = [p.strip() for p in ln.split(":", 1)[1].split("|")]
    ptr, ids = oracle.labels_csr([[int(x) for x in pos.split(",")]])
    got = oracle.precision_at_k(np.array([[int(x) for x in top.split()]]), ptr, ids)
    assert got == pytest.approx(float(val), abs=1e-15)
    # fewer positives than K still divides by K (R16); perfect ranking -> 1
    ptr, ids = oracle.labels_csr([[4], [1, 2, 3]])
    got = oracle.precision_at_k(np.array([[4, 0, 9], [3, 1, 2]]), ptr, ids)
    assert got == pytest.approx((1 / 3 + 1) / 2)


def test_dense_memory_closed_form():
    """1024 x 2,812,281 fp32 = 2.9 B params = 10.7 GiB; > 40 GiB with Adam."""
    ln = [l for l in read_golden("spec_examples.txt") if l.startswith("dense_bytes:")][0]
    d, L, bpe, total = [int(x) for x in ln.split(":")[1].split()]
    assert d * L * bpe == total
    assert round(d * L / 1e9, 1) == 2.9 and round(total / 2 ** 30, 1) == 10.7
    assert 4 * total / 2 ** 30 > 40


# --------------------------------------------------------- composite training step
def test_train_step_uses_pre_update_weights_for_dh_and_updates_bias():
    L, m, k, B = 40, 30, 4, 5
    st = oracle.State.create(L, m, k, seed=2)
    h = synth.hidden_batch(B, m, step=0).astype(np.float64)
    ptr, ids = synth.random_labels_uniform(B, L, 3, seed=2)
    W0 = st.W.copy()
    r = oracle.train_step(st, h, ptr, ids, 1.0 / B, 1e-2)
    dh_pre, _ = oracle.input_grad(W0, st.idx, r.g, m)
    np.testing.assert_allclose(r.dh, dh_pre, atol=0)
    assert st.t == 1 and np.abs(st.bias).max() > 0 and not np.allclose(st.W, W0)
    # t = 1 sign step: |dW| >> eps so every weight moved by ~lr
    moved = np.abs(st.W - W0)[np.abs(r.dW) > 1e-5]
    np.testing.assert_allclose(moved, 1e-2, rtol=1e-3)


# ------------------------------------------------------ squared hinge (NEXT-1)
def test_sqh_closed_forms_and_exact_zeros():
    for ln in read_golden("spec_examples.txt"):
        if ln.startswith("sqh:"):
            yv, t, l_e, g_e = [p.strip() for p in ln.split(":", 1)[1].split("|")]
            ptr = np.array([0, 1], np.int32); ids = np.array([0], np.int32)
            assert int(t) == 1
            g, loss = oracle.sqh_grad(np.array([[float(yv)]]), ptr, ids, 1.0)
            assert loss == float(l_e) and g[0, 0] == float(g_e)
    # negatives use y = -1: yhat = -2 meets the margin (zero), yhat = 0.25 -> grad 2*1.25, loss 1.5625
    g, loss = oracle.sqh_grad(np.array([[-2.0, 0.25]]), np.array([0, 0], np.int32), np.zeros(0, np.int32), 1.0)
    assert g[0, 0] == 0.0 and g[0, 1] == 2.5 and loss == 1.5625


def test_sqh_zero_count_equals_margin_count_and_fd():
    """the number of exact zeros in the gradient equals the number of (b, j) with
    y*yhat >= 1; the gradient is the derivative of the loss (central differences)."""
    rng = np.random.default_rng(3)
    y = rng.standard_normal((6, 50)) * 2
    ptr, ids = synth.random_labels_uniform(6, 50, 4, seed=5)
    g, _ = oracle.sqh_grad(y, ptr, ids, 0.5)
    t = -np.ones_like(y)
    for b in range(6):
        t[b, ids[ptr[b]:ptr[b + 1]]] = 1.0
    assert (g == 0).sum() == (t * y >= 1).sum()
    for pos in [(0, 0), (3, 17), (5, 49)]:
        e = 1e-6
        yp = y.copy(); yp[pos] += e
        ym = y.copy(); ym[pos] -= e
        num = (oracle.sqh_grad(yp, ptr, ids, 0.5)[1] - oracle.sqh_grad(ym, ptr, ids, 0.5)[1]) / (2 * e)
        assert num == pytest.approx(g[pos], rel=1e-6, abs=1e-9)


# ------------------------------------------- NEXT-2: intermediate layer + input dropout
def test_dropout_p0_is_identity_and_kept_values_are_scaled_exactly():
    x = synth.feature_batch(6, 40, step=2).astype(np.float64)
    xt, keep, s = oracle.dropout(x, 0.0, seed=9, step=5)
    assert s == 1.0 and keep.all() and (xt == x).all()
    xt, keep, s = oracle.dropout(x, 0.25, seed=9, step=5)
    assert s == np.float32(1.0) / np.float32(0.75)
    assert (xt[keep == 1] == x[keep == 1] * s).all() and (xt[keep == 0] == 0.0).all()


def test_dropout_decision_uses_the_pinned_philox_stream():
    """The keep decision of (b, f) is word f % 4 of Philox(ctr = (f/4, b, step, 3), key = seed)
    (reading R25), with Philox itself pinned by the Random123 vectors above."""
    B, d, seed, step, p = 3, 9, 0x1234_5678_9ABC, 17, 0.3
    _, keep, _ = oracle.dropout(np.ones((B, d)), p, seed, step)
    for b in range(B):
        for f in range(d):
            u = oracle.philox4x32_10([f // 4, b, step, 3], [seed & 0xFFFFFFFF, seed >> 32])[f % 4]
            assert keep[b, f] == ((u >> 8) / 2.0 ** 24 >= np.float32(p))


def test_dropout_rate_and_keying():
    B, d, p = 32, 2048, 0.1                 # 10% for Amazon-670K features
    _, k1, _ = oracle.dropout(np.ones((B, d)), p, seed=42, step=7)
    n = B * d
    drop = n - int(k1.sum())
    assert abs(drop - p * n) < 5 * math.sqrt(n * p * (1 - p))
    _, k2, _ = oracle.dropout(np.ones((B, d)), p, seed=42, step=8)
    _, k3, _ = oracle.dropout(np.ones((B, d)), p, seed=43, step=7)
    _, k4, _ = oracle.dropout(np.ones((B, d)), p, seed=42, step=7)
    assert (k1 != k2).any() and (k1 != k3).any() and (k1 == k4).all()
    assert (k1[0] != k1[1]).any()           # samples get independent masks


def test_dense_forward_is_a_matmul_plus_bias_then_relu():
    B, d, m = 5, 24, 40
    x = synth.feature_batch(B, d).astype(np.float64)
    Wd = oracle.dense_init(d, m, seed=3).astype(np.float64)
    bd = np.linspace(-0.2, 0.2, m)
    z, Az, h = oracle.dense_forward(Wd, bd, x)
    ref = x @ Wd + bd                       # library matmul (the operation's definition)
    assert np.allclose(z, ref, rtol=0, atol=1e-13)
    assert (h == np.maximum(z, 0.0)).all()
    assert (Az >= np.abs(z) - 1e-15).all()
    assert 0.2 < (h == 0).mean() < 0.8


def test_dense_backward_matches_matmul_and_relu_prime_at_zero_is_zero():
    B, d, m = 7, 10, 12
    xt = synth.feature_batch(B, d, step=1).astype(np.float64)
    z = synth.feature_batch(B, m, step=2).astype(np.float64)
    z[0, :3] = 0.0                           # exactly at the kink: ReLU'(0) = 0 (R26)
    dh = synth.feature_batch(B, m, step=3).astype(np.float64)
    dWd, AdWd, dbd, Adbd = oracle.dense_backward(xt, z, dh)
    dz = dh * (z > 0)
    assert np.allclose(dWd, xt.T @ dz, rtol=0, atol=1e-13)
    assert np.allclose(dbd, dz.sum(0), rtol=0, atol=1e-13)
    dWd0, _, dbd0, _ = oracle.dense_backward(xt[:1], z[:1], dh[:1])
    assert (dWd0[:, :3] == 0).all() and (dbd0[:3] == 0).all()


def test_dense_init_range_uniformity_and_keying():
    d, m = 64, 512
    Wd = oracle.dense_init(d, m, seed=11)
    a = np.float32(np.sqrt(6.0 / (d + m)))
    assert Wd.dtype == np.float32 and np.abs(Wd).max() <= a
    hist, _ = np.histogram(Wd, bins=16, range=(-a, a))
    exp = Wd.size / 16
    assert ((hist - exp) ** 2 / exp).sum() < 50.0          # chi^2, 15 dof
    assert (oracle.dense_init(d, m, seed=11) == Wd).all() and (oracle.dense_init(d, m, seed=12) != Wd).any()


def _model_loss(Wd, bd, xt, st, ptr, ids, s):
    _, _, h = oracle.dense_forward(Wd, bd, xt)
    y, _ = oracle.forward(st.W, st.idx, st.bias, h)
    return oracle.bce_grad(y, ptr, ids, s)[1]


def test_model_gradients_match_central_finite_differences():
    """dWd / dbd of the whole architecture (dropout -> dense -> ReLU -> sparse -> BCE) against
    central finite differences of the loss: pins the dense backward, the ReLU mask and the
    sparse layer's dh feeding it (Fig. 2)."""
    B, d, m, L, k = 4, 6, 16, 30, 4
    x = synth.feature_batch(B, d, step=4).astype(np.float64)
    ds = oracle.DenseState.create(d, m, seed=5)
    ds.bd = np.linspace(-0.05, 0.1, m)
    st = oracle.State.create(L, m, k, seed=6)
    st.bias = np.linspace(-1, 1, L)
    ptr, ids = synth.label_batch(B, L, 3.0, step=1)
    s = 1.0 / B
    r = oracle.model_train_step(ds.copy(), st.copy(), x, step=3, dropout_p=0.2, seed=77, lbl_ptr=ptr,
                                lbl_ids=ids, grad_scale=s, lr=0.0)
    eps = 1e-6
    assert (np.abs(r.z) > 1e-4).all()        # no kink within the FD step
    rng = np.random.default_rng(0)
    for (f, c) in [tuple(rng.integers(0, (d, m))) for _ in range(12)]:
        Wp, Wm = ds.Wd.copy(), ds.Wd.copy()
        Wp[f, c] += eps; Wm[f, c] -= eps
        fd = (_model_loss(Wp, ds.bd, r.xt, st, ptr, ids, s) - _model_loss(Wm, ds.bd, r.xt, st, ptr, ids, s)) / (2 * eps)
        assert abs(fd - r.dWd[f, c]) <= 1e-6 * max(1.0, abs(fd)) + 1e-9, (f, c, fd, r.dWd[f, c])
    for c in range(0, m, 3):
        bp, bm = ds.bd.copy(), ds.bd.copy()
        bp[c] += eps; bm[c] -= eps
        fd = (_model_loss(ds.Wd, bp, r.xt, st, ptr, ids, s) - _model_loss(ds.Wd, bm, r.xt, st, ptr, ids, s)) / (2 * eps)
        assert abs(fd - r.dbd[c]) <= 1e-6 * max(1.0, abs(fd)) + 1e-9


def test_model_step_updates_both_layers_with_their_own_t():
    B, d, m, L, k = 3, 5, 12, 20, 4
    x = synth.feature_batch(B, d).astype(np.float64)
    ds, st = oracle.DenseState.create(d, m, seed=1), oracle.State.create(L, m, k, seed=2)
    ptr, ids = synth.label_batch(B, L, 2.0)
    W0, Wd0 = st.W.copy(), ds.Wd.copy()
    r = oracle.model_train_step(ds, st, x, 0, 0.1, 9, ptr, ids, 1.0 / B, 1e-3)
    assert ds.t == 1 and st.t == 1
    # Adam's first step moves every parameter with a nonzero gradient by ~lr (sign step)
    moved = np.abs(ds.Wd - Wd0)
    nz = np.abs(r.dWd) > 1e-6
    assert np.allclose(moved[nz], 1e-3, rtol=1e-2) and (moved[r.dWd == 0] == 0).all()
    assert (np.abs(st.W - W0) > 0).any()


def test_threaded_timing_mode_equals_sequential_oracle():
    """the OpenMP timing mode (bench.py's cpu_baseline and reference arm)
    computes the same step: y, g, dW, db and the Adam state bit-identical to the sequential
    loops, dh and the loss equal up to the fp64 summation order."""
    import os
    L, m, k, B = 3001, 512, 16, 32
    h = synth.hidden_batch(B, m, step=1)
    ptr, ids = synth.label_batch(B, L, 5.0, step=1)
    a = oracle.State.create(L, m, k, seed=42)
    b = a.copy()
    oracle.set_threads(1)
    ra = oracle.train_step(a, h, ptr, ids, 1.0 / B, 1e-3)
    try:
        oracle.set_threads(max(2, min(8, len(os.sched_getaffinity(0)))))
        rb = oracle.train_step(b, h, ptr, ids, 1.0 / B, 1e-3)
    finally:
        oracle.set_threads(1)
    for x, y in ((ra.y, rb.y), (ra.g, rb.g), (ra.dW, rb.dW), (ra.db, rb.db), (a.W, b.W), (a.mW, b.mW),
                 (a.vW, b.vW), (a.bias, b.bias)):
        assert np.array_equal(x, y)
    assert np.abs(ra.dh - rb.dh).max() <= 1e-12 * ra.Adh.max()
    assert abs(ra.loss - rb.loss) <= 1e-12 * abs(ra.loss)
