"""fp64 CPU oracle for the fixed fan-in sparse output layer (arXiv 2306.03725).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this module.
The product package ``paper_2306_03725_b200`` never imports it and shares no code
with it (the oracle's arithmetic is in ``oracle.c``; this file only marshals
numpy arrays through ctypes and chains the paper's steps in the paper's order).

Every function cites the passage it follows; see ``oracle.c`` for the loops and
DESIGN.md for the readings (R1..R23) of the paper where it is silent/ambiguous.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile oracle.c (plain C, -O2, single thread) into liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-fopenmp", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32, u64, f64, f32 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double, ctypes.c_float
        L.oracle_forward.argtypes = [i64, i32, i32, i32, P, P, P, P, P, P]
        L.oracle_bce_grad.argtypes = [i64, i64, i32, P, P, P, f64, P, P]
        L.oracle_sqh_grad.argtypes = [i64, i64, i32, P, P, P, f64, P, P]
        L.oracle_weight_grad.argtypes = [i64, i32, i32, i32, P, P, P, P, P, P, P]
        L.oracle_input_grad.argtypes = [i64, i32, i32, i32, P, P, P, P, P]
        L.oracle_adam.argtypes = [i64, P, P, P, P, i64, f64, f64, f64, f64]
        L.oracle_philox4x32_10.argtypes = [P, P, P]
        L.oracle_set_threads.argtypes = [i32]
        L.oracle_set_threads.restype = None
        L.oracle_get_threads.argtypes = []
        L.oracle_get_threads.restype = i32
        L.oracle_init.argtypes = [i64, i64, i32, i32, u64, f32, P, P]
        L.oracle_redistribute.argtypes = [i64, i64, i32, i32, i32, u64, u64, P, P, P, P]
        L.oracle_topk.argtypes = [i64, i64, i32, P, i32, P, P]
        L.oracle_score_shortlist.argtypes = [i64, i64, i32, i32, i32, P, P, P, P, P, P, P, P]
        L.oracle_precision_at_k.argtypes = [i32, i32, P, P, P]
        L.oracle_precision_at_k.restype = f64
        L.oracle_dropout.argtypes = [i32, i32, f64, f64, u64, ctypes.c_uint32, P, P, P]
        L.oracle_dense_forward.argtypes = [i32, i32, i32, P, P, P, P, P, P]
        L.oracle_dense_backward.argtypes = [i32, i32, i32, P, P, P, P, P, P, P]
        L.oracle_dense_init.argtypes = [i32, i32, u64, f32, P]
        for f in ("oracle_dropout", "oracle_dense_forward", "oracle_dense_backward", "oracle_dense_init"):
            getattr(L, f).restype = None
        for f in ("oracle_forward", "oracle_bce_grad", "oracle_sqh_grad", "oracle_weight_grad", "oracle_input_grad",
                  "oracle_adam", "oracle_philox4x32_10", "oracle_init", "oracle_redistribute", "oracle_topk",
                  "oracle_score_shortlist"):
            getattr(L, f).restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def set_threads(n: int) -> None:
    """Timing mode: share the label loops over n OpenMP threads (1 = the
    plain sequential loops the parity tests use).  Only bench.py's CPU legs set n > 1."""
    lib().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(lib().oracle_get_threads())


# --------------------------------------------------------------------------- steps
def forward(W, idx, bias, h):
    """Alg. 1 + bias: y[b,j] = bias[j] + sum_i W[j,i] h[b, idx[j,i]].
    Returns (y[B][L], Ay[B][L]) with Ay the |term| companion (reading R19)."""
    W, idx, bias, h = _f64(W), _i32(idx), _f64(bias), _f64(h)
    L, k = W.shape
    B, m = h.shape
    y = np.empty((B, L)); Ay = np.empty((B, L))
    lib().oracle_forward(L, m, k, B, _p(W), _p(idx), _p(bias), _p(h), _p(y), _p(Ay))
    return y, Ay


def score_shortlist(W, idx, bias, h, cand_ptr, cand_ids, row_begin=0):
    """Alg. 1 restricted to a CSR shortlist of (instance, label) pairs
    (P:1057-1059); 0 for labels outside this shard (reading R24).  Returns (y[nnz], Ay[nnz])."""
    W, idx, bias, h = _f64(W), _i32(idx), _f64(bias), _f64(h)
    L, k = W.shape
    B, m = h.shape
    cp, ci = _i32(cand_ptr), _i32(cand_ids if len(cand_ids) else np.zeros(1, np.int32))
    n = int(cp[-1])
    y = np.empty(max(n, 1)); Ay = np.empty(max(n, 1))
    lib().oracle_score_shortlist(L, row_begin, m, k, B, _p(W), _p(idx), _p(bias), _p(h), _p(cp), _p(ci), _p(y), _p(Ay))
    return y[:n], Ay[:n]


def labels_csr(pos_lists):
    """Positive label lists per instance -> (ptr[B+1], ids) int32 CSR."""
    ptr = np.zeros(len(pos_lists) + 1, dtype=np.int32)
    for b, p in enumerate(pos_lists):
        ptr[b + 1] = ptr[b] + len(p)
    ids = np.array([x for p in pos_lists for x in p], dtype=np.int32)
    return ptr, ids


def bce_grad(y, lbl_ptr, lbl_ids, grad_scale, row_begin=0):
    """BCE-with-logits gradient and loss, OvA over all labels."""
    y = _f64(y)
    B, L = y.shape
    g = np.empty_like(y)
    loss = ctypes.c_double(0.0)
    lp, li = _i32(lbl_ptr), _i32(lbl_ids if len(lbl_ids) else np.zeros(1, np.int32))
    lib().oracle_bce_grad(L, row_begin, B, _p(y), _p(lp), _p(li), float(grad_scale), _p(g),
                          ctypes.cast(ctypes.pointer(loss), ctypes.c_void_p))
    return g, loss.value


def sqh_grad(y, lbl_ptr, lbl_ids, grad_scale, row_begin=0):
    """Squared-hinge gradient and loss, exact zeros where y*yhat >= 1."""
    y = _f64(y)
    B, L = y.shape
    g = np.empty_like(y)
    loss = ctypes.c_double(0.0)
    lp, li = _i32(lbl_ptr), _i32(lbl_ids if len(lbl_ids) else np.zeros(1, np.int32))
    lib().oracle_sqh_grad(L, row_begin, B, _p(y), _p(lp), _p(li), float(grad_scale), _p(g),
                          ctypes.cast(ctypes.pointer(loss), ctypes.c_void_p))
    return g, loss.value


def loss_grad(kind, y, lbl_ptr, lbl_ids, grad_scale, row_begin=0):
    return (sqh_grad if kind == "sqh" else bce_grad)(y, lbl_ptr, lbl_ids, grad_scale, row_begin)


def weight_grad(idx, h, g):
    """Alg. 3 and db = sum_b g.  Returns (dW, AdW, db, Adb)."""
    idx, h, g = _i32(idx), _f64(h), _f64(g)
    L, k = idx.shape
    B, m = h.shape
    dW = np.empty((L, k)); AdW = np.empty((L, k)); db = np.empty(L); Adb = np.empty(L)
    lib().oracle_weight_grad(L, m, k, B, _p(idx), _p(h), _p(g), _p(dW), _p(AdW), _p(db), _p(Adb))
    return dW, AdW, db, Adb


def input_grad(W, idx, g, m):
    """Alg. 2 without atomics.  Returns (dh[B][m], Adh)."""
    W, idx, g = _f64(W), _i32(idx), _f64(g)
    L, k = W.shape
    B = g.shape[0]
    dh = np.empty((B, m)); Adh = np.empty((B, m))
    lib().oracle_input_grad(L, m, k, B, _p(W), _p(idx), _p(g), _p(dh), _p(Adh))
    return dh, Adh


def adam(p, q, mo, ve, t, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """Adam with bias correction (readings R6/R7).  Returns new (p, m, v)."""
    p, q, mo, ve = _f64(p).copy(), _f64(q), _f64(mo).copy(), _f64(ve).copy()
    lib().oracle_adam(p.size, _p(p), _p(q), _p(mo), _p(ve), int(t), float(lr), beta1, beta2, eps)
    return p, mo, ve


def philox4x32_10(ctr, key):
    """Philox4x32-10 block function (Random123)."""
    c = np.ascontiguousarray(np.asarray(ctr, dtype=np.uint32))
    k = np.ascontiguousarray(np.asarray(key, dtype=np.uint32))
    out = np.empty(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def init(L, m, k, seed, init_scale=0.0, row_begin=0):
    """Uniform random connection init + W ~ U(+-a) (reading R17).
    init_scale 0 -> a = fp32(1/sqrt(k)).  Returns (idx int32[L][k], W float32[L][k])."""
    a = np.float32(1.0 / np.sqrt(k)) if init_scale == 0 else np.float32(init_scale)
    idx = np.empty((L, k), dtype=np.int32)
    W = np.empty((L, k), dtype=np.float32)
    lib().oracle_init(L, row_begin, m, k, seed, float(a), _p(idx), _p(W))
    return idx, W


def redistribute(W, idx, mW, vW, m, p, seed, step, row_begin=0):
    """SET prune/regrow per row.  Returns new (W, idx, mW, vW)."""
    W, mW, vW = _f64(W).copy(), _f64(mW).copy(), _f64(vW).copy()
    idx = _i32(idx).copy()
    L, k = W.shape
    lib().oracle_redistribute(L, row_begin, m, k, p, seed, step, _p(W), _p(idx), _p(mW), _p(vW))
    return W, idx, mW, vW


def topk(y, K, row_begin=0):
    """top-k by (score desc, global id asc).  Returns (scores, ids int64)."""
    y = _f64(y)
    B, L = y.shape
    s = np.empty((B, K)); ids = np.empty((B, K), dtype=np.int64)
    lib().oracle_topk(L, row_begin, B, _p(y), K, _p(s), _p(ids))
    return s, ids


def precision_at_k(ids, lbl_ptr, lbl_ids):
    """Eq. (1) averaged over instances."""
    ids = np.ascontiguousarray(np.asarray(ids, dtype=np.int64))
    B, K = ids.shape
    lp, li = _i32(lbl_ptr), _i32(lbl_ids if len(lbl_ids) else np.zeros(1, np.int32))
    return lib().oracle_precision_at_k(B, K, _p(ids), _p(lp), _p(li))


# --------------------------------------------------------------------------- state
@dataclass
class State:
    """fp64 layer state for one label shard (W, idx, bias, Adam moments, t)."""
    W: np.ndarray
    idx: np.ndarray
    bias: np.ndarray
    mW: np.ndarray
    vW: np.ndarray
    mb: np.ndarray
    vb: np.ndarray
    t: int = 0

    @staticmethod
    def create(L, m, k, seed, init_scale=0.0, row_begin=0):
        idx, W = init(L, m, k, seed, init_scale, row_begin)
        z = np.zeros((L, k)); zl = np.zeros(L)
        return State(W.astype(np.float64), idx, zl.copy(), z.copy(), z.copy(), zl.copy(), zl.copy(), 0)

    def copy(self):
        return State(self.W.copy(), self.idx.copy(), self.bias.copy(), self.mW.copy(), self.vW.copy(),
                     self.mb.copy(), self.vb.copy(), self.t)


@dataclass
class StepResult:
    y: np.ndarray
    Ay: np.ndarray
    g: np.ndarray
    loss: float
    dW: np.ndarray
    AdW: np.ndarray
    db: np.ndarray
    Adb: np.ndarray
    dh: np.ndarray
    Adh: np.ndarray


def train_step(st: State, h, lbl_ptr, lbl_ids, grad_scale, lr, row_begin=0,
               beta1=0.9, beta2=0.999, eps=1e-8, loss="bce"):
    """One training step in the paper's order: Alg. 1 forward, loss gradient (BCE, or the
    squared hinge with loss="sqh"), Alg. 3 weight gradient (+db), Alg. 2 input gradient
    with the PRE-update weights, then Adam over W and bias with the incremented global t.
    Mutates ``st``."""
    h = _f64(h)
    m = h.shape[1]
    y, Ay = forward(st.W, st.idx, st.bias, h)
    g, loss = loss_grad(loss, y, lbl_ptr, lbl_ids, grad_scale, row_begin)
    dW, AdW, db, Adb = weight_grad(st.idx, h, g)
    dh, Adh = input_grad(st.W, st.idx, g, m)
    st.t += 1
    st.W, st.mW, st.vW = adam(st.W, dW, st.mW, st.vW, st.t, lr, beta1, beta2, eps)
    st.bias, st.mb, st.vb = adam(st.bias, db, st.mb, st.vb, st.t, lr, beta1, beta2, eps)
    return StepResult(y, Ay, g, loss, dW, AdW, db, Adb, dh, Adh)


# --------------------------------------------------------------------------- NEXT-2
# The intermediate layer of the proposed architecture (Fig. 2)
# and input dropout.  Readings R25-R28.
def dropout(x, p, seed, step):
    """Inverted input dropout (reading R25).  Returns (xt[B][d], keep uint8[B][d], s)
    with s = fp32(1/(1-p)) the keep scale."""
    x = _f64(x)
    B, d = x.shape
    s = float(np.float32(1.0) / (np.float32(1.0) - np.float32(p)))
    xt = np.empty_like(x); keep = np.empty((B, d), dtype=np.uint8)
    lib().oracle_dropout(B, d, float(np.float32(p)), s, seed, step & 0xFFFFFFFF, _p(x), _p(xt), _p(keep))
    return xt, keep, s


def dense_forward(Wd, bd, xt):
    """z = xt Wd + bd, h = ReLU(z) (R18).  Returns (z, Az, h)."""
    Wd, bd, xt = _f64(Wd), _f64(bd), _f64(xt)
    d, m = Wd.shape
    B = xt.shape[0]
    z = np.empty((B, m)); Az = np.empty((B, m)); h = np.empty((B, m))
    lib().oracle_dense_forward(B, d, m, _p(Wd), _p(bd), _p(xt), _p(z), _p(Az), _p(h))
    return z, Az, h


def dense_backward(xt, z, dh):
    """dz = dh [z > 0]; dWd = xt^T dz; dbd = sum_b dz (R26).  Returns (dWd, AdWd, dbd, Adbd)."""
    xt, z, dh = _f64(xt), _f64(z), _f64(dh)
    B, d = xt.shape
    m = z.shape[1]
    dWd = np.empty((d, m)); AdWd = np.empty((d, m)); dbd = np.empty(m); Adbd = np.empty(m)
    lib().oracle_dense_backward(B, d, m, _p(xt), _p(z), _p(dh), _p(dWd), _p(AdWd), _p(dbd), _p(Adbd))
    return dWd, AdWd, dbd, Adbd


def dense_init(d, m, seed, init_scale=0.0):
    """Glorot-uniform Wd (reading R27) from the Philox domain-4 stream.  Returns float32 [d][m]."""
    a = np.float32(np.sqrt(6.0 / (d + m))) if init_scale == 0 else np.float32(init_scale)
    Wd = np.empty((d, m), dtype=np.float32)
    lib().oracle_dense_init(d, m, seed, float(a), _p(Wd))
    return Wd


@dataclass
class DenseState:
    """fp64 state of the dense intermediate layer (Wd, bd, Adam moments, its own t)."""
    Wd: np.ndarray
    bd: np.ndarray
    mWd: np.ndarray
    vWd: np.ndarray
    mbd: np.ndarray
    vbd: np.ndarray
    t: int = 0

    @staticmethod
    def create(d, m, seed, init_scale=0.0):
        Wd = dense_init(d, m, seed, init_scale).astype(np.float64)
        z = np.zeros((d, m)); zm = np.zeros(m)
        return DenseState(Wd, zm.copy(), z.copy(), z.copy(), zm.copy(), zm.copy(), 0)

    def copy(self):
        return DenseState(self.Wd.copy(), self.bd.copy(), self.mWd.copy(), self.vWd.copy(), self.mbd.copy(),
                          self.vbd.copy(), self.t)


@dataclass
class ModelStepResult:
    xt: np.ndarray
    keep: np.ndarray
    z: np.ndarray
    Az: np.ndarray
    h: np.ndarray
    sparse: StepResult
    dWd: np.ndarray
    AdWd: np.ndarray
    dbd: np.ndarray
    Adbd: np.ndarray


def model_train_step(ds: DenseState, st: State, x, step, dropout_p, seed, lbl_ptr, lbl_ids, grad_scale, lr,
                     beta1=0.9, beta2=0.999, eps=1e-8, loss="bce"):
    """One step of the proposed architecture (Fig. 2): input dropout, dense
    intermediate layer + ReLU, the sparse layer's step (train_step above; its dh
    uses the pre-update sparse weights), then the dense layer's backward and Adam (its own
    global t, reading R28).  Mutates ``ds`` and ``st``."""
    xt, keep, _ = dropout(x, dropout_p, seed, step)
    z, Az, h = dense_forward(ds.Wd, ds.bd, xt)
    r = train_step(st, h, lbl_ptr, lbl_ids, grad_scale, lr, beta1=beta1, beta2=beta2, eps=eps, loss=loss)
    dWd, AdWd, dbd, Adbd = dense_backward(xt, z, r.dh)
    ds.t += 1
    ds.Wd, ds.mWd, ds.vWd = adam(ds.Wd, dWd, ds.mWd, ds.vWd, ds.t, lr, beta1, beta2, eps)
    ds.bd, ds.mbd, ds.vbd = adam(ds.bd, dbd, ds.mbd, ds.vbd, ds.t, lr, beta1, beta2, eps)
    return ModelStepResult(xt, keep, z, Az, h, r, dWd, AdWd, dbd, Adbd)
