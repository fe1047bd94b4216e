"""Thin ctypes binding of ``libfixedfanin.so`` (C ABI in include/fixedfanin.h).

Argument marshalling only: every step of the hot path runs in the library's sm_100a
kernels.  PyTorch provides device memory (the workspace, inputs, outputs) and streams.
There is no CPU fallback: if the library is missing, loading raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FIXEDFANIN_LIB") or os.path.join(_HERE, "libfixedfanin.so")   # env: dev sweeps only

FF_OK, FF_ERR_ARG, FF_ERR_CONFIG, FF_ERR_RANGE, FF_ERR_NONFINITE, FF_ERR_CUDA, FF_ERR_STATE = range(7)
FF_FLAG_CHECK_FINITE = 1
FF_FLAG_STORE_GRADS = 2
FF_FLAG_NO_PIPE = 4
FF_FLAG_DENSE_SIMT = 8
FF_STEP_AUTO = 2 ** 64 - 1     # dropout keyed on the dense layer's device Adam counter + 1
FF_DH_ATOMIC, FF_DH_CSC, FF_DH_HYBRID = 0, 1, 2
FF_LOSS_BCE, FF_LOSS_SQH = 0, 1
FF_MAX_FANIN, FF_MAX_BATCH, FF_MAX_TOPK = 64, 1024, 8
_STATUS = {1: "FF_ERR_ARG", 2: "FF_ERR_CONFIG", 3: "FF_ERR_RANGE", 4: "FF_ERR_NONFINITE", 5: "FF_ERR_CUDA",
           6: "FF_ERR_STATE"}

EXPORTS = [
    "fixedfanin_workspace_size", "fixedfanin_create", "fixedfanin_destroy", "fixedfanin_set_params",
    "fixedfanin_get_params", "fixedfanin_forward", "fixedfanin_backward", "fixedfanin_get_grads",
    "fixedfanin_adam_step", "fixedfanin_train_step", "fixedfanin_train_step_host", "fixedfanin_redistribute",
    "fixedfanin_predict_topk", "fixedfanin_score_shortlist", "fixedfanin_merge_topk", "fixedfanin_check",
    "fixedfanin_precision_at_k",
    "fixedfanin_profile_begin",
    "fixedfanin_profile_end", "fixedfanin_profile_pause", "fixedfanin_last_launch_count",
    "fixedfanin_last_error",
    # NEXT-2: the intermediate layer and the whole architecture
    "fixedfanin_dense_workspace_size", "fixedfanin_dense_create", "fixedfanin_dense_destroy",
    "fixedfanin_dense_set_params", "fixedfanin_dense_get_params", "fixedfanin_dense_forward",
    "fixedfanin_dense_backward_adam", "fixedfanin_dense_get_grads", "fixedfanin_model_train_step",
    "fixedfanin_model_predict_topk",
]


class FFError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class ff_config(ctypes.Structure):
    _fields_ = [
        ("L_global", ctypes.c_int64), ("row_begin", ctypes.c_int64), ("L_local", ctypes.c_int64),
        ("m", ctypes.c_int32), ("k", ctypes.c_int32), ("max_batch", ctypes.c_int32),
        ("max_topk", ctypes.c_int32), ("max_nnz", ctypes.c_int32), ("dh_mode", ctypes.c_int32),
        ("seed", ctypes.c_uint64), ("init_scale", ctypes.c_float), ("beta1", ctypes.c_float),
        ("beta2", ctypes.c_float), ("eps", ctypes.c_float), ("prune_frac", ctypes.c_float),
        ("flags", ctypes.c_uint32), ("loss", ctypes.c_int32), ("hybrid_frac", ctypes.c_float),
    ]


class ff_dense_config(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32), ("m", ctypes.c_int32), ("max_batch", ctypes.c_int32), ("col_begin", ctypes.c_int32),
        ("seed", ctypes.c_uint64), ("init_scale", ctypes.c_float), ("dropout", ctypes.c_float),
        ("beta1", ctypes.c_float), ("beta2", ctypes.c_float), ("eps", ctypes.c_float), ("flags", ctypes.c_uint32),
        ("m_global", ctypes.c_int32),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load the CUDA library (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not found: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        P, i32, i64, u64, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float
        sig = {
            "fixedfanin_workspace_size": [P, P],
            "fixedfanin_create": [P, P, ctypes.c_size_t, P, P],
            "fixedfanin_destroy": [P],
            "fixedfanin_set_params": [P, P, P, P, P, P, P, P, P, P],
            "fixedfanin_get_params": [P, P, P, P, P, P, P, P, P, P],
            "fixedfanin_forward": [P, P, i32, P, P],
            "fixedfanin_backward": [P, P, P, i32, P, P, f32, P, P, P],
            "fixedfanin_get_grads": [P, P, P, P],
            "fixedfanin_adam_step": [P, f32, P],
            "fixedfanin_train_step": [P, P, i32, P, P, f32, f32, P, P, P],
            "fixedfanin_train_step_host": [P, P, i32, P, P, f32, f32, P, P, P],
            "fixedfanin_redistribute": [P, u64, P],
            "fixedfanin_predict_topk": [P, P, i32, i32, P, P, P],
            "fixedfanin_merge_topk": [P, P, i32, i32, i32, P, P, P],
            "fixedfanin_precision_at_k": [P, i32, i32, P, P, P, P, P],
            "fixedfanin_score_shortlist": [P, P, i32, P, P, P, P],
            "fixedfanin_check": [P, P],
            "fixedfanin_profile_begin": [P, i32],
            "fixedfanin_profile_end": [P, P, P],
            "fixedfanin_profile_pause": [P, i32],
            "fixedfanin_dense_workspace_size": [P, P],
            "fixedfanin_dense_create": [P, P, ctypes.c_size_t, P, P],
            "fixedfanin_dense_destroy": [P],
            "fixedfanin_dense_set_params": [P, P, P, P, P, P, P, P, P],
            "fixedfanin_dense_get_params": [P, P, P, P, P, P, P, P, P],
            "fixedfanin_dense_forward": [P, P, i32, u64, i32, P, P],
            "fixedfanin_dense_backward_adam": [P, P, i32, f32, P],
            "fixedfanin_dense_get_grads": [P, P, P, P],
            "fixedfanin_model_train_step": [P, P, P, i32, u64, P, P, f32, f32, P, P],
            "fixedfanin_model_predict_topk": [P, P, P, i32, i32, P, P, P],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.fixedfanin_last_launch_count.argtypes = []
        L.fixedfanin_last_launch_count.restype = i32
        L.fixedfanin_last_error.argtypes = []
        L.fixedfanin_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(status: int):
    if status != FF_OK:
        raise FFError(status, lib().fixedfanin_last_error().decode())


def _ptr(t):
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "device tensors must be contiguous CUDA tensors"
    return ctypes.c_void_p(t.data_ptr())


def _hptr(t):
    if t is None:
        return None
    assert (not t.is_cuda) and t.is_contiguous()
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def last_launch_count() -> int:
    return int(lib().fixedfanin_last_launch_count())


@dataclass
class LayerConfig:
    L_global: int
    m: int
    k: int
    row_begin: int = 0
    L_local: int | None = None
    max_batch: int = 32
    max_topk: int = 8
    max_nnz: int = 0
    dh_mode: int = FF_DH_ATOMIC
    seed: int = 42
    init_scale: float = 0.0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    prune_frac: float = 0.1
    flags: int = 0
    loss: int = FF_LOSS_BCE
    hybrid_frac: float = 0.0

    def c(self) -> ff_config:
        L_local = self.L_global - self.row_begin if self.L_local is None else self.L_local
        return ff_config(self.L_global, self.row_begin, L_local, self.m, self.k, self.max_batch, self.max_topk,
                         self.max_nnz, self.dh_mode, self.seed, self.init_scale, self.beta1, self.beta2, self.eps,
                         self.prune_frac, self.flags, self.loss, self.hybrid_frac)


def workspace_size(cfg: LayerConfig) -> int:
    n = ctypes.c_size_t(0)
    c = cfg.c()
    _check(lib().fixedfanin_workspace_size(ctypes.byref(c), ctypes.byref(n)))
    return int(n.value)


class FixedFanInLayer:
    """One label shard [row_begin, row_begin + L_local) of the fixed fan-in layer on one GPU."""

    def __init__(self, cfg: LayerConfig, device=None, stream=None):
        self.cfg = cfg
        self._c = cfg.c()
        self.L_local = int(self._c.L_local)
        self.device = torch.device(device if device is not None else "cuda")
        nbytes = workspace_size(cfg)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self._h = ctypes.c_void_p()
        _check(lib().fixedfanin_create(ctypes.byref(self._c), _ptr(self.workspace), nbytes, _stream(stream),
                                       ctypes.byref(self._h)))
        self.m, self.k = cfg.m, cfg.k

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().fixedfanin_destroy(h)
            except Exception:
                pass
            self._h = None

    # ------------------------------------------------------------------ state
    def get_params(self, stream=None):
        L, k, d = self.L_local, self.k, self.device
        W = torch.empty((L, k), dtype=torch.float32, device=d)
        idx = torch.empty((L, k), dtype=torch.int32, device=d)
        bias, mb, vb = (torch.empty(L, dtype=torch.float32, device=d) for _ in range(3))
        mW, vW = torch.empty_like(W), torch.empty_like(W)
        t = ctypes.c_int64(0)
        _check(lib().fixedfanin_get_params(self._h, _ptr(W), _ptr(idx), _ptr(bias), _ptr(mW), _ptr(vW), _ptr(mb),
                                           _ptr(vb), ctypes.byref(t), _stream(stream)))
        return dict(W=W, idx=idx, bias=bias, mW=mW, vW=vW, mb=mb, vb=vb, t=int(t.value))

    def set_params(self, W=None, idx=None, bias=None, mW=None, vW=None, mb=None, vb=None, t=None, stream=None):
        tt = ctypes.c_int64(int(t)) if t is not None else None
        _check(lib().fixedfanin_set_params(self._h, _ptr(W), _ptr(idx), _ptr(bias), _ptr(mW), _ptr(vW), _ptr(mb),
                                           _ptr(vb), ctypes.byref(tt) if tt is not None else None, _stream(stream)))

    # ------------------------------------------------------------------ path
    def forward(self, h, y=None, stream=None):
        B = h.shape[0]
        if y is None:
            y = torch.empty((B, self.L_local), dtype=torch.float32, device=self.device)
        _check(lib().fixedfanin_forward(self._h, _ptr(h), B, _ptr(y), _stream(stream)))
        return y

    def backward(self, h, y, lbl_ptr, lbl_ids, grad_scale=None, dh=None, loss=None, stream=None):
        B = h.shape[0]
        gs = 1.0 / max(B, 1) if grad_scale is None else grad_scale
        if dh is None:
            dh = torch.empty((B, self.m), dtype=torch.float32, device=self.device)
        if loss is None:
            loss = torch.empty(1, dtype=torch.float32, device=self.device)
        _check(lib().fixedfanin_backward(self._h, _ptr(h), _ptr(y), B, _ptr(lbl_ptr), _ptr(lbl_ids), gs, _ptr(dh),
                                         _ptr(loss), _stream(stream)))
        return dh, loss

    def get_grads(self, stream=None):
        dW = torch.empty((self.L_local, self.k), dtype=torch.float32, device=self.device)
        db = torch.empty(self.L_local, dtype=torch.float32, device=self.device)
        _check(lib().fixedfanin_get_grads(self._h, _ptr(dW), _ptr(db), _stream(stream)))
        return dW, db

    def adam_step(self, lr, stream=None):
        _check(lib().fixedfanin_adam_step(self._h, lr, _stream(stream)))

    def train_step(self, h, lbl_ptr, lbl_ids, lr, grad_scale=None, dh=None, loss=None, stream=None):
        B = h.shape[0]
        gs = 1.0 / max(B, 1) if grad_scale is None else grad_scale
        if dh is None:
            dh = torch.empty((B, self.m), dtype=torch.float32, device=self.device)
        _check(lib().fixedfanin_train_step(self._h, _ptr(h), B, _ptr(lbl_ptr), _ptr(lbl_ids), gs, lr, _ptr(dh),
                                           _ptr(loss), _stream(stream)))
        return dh, loss

    def train_step_host(self, h_host, lbl_ptr_host, lbl_ids_host, lr, grad_scale=None, dh_host=None,
                        loss_host=None, stream=None):
        B = h_host.shape[0]
        gs = 1.0 / max(B, 1) if grad_scale is None else grad_scale
        _check(lib().fixedfanin_train_step_host(self._h, _hptr(h_host), B, _hptr(lbl_ptr_host), _hptr(lbl_ids_host),
                                                gs, lr, _hptr(dh_host), _hptr(loss_host), _stream(stream)))

    def redistribute(self, step, stream=None):
        _check(lib().fixedfanin_redistribute(self._h, int(step), _stream(stream)))

    def predict_topk(self, h, K, stream=None):
        B = h.shape[0]
        scores = torch.empty((B, K), dtype=torch.float32, device=self.device)
        ids = torch.empty((B, K), dtype=torch.int32, device=self.device)
        _check(lib().fixedfanin_predict_topk(self._h, _ptr(h), B, K, _ptr(scores), _ptr(ids), _stream(stream)))
        return scores, ids

    def score_shortlist(self, h, cand_ptr, cand_ids, scores=None, stream=None):
        """Scores y[b, cand_ids[p]] of a CSR shortlist; +0 for labels of other
        shards.  h [B][m], cand_ptr int32 [B+1], cand_ids int32 [nnz] (device)."""
        B = h.shape[0]
        if scores is None:
            scores = torch.empty(cand_ids.shape[0], dtype=torch.float32, device=self.device)
        _check(lib().fixedfanin_score_shortlist(self._h, _ptr(h), B, _ptr(cand_ptr), _ptr(cand_ids), _ptr(scores),
                                                _stream(stream)))
        return scores

    def profile_begin(self, max_launches: int):
        _check(lib().fixedfanin_profile_begin(self._h, int(max_launches)))

    def profile_pause(self, paused: bool):
        _check(lib().fixedfanin_profile_pause(self._h, 1 if paused else 0))

    def profile_end(self):
        """-> (summed fused-kernel milliseconds, number of timed launches)"""
        ms, n = ctypes.c_double(0), ctypes.c_int32(0)
        _check(lib().fixedfanin_profile_end(self._h, ctypes.byref(ms), ctypes.byref(n)))
        return float(ms.value), int(n.value)

    def check(self, stream=None):
        _check(lib().fixedfanin_check(self._h, _stream(stream)))


def merge_topk(scores, ids, stream=None):
    """Merge per-shard top-K lists [P][B][K] -> [B][K] on the device (exact total order)."""
    P, B, K = scores.shape
    out_s = torch.empty((B, K), dtype=torch.float32, device=scores.device)
    out_i = torch.empty((B, K), dtype=torch.int32, device=scores.device)
    # the contiguous copies stay bound until the (asynchronous) kernel was enqueued on `stream`:
    # a temporary freed inside the argument list could hand its block to the next temporary
    sc, ic = scores.contiguous(), ids.contiguous()
    _check(lib().fixedfanin_merge_topk(_ptr(sc), _ptr(ic), P, B, K, _ptr(out_s), _ptr(out_i), _stream(stream)))
    return out_s, out_i


def precision_at_k(ids, lbl_ptr, lbl_ids, stream=None):
    """Eq. (1) on the GPU: (hits int32 [B], mean P@K float32 [1]) of predicted
    GLOBAL ids [B][K] against the positives' CSR (device tensors)."""
    B, K = ids.shape
    hits = torch.empty(B, dtype=torch.int32, device=ids.device)
    mean = torch.empty(1, dtype=torch.float32, device=ids.device)
    ic, pc, lc = ids.contiguous(), lbl_ptr.contiguous(), lbl_ids.contiguous()     # bound: see merge_topk
    _check(lib().fixedfanin_precision_at_k(_ptr(ic), B, K, _ptr(pc), _ptr(lc), _ptr(hits), _ptr(mean),
                                           _stream(stream)))
    return hits, mean


# ------------------------------------------------------------------ NEXT-2
@dataclass
class DenseConfig:
    """The intermediate layer of the proposed architecture (Fig. 2), or the column
    shard [col_begin, col_begin + m) of a layer m_global wide."""
    d: int
    m: int
    max_batch: int = 32
    seed: int = 7
    init_scale: float = 0.0
    dropout: float = 0.0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    flags: int = 0
    col_begin: int = 0
    m_global: int = 0

    def c(self) -> ff_dense_config:
        return ff_dense_config(self.d, self.m, self.max_batch, self.col_begin, self.seed, self.init_scale, self.dropout,
                               self.beta1, self.beta2, self.eps, self.flags, self.m_global)


class DenseLayer:
    """Input dropout -> dense Wd -> ReLU on one GPU (a replica under label sharding)."""

    def __init__(self, cfg: DenseConfig, device=None, stream=None):
        self.cfg = cfg
        self._c = cfg.c()
        self.device = torch.device(device if device is not None else "cuda")
        n = ctypes.c_size_t(0)
        _check(lib().fixedfanin_dense_workspace_size(ctypes.byref(self._c), ctypes.byref(n)))
        self.workspace = torch.empty(int(n.value), dtype=torch.uint8, device=self.device)
        self._h = ctypes.c_void_p()
        _check(lib().fixedfanin_dense_create(ctypes.byref(self._c), _ptr(self.workspace), int(n.value),
                                             _stream(stream), ctypes.byref(self._h)))
        self.d, self.m = cfg.d, cfg.m

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().fixedfanin_dense_destroy(h)
            except Exception:
                pass
            self._h = None

    def get_params(self, stream=None):
        d, m, dev = self.d, self.m, self.device
        Wd, mWd, vWd = (torch.empty((d, m), dtype=torch.float32, device=dev) for _ in range(3))
        bd, mbd, vbd = (torch.empty(m, dtype=torch.float32, device=dev) for _ in range(3))
        t = ctypes.c_int64(0)
        _check(lib().fixedfanin_dense_get_params(self._h, _ptr(Wd), _ptr(bd), _ptr(mWd), _ptr(vWd), _ptr(mbd),
                                                 _ptr(vbd), ctypes.byref(t), _stream(stream)))
        return dict(Wd=Wd, bd=bd, mWd=mWd, vWd=vWd, mbd=mbd, vbd=vbd, t=int(t.value))

    def set_params(self, Wd=None, bd=None, mWd=None, vWd=None, mbd=None, vbd=None, t=None, stream=None):
        tt = ctypes.c_int64(int(t)) if t is not None else None
        _check(lib().fixedfanin_dense_set_params(self._h, _ptr(Wd), _ptr(bd), _ptr(mWd), _ptr(vWd), _ptr(mbd),
                                                 _ptr(vbd), ctypes.byref(tt) if tt is not None else None,
                                                 _stream(stream)))

    def forward(self, x, step=None, train=True, h=None, stream=None):
        """step keys the dropout mask (R25).  None: FF_STEP_AUTO for a training forward (the
        device Adam counter + 1, so consecutive training steps draw fresh masks), 0 for
        inference (no dropout is applied then)."""
        B = x.shape[0]
        if step is None:
            step = FF_STEP_AUTO if train else 0
        if h is None:
            h = torch.empty((B, self.m), dtype=torch.float32, device=self.device)
        _check(lib().fixedfanin_dense_forward(self._h, _ptr(x), B, int(step), 1 if train else 0, _ptr(h),
                                              _stream(stream)))
        return h

    def backward_adam(self, dh, lr, stream=None):
        _check(lib().fixedfanin_dense_backward_adam(self._h, _ptr(dh), dh.shape[0], lr, _stream(stream)))

    def get_grads(self, stream=None):
        dWd = torch.empty((self.d, self.m), dtype=torch.float32, device=self.device)
        dbd = torch.empty(self.m, dtype=torch.float32, device=self.device)
        _check(lib().fixedfanin_dense_get_grads(self._h, _ptr(dWd), _ptr(dbd), _stream(stream)))
        return dWd, dbd


def model_train_step(dense: DenseLayer, layer: FixedFanInLayer, x, step, lbl_ptr, lbl_ids, lr, grad_scale=None,
                     loss=None, stream=None):
    """One step of the whole architecture (dropout -> dense -> ReLU -> fixed fan-in -> loss ->
    backward through both layers -> Adam on both) through fixedfanin_model_train_step.
    step keys the dropout mask; None = FF_STEP_AUTO (the dense layer's device counter + 1)."""
    B = x.shape[0]
    if step is None:
        step = FF_STEP_AUTO
    gs = 1.0 / max(B, 1) if grad_scale is None else grad_scale
    _check(lib().fixedfanin_model_train_step(dense._h, layer._h, _ptr(x), B, int(step), _ptr(lbl_ptr), _ptr(lbl_ids),
                                             gs, lr, _ptr(loss), _stream(stream)))
    return loss


def model_predict_topk(dense: DenseLayer, layer: FixedFanInLayer, x, K, stream=None):
    B = x.shape[0]
    scores = torch.empty((B, K), dtype=torch.float32, device=layer.device)
    ids = torch.empty((B, K), dtype=torch.int32, device=layer.device)
    _check(lib().fixedfanin_model_predict_topk(dense._h, layer._h, _ptr(x), B, K, _ptr(scores), _ptr(ids),
                                               _stream(stream)))
    return scores, ids
