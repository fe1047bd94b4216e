"""Seeded synthetic inputs shaped like the paper's workloads.

This module holds NONE of the method's arithmetic: it only draws the hidden batch h,
the sparse positive-label sets and names the benchmark shapes.  It is the one module
both the CUDA path's tests/bench and the oracle's tests feed from (numpy only; it
imports neither the oracle nor the CUDA binding).

* h = ReLU(N(0,1)) float32 [B][m]: h is the output of the (ReLU) intermediate layer
  the sparse layer reads (activation per S:345), ~50% exact zeros.
* labels: n_pos ~ 1 + Poisson(avg - 1) capped at 200 and at L; ids drawn Zipf(1.0)
  over a fixed random permutation of [0, L) (so popular labels spread over shards),
  sorted and unique per instance.  avg = public XMC-repository label statistics
  (not in the paper; SURVEY §8(d) "[ext.]").
* B = 32 ("each consisting of 32 samples in a minibatch").
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

DATA_SEED = 1234
PARAM_SEED = 42


@dataclass(frozen=True)
class Shape:
    name: str
    L: int           # labels ("numlabels")
    m: int           # width of the layer the sparse layer reads (intermediate, "32k")
    k: int           # connections per label (the paper's s; "Uniform-32")
    B: int           # mini-batch
    avg_pos: float   # mean positives per instance [ext.]


SHAPES = {
    "tiny": Shape("tiny", 1000, 256, 16, 32, 5.0),
    "wiki10-31k": Shape("wiki10-31k", 30938, 32768, 32, 32, 18.64),
    "wiki-500k": Shape("wiki-500k", 501070, 32768, 32, 32, 4.77),
    "amazon-670k": Shape("amazon-670k", 670091, 32768, 32, 32, 5.45),
    "amazon-3m": Shape("amazon-3m", 2812281, 32768, 32, 32, 36.04),
    # sweeps of SURVEY §8(d): the paper's Table-5 architecture (64 nnz/label, 65k intermediate,
    # P:869-870) and the 16k intermediate of the loss comparison
    "amazon-670k-k64-m65k": Shape("amazon-670k-k64-m65k", 670091, 65536, 64, 32, 5.45),
    "amazon-670k-m16k": Shape("amazon-670k-m16k", 670091, 16384, 32, 32, 5.45),
}


# The proposed architecture's fixed input features: 512-d fastText-based (Slice)
# or 768-d CascadeXML embeddings; input dropout 10% for Amazon-670K / Wiki-500K Slice, 20% for
# Wiki10 / Wiki-500K Cascade.  NEXT-2 of SURVEY §8(f).
FEATURE_DIMS = {"slice": 512, "cascade": 768}
DROPOUT = {"amazon-670k": 0.1, "wiki-500k": 0.1, "wiki10-31k": 0.2}


def _rng(seed: int, step: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, step, stream])))


def hidden_batch(B: int, m: int, step: int = 0, seed: int = DATA_SEED) -> np.ndarray:
    """h[B][m] float32 = ReLU(N(0,1)), a fresh batch per step."""
    z = _rng(seed, step, 1).standard_normal((B, m), dtype=np.float32)
    return np.maximum(z, np.float32(0.0))


def signed_hidden_batch(B: int, m: int, step: int = 0, seed: int = DATA_SEED, scale: float = 1.0) -> np.ndarray:
    """h[B][m] float32 = scale * N(0,1) without the ReLU: signed inputs for the parity tests
    of regimes a post-ReLU h never reaches (negative h, saturated logits)."""
    return (_rng(seed, step, 5).standard_normal((B, m), dtype=np.float32) * np.float32(scale)).astype(np.float32)


def feature_batch(B: int, d: int, step: int = 0, seed: int = DATA_SEED) -> np.ndarray:
    """x[B][d] float32 ~ N(0,1): stand-in for the fixed dense embeddings (no dataset)."""
    return _rng(seed, step, 3).standard_normal((B, d), dtype=np.float32)


@lru_cache(maxsize=8)
def _zipf_table(L: int, seed: int):
    w = 1.0 / np.arange(1, L + 1, dtype=np.float64)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    perm = _rng(seed, 0, 7).permutation(L).astype(np.int64)
    return cdf, perm


def label_batch(B: int, L: int, avg_pos: float, step: int = 0, seed: int = DATA_SEED,
                cap: int = 200):
    """Sparse positives as CSR (ptr int32[B+1], ids int32[nnz]); ids sorted/unique per row."""
    r = _rng(seed, step, 2)
    cdf, perm = _zipf_table(L, seed)
    cap = min(cap, L)
    ptr = np.zeros(B + 1, dtype=np.int32)
    rows = []
    for b in range(B):
        n = int(min(cap, 1 + r.poisson(max(avg_pos - 1.0, 0.0))))
        chosen: set = set()
        while len(chosen) < n:
            u = r.random(2 * n)
            ranks = np.searchsorted(cdf, u, side="right")
            for q in ranks:
                chosen.add(int(perm[min(int(q), L - 1)]))
                if len(chosen) == n:
                    break
        ids = np.array(sorted(chosen), dtype=np.int32)
        rows.append(ids)
        ptr[b + 1] = ptr[b] + len(ids)
    ids = np.concatenate(rows) if rows else np.zeros(0, dtype=np.int32)
    return ptr, ids.astype(np.int32)


def random_params(L: int, m: int, k: int, seed: int, scale: float = 0.2):
    """Arbitrary valid (W, idx, bias) for parity tests that bypass the Philox init:
    idx rows are k distinct draws from [0, m); W, bias ~ U(-scale, scale) float32."""
    r = _rng(seed, 0, 3)
    idx = np.empty((L, k), dtype=np.int32)
    for j in range(L):
        idx[j] = r.choice(m, size=k, replace=False)
    W = r.uniform(-scale, scale, size=(L, k)).astype(np.float32)
    bias = r.uniform(-scale, scale, size=L).astype(np.float32)
    return W, idx, bias


def random_labels_uniform(B: int, L: int, n_pos: int, seed: int):
    """Small-case labels: n_pos distinct uniform ids per instance (CSR, sorted)."""
    r = _rng(seed, 0, 4)
    ptr = np.zeros(B + 1, dtype=np.int32)
    rows = []
    for b in range(B):
        n = min(n_pos, L)
        ids = np.sort(r.choice(L, size=n, replace=False)).astype(np.int32)
        rows.append(ids)
        ptr[b + 1] = ptr[b] + n
    return ptr, (np.concatenate(rows) if rows else np.zeros(0, np.int32)).astype(np.int32)
