"""CPU-only checks of the C-ABI library: it loads, exports every symbol the header
declares, sizes workspaces and rejects bad configurations — no compute calls (no GPU)."""
import ctypes
import os
import re

import pytest

from paper_2306_03725_b200 import layer as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__ as g
    g.build_lib()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "fixedfanin.h")).read()
    return sorted(set(re.findall(r"\b(fixedfanin_\w+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 15
    lib = L.lib()
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(L.EXPORTS)


def test_no_torch_types_in_header():
    txt = open(os.path.join(ROOT, "include", "fixedfanin.h")).read()
    assert "torch" not in txt.lower().replace("pytorch", "") and "at::" not in txt


def test_workspace_size_matches_layout_model():
    cfg = L.LayerConfig(L_global=670091, m=32768, k=32, max_batch=32)
    n = L.workspace_size(cfg)
    Lk = 670091 * 32
    state = 5 * 4 * Lk + 4 * 4 * 670091 + 4 * 670091          # W idx mW vW dW, bias mb vb db, posmask
    # hd (h|dh lines), top-K candidates, double-buffered h and label staging + dh staging (host entry point)
    scratch = 2 * 4 * 32768 * 32 + 2 * 4 * 1024 * 32 * 8 + 4 * 32 + 3 * 4 * 32 * 32768 + 2 * 4 * (33 + 64 * 32)
    assert state <= n <= state + scratch + 32 * 256
    assert n % 256 == 0


@pytest.mark.parametrize("kw,msg", [
    (dict(L_global=10, m=8, k=9), "k="),            # k > m
    (dict(L_global=10, m=128, k=65), "k="),         # k > FF_MAX_FANIN (64)
    (dict(L_global=10, m=64, k=8, row_begin=5, L_local=6), "shard"),
    (dict(L_global=10, m=64, k=8, max_batch=1025), "max_batch"),
    (dict(L_global=10, m=64, k=8, max_topk=9), "max_topk"),
    (dict(L_global=2 ** 31, m=64, k=8), "L_global"),
    (dict(L_global=10, m=64, k=8, prune_frac=1.0), "prune_frac"),
    # 32-bit connection offsets in every dh mode: 2^26 rows x 32 = 2^31
    (dict(L_global=2 ** 26, m=64, k=32), "connections per shard"),
    (dict(L_global=2 ** 26, m=64, k=32, dh_mode=L.FF_DH_CSC), "connections per shard"),
    (dict(L_global=2 ** 30, m=64, k=64, row_begin=2 ** 20, L_local=2 ** 25), "connections per shard"),
])
def test_bad_configs_rejected(kw, msg):
    with pytest.raises(L.FFError) as e:
        L.workspace_size(L.LayerConfig(**kw))
    assert e.value.status == L.FF_ERR_CONFIG and msg in str(e.value)


def test_largest_shard_below_the_offset_limit_is_accepted():
    """L_local * k = 2^31 - 32 connections: the last shard size the 32-bit offsets allow."""
    n = L.workspace_size(L.LayerConfig(L_global=2 ** 26 - 1, m=64, k=32, max_batch=32))
    assert n >= 5 * 4 * (2 ** 31 - 32)


def test_create_without_gpu_fails_loudly():
    """No CPU fallback: creating a layer on a machine without a usable GPU is an error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = L.LayerConfig(L_global=100, m=64, k=8).c()
    buf = (ctypes.c_char * (1 << 20))()
    aligned = (ctypes.addressof(buf) + 255) // 256 * 256
    out = ctypes.c_void_p()
    st = L.lib().fixedfanin_create(ctypes.byref(cfg), ctypes.c_void_p(aligned), 1 << 19, None, ctypes.byref(out))
    assert st != L.FF_OK


def test_merge_topk_argument_validation():
    st = L.lib().fixedfanin_merge_topk(None, None, 0, 1, 1, None, None, None)
    assert st == L.FF_ERR_ARG
    assert b"P" in L.lib().fixedfanin_last_error()


@pytest.mark.parametrize("kw,msg", [
    (dict(d=0, m=64), "d="),
    (dict(d=16, m=0), "m="),
    (dict(d=16, m=64, max_batch=0), "max_batch"),
    (dict(d=16, m=64, max_batch=1025), "max_batch"),
    (dict(d=16, m=64, dropout=1.0), "dropout"),
    (dict(d=16, m=64, dropout=-0.1), "dropout"),
    (dict(d=16, m=64, beta1=1.0), "Adam"),
    (dict(d=16, m=64, col_begin=10, m_global=70), "column shard"),     # [10, 74) outside [0, 70)
    (dict(d=16, m=64, col_begin=-1, m_global=70), "column shard"),
])
def test_bad_dense_configs_rejected(kw, msg):
    c = L.DenseConfig(**kw).c()
    n = ctypes.c_size_t(0)
    st = L.lib().fixedfanin_dense_workspace_size(ctypes.byref(c), ctypes.byref(n))
    assert st == L.FF_ERR_CONFIG and msg in L.lib().fixedfanin_last_error().decode()


def test_dense_workspace_size_matches_layout_model():
    """Wd, mWd, vWd in 128-column tiles (+ dWd with FF_FLAG_STORE_GRADS), bias vectors, xT and
    its tf32 lo part (the TMA forward), the split-forward scratch, the h|dh lines and the x
    staging."""
    d, m, B = 512, 32768, 32
    sizes = []
    for flags in (0, L.FF_FLAG_STORE_GRADS):
        c = L.DenseConfig(d=d, m=m, max_batch=B, flags=flags).c()
        n = ctypes.c_size_t(0)
        assert L.lib().fixedfanin_dense_workspace_size(ctypes.byref(c), ctypes.byref(n)) == L.FF_OK
        sizes.append(n.value)
    assert sizes[1] - sizes[0] == 4 * d * m                     # dWd
    core = 3 * 4 * d * m + 4 * 4 * m + 2 * 4 * d * 32 + 8 * m * 32 + 4 * B * d
    assert core <= sizes[0] <= core + 2 * 4 * m * 32 + 4 * (m // 128) + 16 * 256


def test_python_constants_match_header_defines():
    """The binding's FF_* constants equal the header's #defines and enum values."""
    import os
    import re
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "fixedfanin.h")).read()
    defines = {k: v for k, v in re.findall(r"#define\s+(FF_\w+)\s+(\w+)", hdr)}
    enums = {k: int(v) for k, v in re.findall(r"\b(FF_\w+)\s*=\s*(\d+)", hdr)}
    checked = 0
    for name, val in defines.items():
        if not hasattr(L, name):
            continue
        want = 2 ** 64 - 1 if val == "UINT64_MAX" else int(val.rstrip("uU"), 0)
        assert getattr(L, name) == want, name
        checked += 1
    for name, val in enums.items():
        if hasattr(L, name):
            assert getattr(L, name) == val, name
            checked += 1
    assert checked >= 8
