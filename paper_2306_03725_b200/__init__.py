"""B200-native fixed fan-in (uniform sparsity) sparse output layer, arXiv 2306.03725.

The hot path lives in the CUDA library ``libfixedfanin.so`` (sm_100a) behind the C ABI
declared in ``include/fixedfanin.h``; ``layer.py`` is the thin ctypes binding and
``sharded.py`` the label-sharded multi-GPU driver.  Importing this package does not load
the library; the first use does, and fails loudly if it is missing (no CPU fallback).
"""
__all__ = ["synth", "layer", "sharded"]
