import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a); run with -m gpu")


def read_golden(name):
    """Lines of a golden fixture without comments/blank lines."""
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.strip() for ln in f if ln.strip() and not ln.lstrip().startswith("#")]


def fig1c():
    """Parse tests/golden/fig1c.txt -> dict with W, idx, m, and the expected values."""
    import numpy as np
    out = {"rows": []}
    for ln in read_golden("fig1c.txt"):
        key, _, val = ln.partition(":") if ":" in ln else (ln.split()[0], "", " ".join(ln.split()[1:]))
        if ln.startswith("m "):
            out["m"] = int(ln.split()[1])
        elif ln.startswith("k "):
            out["k"] = int(ln.split()[1])
        elif ln.startswith("row"):
            a, b = val.split("|")
            out["rows"].append(([int(x) for x in a.split()], [float(x) for x in b.split()]))
        elif key == "candidates":
            out[key] = [sorted(int(x) for x in grp.split(",")) for grp in val.split()]
        else:
            out[key.strip()] = [float(x) for x in val.split()]
    out["idx"] = np.array([r[0] for r in out["rows"]], dtype=np.int32)
    out["W"] = np.array([r[1] for r in out["rows"]], dtype=np.float64)
    return out
