"""Build library variants for A/B sweeps: python tools/variants.py NAME="-DMACRO=V ..." ...
Each lands in build/libs/NAME.so (git-ignored; travels to the GPU box with gpurun) and is
selected at run time with FIXEDFANIN_LIB=build/libs/NAME.so (tools/gpu_sweep.sh)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as g  # noqa: E402


def build(spec):
    name, _, defs = spec.partition("=")
    out = os.path.join(ROOT, "build", "libs", name + ".so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = ["nvcc", *[f for f in g.NVCC_FLAGS if f != "-v" and f != "-Xptxas"], *defs.split(), "-I",
           os.path.join(ROOT, "include"), "-o", out, os.path.join(g.CSRC, "fixedfanin.cu")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return name, r.returncode, r.stderr[-2000:]


if __name__ == "__main__":
    with ThreadPoolExecutor(4) as ex:
        for name, rc, err in ex.map(build, sys.argv[1:]):
            print(name, "ok" if rc == 0 else "FAILED\n" + err)
