"""CPU check of bench.py's reference arm (the fp64 oracle timed on the host, this tier's
reference implementation): it runs without a GPU and prints one JSON line with the keys
the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_the_contract_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--shape", "tiny",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["config"]["workload"] == "tiny"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_dh_mode_defaults_to_the_mode_measured_faster_for_the_loss():
    """CSC for BCE (register-gather row pass), atomic for the squared hinge."""
    code = ("import sys; sys.argv = ['bench.py'] + sys.argv[1:]; import bench; a = bench.args_(); "
            "print(a.dh_mode)")
    out = lambda *extra: subprocess.run([sys.executable, "-c", code, *extra], capture_output=True, text=True,
                                        timeout=120, cwd=ROOT).stdout.strip().splitlines()[-1]
    assert out() == "csc"
    assert out("--loss", "sqh") == "atomic"
    assert out("--dh-mode", "atomic") == "atomic"
    assert out("--loss", "sqh", "--dh-mode", "csc") == "csc"
