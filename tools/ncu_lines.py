"""Per-CUDA-source-line executed warp instructions of one kernel in an ncu report, normalised
per unit (e.g. label row): python tools/ncu_lines.py REP KERNEL_REGEX UNITS [TOP]"""
import csv, io, subprocess, sys

rep, kre, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
fname, res, tot = "", [], 0
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    elif len(r) > 8 and r[0].isdigit() and r[7].isdigit():
        n = int(r[7]); tot += n
        res.append((n, f"{fname}:{r[0]}", r[1].strip()[:100]))
res.sort(reverse=True)
print(f"total {tot / units:.1f} per unit")
for n, where, src in res[:top]:
    print(f"{n / units:7.1f}  {where:22s} {src}")
