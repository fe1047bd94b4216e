"""Per-opcode executed-instruction and stall-sample totals of one kernel in an ncu report
(`ncu -i REP --page source --csv --print-source sass`), normalised per unit (e.g. label row)."""
import csv, collections, io, re, subprocess, sys

rep, kregex, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kregex],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Instructions Executed" in r)
data = rows[rows.index(hdr) + 1:]
ie, src, st = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot, stot = 0, 0
byop, stall = collections.Counter(), collections.Counter()
for r in data:
    if len(r) <= ie or not r[ie].isdigit():
        continue
    s = re.sub(r'^@!?U?P\w+\s+', '', r[src].strip())
    op = s.split()[0] if s else '?'
    op = op if op.startswith(("SHFL", "LDG", "STG", "RED", "MUFU")) else op.split('.')[0]
    n = int(r[ie]); byop[op] += n; tot += n
    sv = int(r[st] or 0); stall[op] += sv; stot += sv
print(f"total {tot}  per unit {tot/units:.1f}")
for op, n in byop.most_common(45):
    print(f"{op:22s} {n/units:8.1f}   stall {100*stall[op]/max(stot,1):5.1f}%")
